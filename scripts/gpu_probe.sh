cd $GRAFT_REPO_ROOT
for t in tma_stride_probe; do
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/$t scripts/$t.cu && timeout 60 /tmp/$t
echo "$t rc=$?"
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tc_sw128_test scripts/tc_sw128_test.cu && timeout 60 /tmp/tc_sw128_test
echo "rc=$?"

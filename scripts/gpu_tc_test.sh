cd $GRAFT_REPO_ROOT
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tc_gemm_test scripts/tc_gemm_test.cu && timeout 60 /tmp/tc_gemm_test
echo "rc=$?"

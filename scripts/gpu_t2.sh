cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -q 2>&1 | tail -30 > gpurun_out/t2_tests.log; echo "tile tests rc=$?"; tail -8 gpurun_out/t2_tests.log
LFM_TILE_AUTO=1 timeout 900 python -m pytest tests/test_gpu_c3_parity.py -q -x 2>&1 | tail -30 > gpurun_out/t2_c3.log; echo "c3 tiles rc=$?"; tail -8 gpurun_out/t2_c3.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
python scripts/prof_frames.py --config c3 --frames 32 --iters 1 > gpurun_out/r2o_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"mac_f16_kernel" -c 2 -o gpurun_out/r2o_mf python scripts/prof_frames.py --config c3 --frames 32 --iters 1 > gpurun_out/r2o_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2o_ncu.log

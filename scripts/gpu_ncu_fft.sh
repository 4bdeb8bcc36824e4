cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
python scripts/prof_step.py --iters 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"r2c_fast|c2r_fast" -s 4 -c 4 -o gpurun_out/prof_fft python scripts/prof_step.py --iters 2 > gpurun_out/ncu_fft.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_fft.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
LFM_SERIAL=1 python scripts/prof_step.py --iters 3 > gpurun_out/r2h_ps_serial.log 2>&1 && \
LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2h_launches_serial.csv python scripts/prof_step.py --iters 3 > gpurun_out/r2h_ncu_serial.log 2>&1
echo "serial list rc=$?"
python scripts/prof_step.py --iters 10 > gpurun_out/r2h_ps.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --launch-skip 150 --launch-count 64 --csv --log-file gpurun_out/r2h_launches_part.csv python scripts/prof_step.py --iters 10 > gpurun_out/r2h_ncu_part.log 2>&1
echo "part list rc=$?"
LFM_SERIAL=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tcdir_kernel|fwd_mac_kernel|bwd_mac_kernel" -s 4 -c 4 -o gpurun_out/r2h_full python scripts/prof_step.py --iters 3 > gpurun_out/r2h_ncu_full.log 2>&1
echo "full rc=$?"

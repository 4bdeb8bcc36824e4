# round-2 evidence: GPU tests, default bench (cpu baseline, e2e, clocks), reference arm, c5 / c4 lines, serial launch
# list of the bench plan with DRAM bytes (ncu, LFM_SERIAL=1: green-context kernels cannot be profiled), smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 2400 python -m pytest tests -q -m gpu -rs --durations=12 > gpurun_out/f_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -16 gpurun_out/f_gputest.log
LFM_PLAN_VERBOSE=1 timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_ref.json 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --config c5 --frames 32 --steps 5 --warmup 2 > gpurun_out/f_c5.json 2>&1; echo "c5 rc=$?"
timeout 900 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c4 --steps 8 --warmup 2 --no-cpu-baseline --e2e-calls 1 > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err; echo "c4 rc=$?"
LFM_SERIAL=1 python scripts/prof_step.py --iters 3 > gpurun_out/f_ps.log 2>&1 && \
LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/f_launches_serial.csv python scripts/prof_step.py --iters 3 > gpurun_out/f_ncu.log 2>&1
echo "launch list rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2

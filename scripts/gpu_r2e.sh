cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for sch in 0 1; do
  LFM_TC_SCHED=$sch timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2e_sched$sch.json 2> gpurun_out/r2e_sched$sch.err; echo "sched $sch rc=$?"
done
LFM_TC_SCHED=1 LFM_SERIAL=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2e_serial1.json 2>&1; echo "serial1 rc=$?"
LFM_SERIAL=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2e_serial0.json 2>&1; echo "serial0 rc=$?"
python scripts/prof_step.py --iters 2 > gpurun_out/r2e_ps.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2e_launches.csv python scripts/prof_step.py --iters 2 > gpurun_out/r2e_ncu.log 2>&1
echo "ncu rc=$?"

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for i in 1 2; do
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2p_bench$i.json 2> gpurun_out/r2p_bench$i.err; echo "bench rc=$?"
done
LFM_SERIAL=1 python scripts/prof_step.py --iters 3 > gpurun_out/r2p_ps_serial.log 2>&1 && \
LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2p_launches_serial.csv python scripts/prof_step.py --iters 3 > gpurun_out/r2p_ncu_serial.log 2>&1
echo "serial list rc=$?"

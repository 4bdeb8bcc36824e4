cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -q -x 2>&1 | tail -3 > gpurun_out/t9_tests.log; echo "tests rc=$?"; tail -2 gpurun_out/t9_tests.log
python scripts/prof_step.py --iters 3 > gpurun_out/t9_ps.log 2>&1 && LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/t9_launches.csv python scripts/prof_step.py --iters 3 > gpurun_out/t9_ncu.log 2>&1
echo "launch list rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t9_bench.json 2> gpurun_out/t9_bench.err; echo "bench rc=$?"
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t9_bench*.json")):
    d=json.loads(open(n).read().strip().splitlines()[-1])
    print(n, round(d["value"],1), round(d["ms_per_step"],3), d["config"].get("kernel_avg_ms"), d["clocks"]["sm_mhz"], d["config"]["sm_partitions"]["forward"])
PY

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_c3_parity.py -q -x 2>&1 | tail -5 > gpurun_out/t8_tests.log; echo "tests rc=$?"; tail -3 gpurun_out/t8_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t8_bench.json 2> gpurun_out/t8_bench.err; echo "bench rc=$?"
LFM_TC_SMS_F=0 LFM_TC_SMS_B=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t8_bench_serial.json 2> gpurun_out/t8_bench_serial.err; echo "bench serial rc=$?"
python scripts/prof_step.py --iters 3 > gpurun_out/t8_ps.log 2>&1 && LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/t8_launches.csv python scripts/prof_step.py --iters 3 > gpurun_out/t8_ncu.log 2>&1
echo "launch list rc=$?"
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t8_bench*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        print(n, round(d["value"],1), round(d["ms_per_step"],3), d["config"].get("kernel_avg_ms"), d["clocks"]["sm_mhz"], d["roofline"]["kernel"], round(d["roofline"]["frac"],3), d["roofline"].get("traffic"))
    except Exception as e: print(n, "ERR", e)
PY

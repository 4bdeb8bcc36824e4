cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -q -x 2>&1 | tail -3 > gpurun_out/t13_tests.log; echo "tests rc=$?"; tail -2 gpurun_out/t13_tests.log
LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t13_c3.json 2> gpurun_out/t13_c3.err; echo "c3 rc=$?"; grep -v "lfm plan\] tc" gpurun_out/t13_c3.err | tail -3
timeout 1200 python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t13_c4.json 2> gpurun_out/t13_c4.err; echo "c4 rc=$?"
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t13_c*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        print(n, round(d["value"],2), round(d["ms_per_step"],3), d["config"]["hybrid"], d["config"]["transform"], d["config"].get("kernel_avg_ms"), d["clocks"]["sm_mhz"], d["config"]["sm_partitions"]["forward"], d["roofline"]["kernel"], round(d["roofline"]["frac"],3))
    except Exception as e: print(n, "ERR", e)
PY
timeout 1500 python -m pytest tests/test_gpu_c3_parity.py -q -x 2>&1 | tail -3 > gpurun_out/t13_c3tests.log; echo "c3 tests rc=$?"; tail -2 gpurun_out/t13_c3tests.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t11_c5_reg.json 2> gpurun_out/t11_c5_reg.err; echo "c5 reg rc=$?"
LFM_WHOLE_WARP=1 timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t11_c5_warp.json 2> gpurun_out/t11_c5_warp.err; echo "c5 warp rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 8192 > gpurun_out/t11_c3_notiles_reg.json 2> gpurun_out/t11_c3n.err; echo "c3 notiles rc=$?"
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t11_*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        print(n, round(d["value"],1), round(d["ms_per_step"],3), d["config"].get("batch_stage_avg_ms") or d["config"].get("kernel_avg_ms"), d["clocks"]["sm_mhz"])
    except Exception as e: print(n, "ERR", e)
PY
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/t11_gpu_tests.log; echo "gpu tests rc=$?"; tail -3 gpurun_out/t11_gpu_tests.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "whole_image_75 or frames_plan or batched_frames" 2>&1 | tail -15 > gpurun_out/t17_tests.log; echo "tests rc=$?"; tail -4 gpurun_out/t17_tests.log
timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t17_c5.json 2> gpurun_out/t17_c5.err; echo "c5 rc=$?"; tail -2 gpurun_out/t17_c5.err
LFM_WHOLE_WARP=1 timeout 600 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t17_c5_warp.json 2> gpurun_out/t17_c5w.err; echo "c5 warp rc=$?"
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t17_c5*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        print(n, round(d["value"],1), round(d["ms_per_step"],3), d["config"].get("batch_stage_avg_ms"), d["clocks"]["sm_mhz"])
    except Exception as e: print(n, "ERR", e)
PY

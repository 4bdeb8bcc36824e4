cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_tiles.py -x -q 2>&1 | tail -25 > gpurun_out/t1_tests.log; echo "tile tests rc=$?"; tail -5 gpurun_out/t1_tests.log
LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 4096 > gpurun_out/t1_bench_tiles.json 2> gpurun_out/t1_bench_tiles.err; echo "bench tiles rc=$?"
LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 4100 > gpurun_out/t1_bench_tiles_fft.json 2> gpurun_out/t1_bench_tiles_fft.err; echo "bench tiles fft rc=$?"
python - <<'PY'
import json
for n in ["t1_bench_tiles","t1_bench_tiles_fft"]:
    try:
        d=json.loads(open(f"gpurun_out/{n}.json").read().strip().splitlines()[-1])
        print(n, d["value"], d["ms_per_step"], d["config"].get("hybrid"), d["config"].get("stage_avg_ms"), d.get("clocks"))
    except Exception as e: print(n, "ERR", e)
PY

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/t7_bench.json 2> gpurun_out/t7_bench.err; echo "bench rc=$?"
grep -v "lfm plan\] tc" gpurun_out/t7_bench.err | tail -5
timeout 2400 python -m pytest tests -q -m gpu --durations=12 2>&1 | tail -40 > gpurun_out/t7_gpu_tests.log; echo "gpu tests rc=$?"; tail -22 gpurun_out/t7_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python - <<'PY'
import json
d=json.loads(open("gpurun_out/t7_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["config"]["hybrid"], d["config"].get("sm_partitions"), d["e2e"]["value"], d["clocks"], d["roofline"]["kernel"], d["roofline"]["frac"])
PY

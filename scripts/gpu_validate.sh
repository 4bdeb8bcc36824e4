cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_tiles.py -q 2>&1 | tail -1; done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err; echo "bench rc=$?"
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/val_gpu_tests.log; echo "gpu tests rc=$?"; tail -2 gpurun_out/val_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python - <<'PY'
import json
d=json.loads(open("gpurun_out/val_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["config"]["hybrid"], d["config"]["sm_partitions"]["forward"], d["e2e"]["value"], d["clocks"], d["roofline"]["kernel"], round(d["roofline"]["frac"],3), d["cpu_baseline"]["value"])
PY

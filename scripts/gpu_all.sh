# full GPU suite + bench (usage: bash scripts/gpu_all.sh [bench args...])
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -rs 2>&1 | tail -8
timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "roof", d["roofline"]["kernel"], d["roofline"]["frac"])
print("stage_avg_ms", {k: round(v, 4) for k, v in d["config"]["stage_avg_ms"].items()})
print("e2e", d["e2e"]["value"], "cpu", (d["cpu_baseline"] or {}).get("value"), "clocks", d["clocks"])
PY
tail -3 gpurun_out/bench.err

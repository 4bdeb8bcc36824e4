cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "column_ranges or c3 or tc or partitions or projections or rl_tiny or isra or ht" 2>&1 | tail -2
LFM_TC_EXP=4 python scripts/prof_step.py --iters 1 2>&1 | grep "\[tc" | tail -2
for i in 1 2; do python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print(round(d['value'],2), d['clocks']['sm_mhz'], {a: round(b,3) for a,b in c['kernel_avg_ms'].items()})"; done

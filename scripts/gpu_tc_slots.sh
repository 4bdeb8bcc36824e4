cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "tc or projections or c2_operators" 2>&1 | tail -2
for a in 2 3; do
  LFM_TC_ASLOTS=$a timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/as_$a.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/as_$a.json').read().strip().splitlines()[-1]); s=d['config']['stage_avg_ms']
print('aslots $a', round(d['value'],2), 'it/s', round(d['ms_per_step'],3), 'dir_fwd', round(s['dir_fwd'],3), 'dir_bwd', round(s['dir_bwd'],3))"
done
LFM_TC_EXP=4 timeout 300 python scripts/prof_step.py --iters 1 2>&1 | grep "^\[tc" | tail -2

cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for b in 3 4 5; do
  LFM_TC_BSLOTS=$b timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/bs_$b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bs_$b.json').read().strip().splitlines()[-1]); s=d['config']['stage_avg_ms']
print('bslots $b', round(d['value'],2), 'it/s', round(d['ms_per_step'],3), 'dir_fwd', round(s['dir_fwd'],3), 'dir_bwd', round(s['dir_bwd'],3))"
done

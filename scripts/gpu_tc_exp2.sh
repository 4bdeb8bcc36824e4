cd $GRAFT_REPO_ROOT
for e in 11 43; do
  LFM_TC_EXP=$e timeout 300 python bench.py --steps 10 --warmup 2 --no-cpu-baseline --e2e-calls 1 > gpurun_out/exp_$e.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp_$e.json').read().strip().splitlines()[-1]); s=d['config']['stage_avg_ms']
print('exp $e', round(d['ms_per_step'],3), 'dir_fwd', round(s['dir_fwd'],3), 'dir_bwd', round(s['dir_bwd'],3))"
done

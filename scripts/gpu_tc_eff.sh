cd $GRAFT_REPO_ROOT
for e in 0.56 0.75 0.95; do
  LFM_TC_EFF=$e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/eff_$e.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/eff_$e.json').read().strip().splitlines()[-1]); s=d['config']['stage_avg_ms']
print('eff $e', round(d['value'],2), 'it/s', round(d['ms_per_step'],3), d['config']['hybrid'], 'dir', round(s['dir_fwd'],3), round(s['dir_bwd'],3), 'mac', round(s['fwd_mac'],3), round(s['bwd_mac'],3))"
done

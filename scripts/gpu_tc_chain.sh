cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "tc or projections or c2_operators or adjoint or isra or supplied" 2>&1 | tail -3
for ck in 8 16; do
  echo "== chain $ck"
  LFM_TC_CHAIN=$ck timeout 600 python scripts/tc_err.py s15 c2 2>&1 | grep -v Warn
  LFM_TC_CHAIN=$ck timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/ck_$ck.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ck_$ck.json').read().strip().splitlines()[-1]); s=d['config']['stage_avg_ms']
print('chain $ck', round(d['value'],2), 'it/s', round(d['ms_per_step'],3), 'dir_fwd', round(s['dir_fwd'],3), 'dir_bwd', round(s['dir_bwd'],3))"
done

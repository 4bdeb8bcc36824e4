cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
python scripts/tc_err.py s15 c2 2>&1 | tail -12
for r in 1 2; do for fb in model 96:104 96:112; do
  if [ $fb = model ]; then unset LFM_TC_SMS_F LFM_TC_SMS_B; else export LFM_TC_SMS_F=${fb%:*} LFM_TC_SMS_B=${fb#*:}; fi
  LFM_PLAN_VERBOSE=1 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print('split', '$fb', [c['sm_partitions'][x]['tc_sms'] for x in ('forward','backward')], round(d['value'],2), d['clocks']['sm_mhz'], {a: round(b,3) for a,b in c['kernel_avg_ms'].items()})"
done; done

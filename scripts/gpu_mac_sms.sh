cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for n in 148 96 74 56 40 28; do
  LFM_MAC_SMS=$n timeout 300 python bench.py --steps 10 --warmup 2 --no-cpu-baseline --e2e-calls 1 --flags 4 > gpurun_out/ms_$n.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ms_$n.json').read().strip().splitlines()[-1]); s=d['config']['stage_avg_ms']
print('mac sms $n', 'fwd_mac', round(s['fwd_mac'],3), 'ms', round(d['roofline']['achieved'],0), 'GB/s')"
done

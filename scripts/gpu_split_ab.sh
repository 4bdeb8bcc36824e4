# A/B of partition sizes in one call: PAIRS="F:B ..." (tensor-core SMs forward:backward), alternating, REPS times
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for r in $(seq ${REPS:-2}); do
 for fb in ${PAIRS:-96:104 96:112 104:104 104:112}; do
  f=${fb%:*}; b=${fb#*:}
  LFM_TC_SMS_F=$f LFM_TC_SMS_B=$b python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print('split', '$fb', round(d['value'],2), d['clocks']['sm_mhz'], {a: round(b,3) for a,b in c['kernel_avg_ms'].items()})"
 done
done

# c3 backward partition size sweep with the forward one after the other (LFM_TC_SMS_F / _B, dev)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
for fb in "0 24" "0 32" "0 40" "0 0"; do
  set -- $fb
  LFM_TC_SMS_F=$1 LFM_TC_SMS_B=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/sf.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sf.json').read().strip().splitlines()[-1]); c=d['config']
print('$1 $2', round(d['value'],1), round(d['e2e']['value'],1), c['sm_partitions']['backward'], d['clocks']['reasons'])"
done
done

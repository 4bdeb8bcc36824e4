# c3: each half of the partitioned projections alone on its partition (LFM_PART_SKIP, timing only, wrong results)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sk in 0 1 2; do
  LFM_PART_SKIP=$sk timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ps.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ps.json').read().strip().splitlines()[-1]); c=d['config']
print('skip $sk', round(d['value'],1), {k:round(x,3) for k,x in c['stage_avg_ms'].items() if x>0.03}, {k:round(x,3) for k,x in c['kernel_avg_ms'].items()})"
done

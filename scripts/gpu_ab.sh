# same-box A/B of two builds of liblfm.so (ab_tmp/liblfm_{A,B}.so), alternating c3 bench runs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in A B A B; do
  cp ab_tmp/liblfm_$v.so paper_2208_11422_b200/liblfm.so
  for env in "" "LFM_SERIAL=1"; do
    env $env timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); c=d['config']
print('$v $env', round(d['value'],1), round(d['e2e']['value'],1), {k:round(x,3) for k,x in c['stage_avg_ms'].items() if x>0.03}, {k:round(x,3) for k,x in c['kernel_avg_ms'].items()})"
  done
done

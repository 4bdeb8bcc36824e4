# same-box A/B of two builds of liblfm.so (ab_tmp/liblfm_{A,B}.so), alternating c3 bench runs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in A B A B A B A B; do
  cp ab_tmp/liblfm_$v.so paper_2208_11422_b200/liblfm.so
  timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:round(x,3) for k,x in d['config']['stage_avg_ms'].items() if x>0.03})"
done

# partition check: c3 default plan (verbose planner), c2 at backward 32 vs 40 tc SMs, c4 planner choice
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
show() { python -c "
import json; d=json.loads(open('gpurun_out/sf.json').read().strip().splitlines()[-1]); c=d['config']
print('$1', round(d['value'],1), c['sm_partitions']['forward'], c['sm_partitions']['backward'], {k:round(x,3) for k,x in c['stage_avg_ms'].items() if x>0.05})"; }
for i in 1 2; do LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sf.json 2> gpurun_out/sf_c3.err; show c3-default; done
grep "tiles, direction" gpurun_out/sf_c3.err
for b in 32 40 32 40; do LFM_TC_SMS_F=32 LFM_TC_SMS_B=$b timeout 600 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sf.json 2>/dev/null; show c2-B$b; done
LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sf.json 2> gpurun_out/sf_c2.err; show c2-default; grep "tiles, direction" gpurun_out/sf_c2.err
LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --config c4 --steps 6 --warmup 2 --no-cpu-baseline --e2e-calls 1 > gpurun_out/sf.json 2> gpurun_out/sf_c4.err; show c4-default; grep "tiles, direction" gpurun_out/sf_c4.err

# default plan on c2 / c3 / c4 with the planner's partition choice printed; tile + partition parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py tests/test_gpu_c3_parity.py -q -x -k "tile or c3 or c2 or partition or host or c4" > gpurun_out/sc_tests.log 2>&1; tail -1 gpurun_out/sc_tests.log
for c in c3 c2 c3 c2 c4; do
  LFM_PLAN_VERBOSE=1 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 2 > gpurun_out/sc.json 2> gpurun_out/sc.err
  python -c "
import json; d=json.loads(open('gpurun_out/sc.json').read().strip().splitlines()[-1]); c=d['config']
print('$c', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['reasons'], c['sm_partitions']['forward']['tc_sms'], c['sm_partitions']['backward']['tc_sms'])"
done

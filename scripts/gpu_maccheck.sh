# a tile / frames MAC change: tile + frames parity tests, c3 / c5 / c2 bench, serialised launch list of c3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py tests/test_gpu_c3_parity.py -q -x -k "tile or frames or batched or c3 or c2 or host" > gpurun_out/mc_tests.log 2>&1; tail -2 gpurun_out/mc_tests.log
for c in c3 c3 c5 c2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mc_$c.json 2>/dev/null; echo "$c rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/mc_$c.json').read().strip().splitlines()[-1]); c=d['config']
print('$c', round(d['value'],1), (d.get('e2e') or {}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:round(x,3) for k,x in (c.get('stage_avg_ms') or c.get('batch_stage_avg_ms') or {}).items() if x>0.03}, c.get('kernel_avg_ms'))"
done
LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/mc_launches.csv python scripts/prof_step.py --iters 2 > gpurun_out/mc_ncu.log 2>&1; echo "ncu rc=$?"
tail -1 gpurun_out/mc_tests.log

cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "partitions or c3 or projections or rl_tiny or graph or device_loop" 2>&1 | tail -2
for i in 1 2; do LFM_PLAN_VERBOSE=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; grep "lfm plan" gpurun_out/b.err; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], {a: round(b,3) for a,b in c['stage_avg_ms'].items() if b > 0.01}, c['kernel_avg_ms'])"; done

cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q -k "memory_aware or projections" 2>&1 | tail -3
timeout 1500 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "c4 rc=$?"; tail -5 gpurun_out/bench_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], c.get('hybrid'), c.get('plan_ms'), c.get('transfer_matrix_gb_per_gpu'))
print({k: round(v,3) for k,v in c.get('stage_avg_ms',{}).items()})"

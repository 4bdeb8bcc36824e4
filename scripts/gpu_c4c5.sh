# c4 (one GPU, memory-aware hybrid, SM partitions if the model picks them) and c5 (frame-batched) bench lines
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
LFM_PLAN_VERBOSE=1 timeout 1500 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "c4 rc=$?"; grep "lfm plan" gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['ms_per_step'], c.get('hybrid'), c.get('plan_ms'), c.get('sm_partitions'), c.get('kernel_avg_ms'))"
timeout 900 python bench.py --config c5 --frames 16 --steps 5 --warmup 2 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_c5.json').read().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['config']['batch_stage_avg_ms'].items()})"
tail -2 gpurun_out/bench_c5.err

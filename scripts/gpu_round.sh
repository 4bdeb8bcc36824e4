# full GPU round: tests, c3 bench (eager and graphs), tiny/c2 timing
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rs 2>&1 | tail -4
for FL in 0 32; do
timeout 900 python bench.py --steps 30 --no-cpu-baseline --flags $FL > gpurun_out/bench_f$FL.json 2> gpurun_out/bench_f$FL.err; echo "flags=$FL rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_f$FL.json').read().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
done
for C in tiny c2; do for FL in 0 32; do
timeout 300 python bench.py --config $C --steps 50 --no-cpu-baseline --flags $FL > gpurun_out/bench_${C}_f$FL.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_${C}_f$FL.json').read().splitlines()[-1]); print('$C flags=$FL', round(d['value'],1), 'it/s', round(d['ms_per_step'],3), 'ms')"
done; done

cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for C in tiny c2 c3; do for FL in 0 32 128; do
  ST=50; [ $C = c3 ] && ST=20
  timeout 600 python bench.py --config $C --steps $ST --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags $FL > gpurun_out/dl_${C}_$FL.json 2> gpurun_out/dl_${C}_$FL.err
  python -c "import json; d=json.loads(open('gpurun_out/dl_${C}_$FL.json').read().strip().splitlines()[-1]); print('$C flags=$FL', round(d['value'],1), 'it/s', round(d['ms_per_step'],4), 'ms  e2e', round(d['e2e']['value'],1))" || tail -3 gpurun_out/dl_${C}_$FL.err
done; done

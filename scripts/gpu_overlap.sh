# SM-partitioned projections (§5.5): parity subset, then c3 bench across partition sizes and serial (LFM_SERIAL=1)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-c3 or projections or rl_tiny or graph or device_loop}" 2>&1 | tail -3
for v in ${SWEEP:-serial 80 96 104 112}; do
  if [ $v = serial ]; then export LFM_SERIAL=1; else unset LFM_SERIAL; export LFM_TC_SMS=$v; fi
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $BENCHARGS > gpurun_out/ov_$v.json 2> gpurun_out/ov_$v.err
  echo "tc_sms=$v rc=$?"
  python - $v <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ov_{v}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("no json", e); print(open(f"gpurun_out/ov_{v}.err").read()[-2000:]); sys.exit()
print(f"value {d['value']:.2f} it/s ms {d['ms_per_step']:.3f} e2e {d['e2e']['value']:.2f}")
print({k: round(v,3) for k,v in d['config'].get('stage_avg_ms',{}).items()})
PY
done
unset LFM_SERIAL LFM_TC_SMS

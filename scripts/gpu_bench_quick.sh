# quick c3 bench variants (no cpu baseline): default flags and the ones given as arguments
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for f in 0 "$@"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --flags $f --no-cpu-baseline > gpurun_out/bq_$f.json 2> gpurun_out/bq_$f.err
  echo "flags=$f rc=$?"
  python - "$f" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/bq_{f}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("no json", e); print(open(f"gpurun_out/bq_{f}.err").read()[-2000:]); sys.exit()
c=d["config"]
print(f"value {d['value']:.2f} it/s  ms {d['ms_per_step']:.3f} frac {d['roofline']['frac']:.3f} e2e {d['e2e']['value']:.2f}")
print("hybrid", c.get("hybrid"), "plan_ms", c.get("plan_ms"), "e2e", d['e2e'])
print({k: round(v,3) for k,v in c.get("stage_avg_ms",{}).items()})
PY
done

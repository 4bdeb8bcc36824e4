# dev: partition sizes (LFM_TC_SMS_F / _B) -- each half alone (LFM_PART_SKIP=1 MAC only, 2 tensor cores only) and both
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for v in ${SMS:-88 96 104 112 120}; do
 for sk in ${SKIPS:-0 1 2}; do
  LFM_TC_SMS_F=$v LFM_TC_SMS_B=$v LFM_PART_SKIP=$sk timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pe.json 2> gpurun_out/pe.err
  python - $v $sk <<'PY'
import json,sys
try:
    d=json.loads(open("gpurun_out/pe.json").read().strip().splitlines()[-1])
except Exception as ex:
    print("fail", ex, open("gpurun_out/pe.err").read()[-1500:]); sys.exit()
c=d['config']; k=c['kernel_avg_ms']; st=c['stage_avg_ms']
print("tc_sms",sys.argv[1],"skip",sys.argv[2], "it/s %.2f"%d['value'],
      "fwd region %.3f bwd region %.3f"%(st['fwd_mac'], st['bwd_mac']), {a: round(b,3) for a,b in k.items()})
PY
 done
done

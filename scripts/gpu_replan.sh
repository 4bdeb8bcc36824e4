# dev: more planes on the frequency path under SM partitions (LFM_TC_EFF lowers the tensor-core plane estimate)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for eff in ${EFFS:-0.55 0.45}; do
 for v in ${SMS:-80 88 96 104}; do
  LFM_TC_EFF=$eff LFM_TC_SMS_F=$v LFM_TC_SMS_B=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pe.json 2> gpurun_out/pe.err
  python - $eff $v <<'PY'
import json,sys
try:
    d=json.loads(open("gpurun_out/pe.json").read().strip().splitlines()[-1])
except Exception as ex:
    print("fail", ex, open("gpurun_out/pe.err").read()[-1500:]); sys.exit()
c=d['config']; k=c['kernel_avg_ms']; st=c['stage_avg_ms']
print("eff",sys.argv[1],"tc_sms",sys.argv[2], "it/s %.2f"%d['value'], "tc_planes", c['hybrid']['tc_planes'],
      "fwd %.3f bwd %.3f"%(st['fwd_mac'], st['bwd_mac']), {a: round(b,3) for a,b in k.items()})
PY
 done
done

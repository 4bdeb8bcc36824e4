# dev timing of the SM-partitioned projections: LFM_OV_SKIP=1 times the MAC partition alone, 2 the tensor-core one
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for co in 0; do
 for sk in ${SKIPS:-1 0}; do
  for v in ${SMS:-96 112}; do
   LFM_OV_SKIP=$sk LFM_TC_SMS_F=$v LFM_TC_SMS_B=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sk.json 2> gpurun_out/sk.err
   python - $co $sk $v <<'PY'
import json,sys
d=json.loads(open("gpurun_out/sk.json").read().strip().splitlines()[-1])
st=d['config'].get('stage_avg_ms',{})
print("fwd_co",sys.argv[1],"skip",sys.argv[2],"tc_sms",sys.argv[3], "fwd", round(st['fwd_mac'],3), "bwd", round(st['bwd_mac'],3), "it/s", round(d['value'],2))
PY
  done
 done
done

# dev: partitioned projections -- kernel times with both halves, each half alone (LFM_PART_SKIP), with and without
# the tcgen05 L2 evict-last hint (LFM_TC_EXP=8 turns it off); extra env via EXTRA
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for e in ${EXPS:-0 8}; do
 for sk in ${SKIPS:-0 1 2}; do
  env $EXTRA LFM_TC_EXP=$e LFM_PART_SKIP=$sk timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pe.json 2> gpurun_out/pe.err
  python - $e $sk <<'PY'
import json,sys
try:
    d=json.loads(open("gpurun_out/pe.json").read().strip().splitlines()[-1])
except Exception as ex:
    print("fail", ex, open("gpurun_out/pe.err").read()[-1500:]); sys.exit()
c=d['config']; k=c['kernel_avg_ms']; st=c['stage_avg_ms']
print("tcexp",sys.argv[1],"skip",sys.argv[2], "it/s %.2f"%d['value'], "parts", [c['sm_partitions'][x]['tc_sms'] for x in ('forward','backward')],
      "fwd region %.3f bwd region %.3f"%(st['fwd_mac'], st['bwd_mac']), {a: round(b,3) for a,b in k.items()})
PY
 done
done

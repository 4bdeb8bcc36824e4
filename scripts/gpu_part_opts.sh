# dev: placement of staging / R2C (inside the partitions) and C2R (after the join): LFM_PART_OPTS 0..3
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for o in ${OPTS:-0 1 2 3 0 1 2 3}; do
  LFM_PART_OPTS=$o timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/po.json 2> gpurun_out/po.err
  python - $o <<'PY'
import json,sys
d=json.loads(open("gpurun_out/po.json").read().strip().splitlines()[-1])
c=d['config']; k=c['kernel_avg_ms']; st=c['stage_avg_ms']
print("opts",sys.argv[1], "it/s %.2f"%d['value'], "clk", d['clocks']['sm_mhz'], {a: round(b,3) for a,b in st.items() if b > 0.01})
PY
done

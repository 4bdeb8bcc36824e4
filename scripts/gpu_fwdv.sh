# dev: forward MAC variants (LFM_FWD_V) alone on the MAC partition (LFM_OV_SKIP=1) and on the whole GPU (LFM_SERIAL=1)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for fv in ${FVS:-0 1 2 3 4 5}; do
  LFM_FWD_V=$fv LFM_OV_SKIP=1 LFM_TC_SMS=96 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sk.json 2> gpurun_out/sk.err
  a=$(python -c "import json; d=json.loads(open('gpurun_out/sk.json').read().strip().splitlines()[-1]); print(round(d['config']['stage_avg_ms']['fwd_mac'],3))")
  LFM_FWD_V=$fv LFM_SERIAL=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sk.json 2> gpurun_out/sk.err
  b=$(python -c "import json; d=json.loads(open('gpurun_out/sk.json').read().strip().splitlines()[-1]); print(round(d['config']['stage_avg_ms']['fwd_mac'],3))")
  echo "fwd_v $fv partition52 $a full $b"
done

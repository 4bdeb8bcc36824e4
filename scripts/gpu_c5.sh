cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
for F in ${FRAMES:-16}; do
timeout 900 python bench.py --config c5 --frames $F --steps 5 --warmup 2 $C5ARGS > gpurun_out/c5_$F.json 2> gpurun_out/c5_$F.err; echo "F=$F rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c5_$F.json').read().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['auto_stop'], {k: round(v,2) for k,v in d['config']['batch_stage_avg_ms'].items()})"
tail -2 gpurun_out/c5_$F.err
done

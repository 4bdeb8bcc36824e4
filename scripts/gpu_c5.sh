cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out
for F in 4 8 16; do
timeout 600 python bench.py --config c5 --frames $F --steps 5 --warmup 2 > gpurun_out/c5_$F.json 2> gpurun_out/c5_$F.err; echo "F=$F rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/c5_$F.json').read().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['config']['auto_stop'])"
tail -2 gpurun_out/c5_$F.err
done

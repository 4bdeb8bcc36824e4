# c5 frame-batched: parity (batched vs single frame) and the F=16 bench line
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batched" 2>&1 | tail -2
timeout 900 python bench.py --config c5 --frames 16 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_c5.json').read().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['config']['batch_stage_avg_ms'].items()})"

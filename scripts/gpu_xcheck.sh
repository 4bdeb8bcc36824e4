# quick check of a transform-kernel change: tile parity tests, c3 bench, c4 bench, serial launch list of c3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py -q -x -k "tile or c3 or c2 or host" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/xc_bench$i.json 2> gpurun_out/xc_bench$i.err; echo "bench rc=$?"; done
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/xc_c4.json 2> gpurun_out/xc_c4.err; echo "c4 rc=$?"
python - <<'PY'
import json
for f in ["xc_bench1","xc_bench2","xc_c4"]:
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["value"],1), round(d["ms_per_step"],3), d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e: print(f, "ERR", e)
PY
LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/xc_launches.csv python scripts/prof_step.py --iters 2 > gpurun_out/xc_ncu.log 2>&1; echo "ncu rc=$?"

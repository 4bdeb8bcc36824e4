cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -q -x 2>&1 | tail -30 > gpurun_out/t4_tests.log; echo "tile tests rc=$?"; tail -4 gpurun_out/t4_tests.log
python scripts/prof_step.py --iters 3 --flags 4096 > gpurun_out/t4_ps.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/t4_launches.csv python scripts/prof_step.py --iters 3 --flags 4096 > gpurun_out/t4_ncu.log 2>&1
echo "launch list rc=$?"
for fb in "0 0" "48 64" "56 56" "40 56"; do set -- $fb
LFM_TC_SMS_F=$1 LFM_TC_SMS_B=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 4096 > gpurun_out/t4_b_$1_$2.json 2> gpurun_out/t4_b_$1_$2.err; echo "bench $1 $2 rc=$?"
done
LFM_C2R_FULL=1 LFM_TC_SMS_F=48 LFM_TC_SMS_B=64 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 4096 > gpurun_out/t4_b_c2rfull.json 2> gpurun_out/t4_b_c2rfull.err
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t4_b_*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        print(n, round(d["value"],1), round(d["ms_per_step"],3), {k:round(v,3) for k,v in d["config"].get("stage_avg_ms").items() if v>0.01}, d["config"].get("kernel_avg_ms"), d["clocks"]["sm_mhz"])
    except Exception as e: print(n, "ERR", e)
PY

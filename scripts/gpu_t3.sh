cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py -q 2>&1 | tail -30 > gpurun_out/t3_tests.log; echo "tile tests rc=$?"; tail -4 gpurun_out/t3_tests.log
python scripts/prof_step.py --iters 3 --flags 4096 > gpurun_out/t3_ps.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/t3_launches.csv python scripts/prof_step.py --iters 3 --flags 4096 > gpurun_out/t3_ncu.log 2>&1
echo "launch list rc=$?"
for fb in "64 64" "80 80" "96 96" "48 64" "72 88"; do set -- $fb
LFM_TC_SMS_F=$1 LFM_TC_SMS_B=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 4096 > gpurun_out/t3_b_$1_$2.json 2> gpurun_out/t3_b_$1_$2.err; echo "bench $1 $2 rc=$?"
done
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t3_b_*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        print(n, round(d["value"],1), round(d["ms_per_step"],3), d["config"].get("sm_partitions"), {k:round(v,3) for k,v in d["config"].get("stage_avg_ms").items()}, d["config"].get("kernel_avg_ms"), d["clocks"]["sm_mhz"])
    except Exception as e: print(n, "ERR", e)
PY

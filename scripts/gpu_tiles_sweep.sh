cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for fb in "24 24" "32 32" "40 40" "32 40" "16 24" "0 0"; do set -- $fb
LFM_TC_SMS_F=$1 LFM_TC_SMS_B=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/sweep_b_$1_$2.json 2> gpurun_out/sweep_b_$1_$2.err; echo "bench $1 $2 rc=$?"
done
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/sweep_b_*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        st=d["config"]["stage_avg_ms"]
        print(n, round(d["value"],1), round(d["ms_per_step"],3), round(st["fwd_mac"],3), round(st["bwd_mac"],3), {k: round(v,3) for k,v in d["config"].get("kernel_avg_ms").items()}, d["clocks"]["sm_mhz"])
    except Exception as e: print(n, "ERR", e)
PY
python scripts/prof_step.py --iters 3 > gpurun_out/sweep_ps.log 2>&1 && LFM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sweep_launches.csv python scripts/prof_step.py --iters 3 > gpurun_out/sweep_ncu.log 2>&1
echo "launch list rc=$?"

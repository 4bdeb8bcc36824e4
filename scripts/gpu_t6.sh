cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pf in 0 8 16 32; do
LFM_MF_PF=$pf LFM_TC_SMS_F=0 LFM_TC_SMS_B=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 4096 > gpurun_out/t6_s_pf$pf.json 2> gpurun_out/t6_s_pf$pf.err; echo "serial pf$pf rc=$?"
LFM_MF_PF=$pf LFM_TC_SMS_F=56 LFM_TC_SMS_B=56 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-calls 1 --flags 4096 > gpurun_out/t6_p_pf$pf.json 2> gpurun_out/t6_p_pf$pf.err; echo "part pf$pf rc=$?"
done
LFM_MF_PF=16 timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-calls 1 > gpurun_out/t6_c5_pf16.json 2> gpurun_out/t6_c5.err; echo "c5 rc=$?"
python - <<'PY'
import json,glob
for n in sorted(glob.glob("gpurun_out/t6_*.json")):
    try:
        d=json.loads(open(n).read().strip().splitlines()[-1])
        print(n, round(d["value"],1), round(d["ms_per_step"],3), d["config"].get("kernel_avg_ms") or d["config"].get("batch_stage_avg_ms"), d["clocks"]["sm_mhz"])
    except Exception as e: print(n, "ERR", e)
PY

# A/B of LFM_TC_EXP values on the c3 bench, alternating (usage: EXPS="0 16 0 16" bash scripts/gpu_tcab.sh)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
for e in ${EXPS:-0 16 0 16 0 16}; do LFM_TC_EXP=$e python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print('exp', $e, round(d['value'],2), d['clocks']['sm_mhz'], {a: round(b,3) for a,b in c['kernel_avg_ms'].items()})"; done

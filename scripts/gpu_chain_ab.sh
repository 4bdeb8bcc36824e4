# A/B of the TMEM drain-group length (LFM_TC_CHAIN K-steps) on c3, plus the tensor-core parity tests at the longest
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
LFM_TC_CHAIN=${TESTCHAIN:-32} timeout 900 python -m pytest tests -m gpu -x -q -k "tc or c3 or c4_geometry or rl_tiny or auto_stop" 2>&1 | tail -2
for r in 1 2; do for ch in ${CHAINS:-16 24 32}; do
  LFM_TC_CHAIN=$ch python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print('chain', $ch, round(d['value'],2), d['clocks']['sm_mhz'], {a: round(b,3) for a,b in c['kernel_avg_ms'].items()})"
done; done

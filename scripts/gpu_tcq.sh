# quick: c3 bench x2 with kernel times (LFM_TC_EXP passes through)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "${TESTK:-column_ranges or c3_forward}" 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print(d['value'], d['clocks']['sm_mhz'], c['sm_partitions']['forward']['tc_sms'], c['sm_partitions']['backward']['tc_sms'], {a: round(b,3) for a,b in c['kernel_avg_ms'].items()})"; done

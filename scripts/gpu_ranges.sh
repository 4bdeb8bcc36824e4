cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "column_ranges or partitions or tc or c3 or projections or rl_tiny" 2>&1 | tail -3
for e in 0 16 0 16; do LFM_TC_EXP=$e python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print('exp', $e, d['value'], d['clocks']['sm_mhz'], c['sm_partitions']['forward']['tc_sms'], c['sm_partitions']['backward']['tc_sms'], c['kernel_avg_ms'], d['roofline_tc']['executed_tensor_tflops'])"; done

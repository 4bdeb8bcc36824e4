cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "c3 or projections or rl_tiny" 2>&1 | tail -2
SKIPS="1 0" SMS="96 112" bash scripts/gpu_ov_skip.sh
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
c=d['config']; print(d['value'], c['sm_partitions']['forward'], c['sm_partitions']['backward']); print(c['kernel_avg_ms'])"

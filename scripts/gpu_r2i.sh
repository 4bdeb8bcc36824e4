cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c3_parity.py -q -m gpu -rs -x -k "partitions or nccl or c3_auto or c3g13 or column_ranges or graph or device_loop" 2>&1 | tail -4
python - <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2208_11422_b200 import lfm as L
from lfm_inputs import CONFIGS, OPTICS, gen_psf
cfg = CONFIGS["c2"]
h = gen_psf(cfg, np.float32)
with L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), nccl_id=L.lfm_comm_unique_id(),
            flags=L.LFM_PLAN_FORCE_COMM | L.LFM_PLAN_SYMMETRIC) as p:
    print("symmetric C1 mode on one rank:", p.info()["c1_mode"])
PY
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-calls 1 > gpurun_out/r2i_bench$i.json 2> gpurun_out/r2i_bench$i.err; echo "bench rc=$?"
done

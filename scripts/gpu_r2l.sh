cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -rs -k "repeatable" 2>&1 | tail -3
LFM_MT_PG=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -rs -k "repeatable" 2>&1 | tail -3
cat > /tmp/c5prof.py <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2208_11422_b200 import lfm as L
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume
cfg = CONFIGS["c3"]
h = gen_psf(cfg, np.float32)
plan = L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=L.LFM_PLAN_FFT_ONLY)
xt = torch.from_numpy(gen_volume(cfg, 1, np.float32)).cuda()
yh = torch.zeros((cfg.height, cfg.width), device="cuda"); plan.forward(xt, yh)
y = (yh.clamp_min(0) + 1).contiguous()
x = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
r = plan.rl_iterate(y, x, L.make_policy(mode="fixed", n_iters=2)); torch.cuda.synchronize(); print("ok")
PY
python /tmp/c5prof.py > gpurun_out/r2l_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"r2c_fast_kernel|c2r_fast_kernel" -s 4 -c 4 -o gpurun_out/r2l_fft python /tmp/c5prof.py > gpurun_out/r2l_ncu.log 2>&1
echo "ncu rc=$?"

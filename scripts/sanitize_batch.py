"""Small driver for compute-sanitizer: the frame-batched tcgen05 MACs (fmb_tc_kernel / bmb_tc_kernel) at s15, F = 16,
two lockstep RL iterations (all-frequency plan so every plane goes through the batched MACs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume  # noqa: E402
from paper_2208_11422_b200 import lfm as L  # noqa: E402

cfg = CONFIGS["s15"]
F = int(os.environ.get("FRAMES", "16"))
h = gen_psf(cfg, np.float32)
plan = L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=L.LFM_PLAN_FFT_ONLY)
xt = torch.from_numpy(gen_volume(cfg, 1, np.float32)).cuda()
yh = torch.zeros((cfg.height, cfg.width), device="cuda")
plan.forward(xt, yh)
yb = torch.stack([yh.clamp_min(0) * (1 + 0.05 * f) + 1.0 for f in range(F)]).contiguous()
xb = torch.zeros((F, cfg.nz, cfg.height, cfg.width), device="cuda")
r = plan.rl_iterate_batch(yb, xb, L.make_policy(mode="fixed", n_iters=2))
torch.cuda.synchronize()
print("ok", r["stop_iter"][:2], r["series"][0])

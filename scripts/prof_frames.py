"""Small driver for ncu: an LFM_PLAN_FRAMES plan (all planes on the fp16 batched MACs), F frames, 2 lockstep RL
iterations on a BASELINE geometry (default c2 to keep the plan small)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume  # noqa: E402
from paper_2208_11422_b200 import lfm as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--frames", type=int, default=32)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.config]
h = gen_psf(cfg, np.float32)
with L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS)) as p1:
    xt = torch.from_numpy(gen_volume(cfg, 1, np.float32)).cuda()
    yh = torch.zeros((cfg.height, cfg.width), device="cuda")
    p1.forward(xt, yh)
yb = torch.stack([yh.clamp_min(0) * (1 + 0.02 * f) + 1.0 for f in range(a.frames)]).contiguous()
plan = L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=L.LFM_PLAN_FRAMES)
xb = torch.zeros((a.frames, cfg.nz, cfg.height, cfg.width), device="cuda")
r = plan.rl_iterate_batch(yb, xb, L.make_policy(mode="fixed", n_iters=a.iters))
torch.cuda.synchronize()
print("ok", r["series"][0])

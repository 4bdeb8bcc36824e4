"""Small driver for ncu --set full: c3 plan, y = Poisson(H x_true), then `--iters` RL iterations."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson  # noqa: E402
from paper_2208_11422_b200 import lfm as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
cfg = CONFIGS[a.config]
h = gen_psf(cfg)
xt = torch.from_numpy(gen_volume(cfg, 1, np.float32)).cuda()
plan = L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=a.flags)
yh = torch.zeros((cfg.height, cfg.width), device="cuda")
plan.forward(xt, yh)
y = torch.from_numpy(poisson(np.maximum(yh.cpu().numpy(), 0), 101).astype(np.float32)).cuda()
x = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
r = plan.rl_iterate(y, x, L.make_policy(mode="fixed", n_iters=a.iters))
torch.cuda.synchronize()
print("ok", r["series"])

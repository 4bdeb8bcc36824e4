import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson
from oracle import lfm_oracle as O
from paper_2208_11422_b200 import lfm as L
cfg = CONFIGS["tiny"]; F = 4
h = gen_psf(cfg, np.float32); hd = h.astype(np.float64)
ys = [poisson(O.forward_project(gen_volume(cfg, 1 + f % 3), hd), 300 + f) for f in range(F)]
for flags in (0, 4):
    plan = L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=flags)
    print("info", {k: v for k, v in plan.info().items() if k in ("fft_units", "direct_planes", "tc_planes")})
    yb = torch.tensor(np.stack(ys), dtype=torch.float32, device="cuda")
    xb = torch.zeros((F, cfg.nz, cfg.height, cfg.width), device="cuda")
    rb = plan.rl_iterate_batch(yb, xb, L.make_policy(mode="fixed", n_iters=2))
    print(flags, rb, float(xb.abs().sum()))
    x1 = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
    print(plan.rl_iterate(yb[0].contiguous(), x1, L.make_policy(mode="fixed", n_iters=2)))

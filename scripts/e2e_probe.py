"""Dev: where the e2e (host-buffer) call spends its time at c3 -- device-only loop, host call into pinned memory
(improving iterates mirrored on a side stream) and into pageable memory (one copy at the end)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson  # noqa: E402
from paper_2208_11422_b200 import lfm as L  # noqa: E402

cfg = CONFIGS["c3"]
plan = L.Plan(gen_psf(cfg), cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS))
xt = torch.from_numpy(gen_volume(cfg, 1, np.float32)).cuda()
yh = torch.zeros((cfg.height, cfg.width), device="cuda")
plan.forward(xt, yh)
y = poisson(np.maximum(yh.cpu().numpy(), 0), 101).astype(np.float32)
y_d = torch.from_numpy(y).cuda()
pol = L.make_policy(mode="auto", max_iters=50)
x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
pinned = torch.zeros((cfg.nz, cfg.height, cfg.width), dtype=torch.float32).pin_memory()
pageable = np.zeros((cfg.nz, cfg.height, cfg.width), np.float32)
for name, fn in [("device", lambda: plan.rl_iterate(y_d, x_d, pol)),
                 ("device+d2h", lambda: (plan.rl_iterate(y_d, x_d, pol), pinned.copy_(x_d.cpu() if False else x_d))[0]),
                 ("host pinned", lambda: plan.deconvolve_host(y, pinned.numpy(), pol)),
                 ("host pageable", lambda: plan.deconvolve_host(y, pageable, pol))]:
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    k = r["stop_iter"]
    print(f"{name:14s} {k} iterations: {min(ts) * 1e3:7.2f} ms per call, {min(ts) / k * 1e3:6.3f} ms per iteration")

"""Dev: measured operator error of each path (flags) against the fp64 oracle on s15 / c2-like inputs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume  # noqa: E402
from oracle import lfm_oracle as O  # noqa: E402
from paper_2208_11422_b200 import lfm as L  # noqa: E402

for name in sys.argv[1:] or ["s15"]:
    cfg = CONFIGS[name]
    h = gen_psf(cfg)
    hd = h.astype(np.float64)
    x = gen_volume(cfg, 1, np.float32)
    rng = np.random.default_rng(5)
    r = rng.uniform(0.5, 1.5, (cfg.height, cfg.width)).astype(np.float32)
    yref = O.forward_project(x.astype(np.float64), hd)
    bref = O.backward_project(r.astype(np.float64), hd)
    for flags in (0, 18, 2, 4):
        with L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=flags) as p:
            info = p.info()
            y = torch.zeros((cfg.height, cfg.width), device="cuda")
            p.forward(torch.from_numpy(x).cuda(), y)
            b = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
            p.backward(torch.from_numpy(r).cuda(), b)
            y = y.cpu().numpy().astype(np.float64)
            b = b.cpu().numpy().astype(np.float64)
            ey = np.linalg.norm(y - yref) / np.linalg.norm(yref)
            eb = np.linalg.norm(b - bref) / np.linalg.norm(bref)
            my = np.abs(y - yref).max() / np.abs(yref).max()
            mb = np.abs(b - bref).max() / np.abs(bref).max()
            by = (y - yref).sum() / np.abs(yref).sum()
            bb = (b - bref).sum() / np.abs(bref).sum()
            print(f"{name} flags={flags:2d} tc={info['tc_planes']} fwd relL2 {ey:.2e} max {my:.2e} bias {by:+.2e} | "
                  f"bwd relL2 {eb:.2e} max {mb:.2e} bias {bb:+.2e}", flush=True)

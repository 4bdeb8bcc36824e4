"""dev: tile groups vs whole-image plan on s15 -- operators, one RL step (rl_step) and a short rl_iterate."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson  # noqa: E402
from oracle import lfm_oracle as O  # noqa: E402
from paper_2208_11422_b200 import lfm as L  # noqa: E402

cfg = CONFIGS["s15"]
h = gen_psf(cfg, np.float32)
hd = h.astype(np.float64)
y = poisson(O.forward_project(gen_volume(cfg, 1), hd), 77).astype(np.float32)
res = {}
for flags in [4 | 4096, 4 | 8192]:
    with L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=flags) as p:
        yd = torch.from_numpy(y).cuda()
        c0 = float(y.sum()) / float(O.compute_normalizer(hd, cfg.height, cfg.width).sum())
        xa = torch.full((cfg.nz, cfg.height, cfg.width), c0, device="cuda")
        xn = torch.zeros_like(xa)
        yh = torch.zeros_like(yd)
        e = p.rl_step(yd, xa, xn, yhat_out=yh)
        torch.cuda.synchronize()
        x2 = torch.zeros_like(xa)
        r = p.rl_iterate(yd, x2, L.make_policy(mode="fixed", n_iters=3))
        torch.cuda.synchronize()
        res[flags] = (e, yh.cpu().numpy(), xn.cpu().numpy(), r["series"], x2.cpu().numpy())
        print(flags, p.info()["tile_groups"], "E1", e, "series", r["series"])
a, b = res[4 | 4096], res[4 | 8192]
rel = lambda u, v: float(np.linalg.norm(u - v) / np.linalg.norm(v))
print("yhat rel", rel(a[1], b[1]), "x1 rel", rel(a[2], b[2]), "x3 rel", rel(a[4], b[4]))

# auto-stop on a side stream (as tests/test_gpu_tiles.py::test_tiled_rl_auto_stop)
for flags in [4 | 4096, 4 | 8192]:
    st = torch.cuda.Stream()
    with torch.cuda.stream(st), L.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L.make_optics(**OPTICS), flags=flags,
                                       stream=st) as p:
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        r = p.rl_iterate(torch.from_numpy(y).cuda(), x_d, L.make_policy(mode="auto", max_iters=25), stream=st)
        st.synchronize()
        print("side stream", flags, r["stop_iter"], r["best_iter"], [round(v, 6) for v in r["series"]])

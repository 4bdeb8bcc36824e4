#!/usr/bin/env python
"""Writes tests/golden/c3_auto.json: the fp64 oracle's auto-stop RL run on the c3 workload (BASELINE.json
configs[2]: Nnum=15, 1005x1005, 51 planes), used by the -m gpu test that checks the benchmarked plan's stop
iteration, best iteration, entropy series and returned volume.

Calls only oracle/ and lfm_inputs/ (no product code): y = Poisson(H_oracle x_true), then oracle.deconvolve
(P:99 stop rule, reading C15).  The volume is stored as
  * per-plane sums and per-(plane, input phase) unit sums of x_best (every (z,a) unit of the plan),
  * x_best at ~14k voxels: per plane the 4 corners, 4 edge midpoints, 150 seeded random voxels, and full image
    rows (every coarse column and phase of one row) on 6 planes.
y itself is stored as Poisson counts (uint16) in tests/golden/c3_y.npz (its sha256 in the JSON).
Takes ~45 min on 8 cores:  python scripts/make_golden_c3.py

    python scripts/make_golden_c3.py c3g13     (~15 min)
writes tests/golden/c3g13_30.json: the c3 geometry (1005x1005, Nnum=15, the c3 PSF recipe) with 13 planes, whose
tap boxes span D = 1..11 so the default plan mixes tcgen05 planes with frequency-path planes; 30 fixed RL
iterations chained from oracle.initial_volume with oracle.rl_step (the north-star 1- and 30-iteration gates): the
series E_1..E_30 and, for x_1, x_best (argmax of the series) and x_30, the same unit sums and voxel samples
(y stored in tests/golden/c3g13_y.npz).
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson  # noqa: E402
from oracle import lfm_oracle as O  # noqa: E402

VOLUME_SEED, NOISE_SEED = 1, 101
FULL_ROW_PLANES = (0, 12, 20, 25, 33, 50)


def sample_voxels(nz, H, W, seed=2024, full_rows=FULL_ROW_PLANES):
    rng = np.random.default_rng(seed)
    z, p, q = [], [], []
    fixed = [(0, 0), (0, W - 1), (H - 1, 0), (H - 1, W - 1), (0, W // 2), (H - 1, W // 2), (H // 2, 0), (H // 2, W - 1)]
    for k in range(nz):
        pts = fixed + [(int(a), int(b)) for a, b in zip(rng.integers(0, H, 150), rng.integers(0, W, 150))]
        for a, b in pts:
            z.append(k), p.append(a), q.append(b)
    for k in full_rows:
        row = int(rng.integers(0, H))
        for b in range(W):
            z.append(k), p.append(row), q.append(b)
    return np.array(z), np.array(p), np.array(q)


def y_digest(y):
    return hashlib.sha256(np.ascontiguousarray(y, np.float64).tobytes()).hexdigest()


def c3g13_config():
    import dataclasses
    return dataclasses.replace(CONFIGS["c3"], name="c3g13", nz=13, n_objects=100, background=0.05 * 9 / 13)


def volume_record(x, N, z, p, q):
    nz, H, W = x.shape
    return {"plane_sums": [math.fsum(x[i].ravel().tolist()) for i in range(nz)],
            "unit_sums": x.reshape(nz, H // N, N, W // N, N).sum(axis=(1, 3)).reshape(nz, N * N).tolist(),
            "x": x[z, p, q].tolist()}


def main_c3g13():
    cfg = c3g13_config()
    t0 = time.time()
    hd = gen_psf(cfg, np.float32).astype(np.float64)
    xt = gen_volume(cfg, VOLUME_SEED)
    y = poisson(O.forward_project(xt, hd), NOISE_SEED)
    print(f"y formed ({time.time() - t0:.0f} s)", flush=True)
    reg = O.cutoff_region(O.Optics(nnum=cfg.nnum, **OPTICS), cfg.height, cfg.width)
    norm = O.compute_normalizer(hd, cfg.height, cfg.width)
    x = O.initial_volume(y, hd, cfg.nz, cfg.height, cfg.width)
    series, x1, xbest, best = [], None, None, -math.inf
    for k in range(1, 31):
        x, _ = O.rl_step(x, y, hd, norm)
        e = O.evaluate_iteration(x, reg)
        series.append(e)
        if k == 1:
            x1 = x.copy()
        if e > best:
            best, xbest = e, x.copy()
        print(f"  k={k} E={e:.9f} ({time.time() - t0:.0f} s)", flush=True)
    z, p, q = sample_voxels(cfg.nz, cfg.height, cfg.width, full_rows=(0, 3, 5, 6, 9, 12))
    N = cfg.nnum
    out = {
        "what": "fp64 oracle: 30 RL iterations on the c3 geometry with 13 planes (scripts/make_golden_c3.py c3g13)",
        "cite": "S:269 RL update (reading C1), S:287 initial volume (C2), Eq. 12 P:97 metric; BASELINE north star "
                "(rel-L2 <= 1e-4 after 1 iteration, <= 1e-3 after 30)",
        "recipe": {"config": "dataclasses.replace(CONFIGS['c3'], name='c3g13', nz=13, n_objects=100, "
                             "background=0.05*9/13)",
                   "x_true": f"gen_volume(cfg, {VOLUME_SEED})", "y": f"poisson(oracle.forward_project(x_true, psf), {NOISE_SEED})",
                   "optics": OPTICS},
        "y_sha256": y_digest(y), "y_sum": float(y.sum()), "series": series,
        "best_iter": int(np.argmax(series)) + 1,
        "samples": {"z": z.tolist(), "p": p.tolist(), "q": q.tolist()},
        "x1": volume_record(x1, N, z, p, q), "x_best": volume_record(xbest, N, z, p, q), "x30": volume_record(x, N, z, p, q),
        "seconds": time.time() - t0,
    }
    assert float(y.max()) < 65536 and np.array_equal(y, np.round(y))
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3g13_y.npz"), y=y.astype(np.uint16))
    path = os.path.join(ROOT, "tests", "golden", "c3g13_30.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB, {time.time() - t0:.0f} s)")


def main():
    cfg = CONFIGS["c3"]
    t0 = time.time()
    hd = gen_psf(cfg, np.float32).astype(np.float64)
    xt = gen_volume(cfg, VOLUME_SEED)
    y = poisson(O.forward_project(xt, hd), NOISE_SEED)
    print(f"y formed ({time.time() - t0:.0f} s)", flush=True)
    opt = O.Optics(nnum=cfg.nnum, **OPTICS)
    res = O.deconvolve(y, hd, opt, O.Policy(mode="auto", max_iters=50))
    print(f"deconvolve: stop {res.stop_iter} best {res.best_iter} ({time.time() - t0:.0f} s)", flush=True)
    x = res.volume
    s = res.series
    k = res.stop_iter
    margin = min(abs(s[i] - s[i - 1]) / abs(s[i]) for i in range(1, k)) if k > 1 else None
    N = cfg.nnum
    unit_sums = x.reshape(cfg.nz, cfg.height // N, N, cfg.width // N, N).sum(axis=(1, 3))   # [z][a1][a2]
    z, p, q = sample_voxels(cfg.nz, cfg.height, cfg.width)
    out = {
        "what": "fp64 oracle auto-stop RL on c3 (scripts/make_golden_c3.py; oracle/ + lfm_inputs/ only)",
        "cite": "P:99 stop rule (reading C15), Fig. 2d P:103-105; S:284-299 deconvolve; S:269 RL update",
        "recipe": {"config": "c3", "psf": "lfm_inputs.gen_psf(CONFIGS['c3'], float32) as float64",
                   "x_true": f"lfm_inputs.gen_volume(CONFIGS['c3'], {VOLUME_SEED})",
                   "y": f"lfm_inputs.poisson(oracle.forward_project(x_true, psf), {NOISE_SEED})",
                   "policy": "auto, max_iters 50, min_iters 2, patience 1, eps 1e-6, triangle region",
                   "optics": OPTICS},
        "y_sha256": y_digest(y), "y_sum": float(y.sum()),
        "stop_iter": res.stop_iter, "best_iter": res.best_iter, "series": list(s), "decision_margin": margin,
        "plane_sums": [math.fsum(x[i].ravel().tolist()) for i in range(cfg.nz)],
        "unit_sums": unit_sums.reshape(cfg.nz, N * N).tolist(),
        "samples": {"z": z.tolist(), "p": p.tolist(), "q": q.tolist(), "x": x[z, p, q].tolist()},
        "seconds": time.time() - t0,
    }
    assert float(y.max()) < 65536 and np.array_equal(y, np.round(y))
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3_y.npz"), y=y.astype(np.uint16))
    path = os.path.join(ROOT, "tests", "golden", "c3_auto.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB, {time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main_c3g13() if sys.argv[1:] == ["c3g13"] else main()

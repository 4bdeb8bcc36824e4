"""Seeded synthetic inputs for the light-field RL hot path (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no projection, no RL update, no metric): only the
synthetic PSF bank, phantom volumes, model-free light-field-like images and Poisson sampling that
SPEC.md's phantom module describes and SURVEY.md §8(d) sizes.  Both the oracle side
(tests) and the CUDA side (bench / tests) draw their inputs from here; measurements that need the
forward model y = Poisson(H x_true) are formed by the caller with whichever projector it is allowed
to use (the oracle in tests, the product in bench.py -- see DESIGN.md §4).

Recipes:
  * PSF  -- Gaussian with parallax: sigma(z) = sigma0 + slope*|z - zc|, centre shifted by
            shear*(z - zc)*((a,b) - (c,c))/N, support K(z) = N*(2 r(z) + 1) with
            r(z) = round(r_max*|z - zc|/zc), zero-padded to K_max, each kernel normalised to sum 1
            (reading C7).  Separable, so the 5-D bank is an outer product of 1-D factors.
  * beads   -- hard spheres for tiny / c2.
  * somata  -- neuron-like ellipsoids, lateral radius 3 +- 40 % px, axial half-thickness ~1.5 planes,
               intensity U(0.3,1)*scale, plus a uniform background for c3 / c4.
  * lf_like -- a model-free positive image with light-field-like lenslet structure used where a
               parity test needs a full-size y without running any projector.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    nnum: int
    height: int
    width: int
    nz: int
    k_max: int
    r_max: int
    sigma0: float
    slope: float
    shear: float
    n_iters: int          # fixed-mode iteration count of the BASELINE config (0 = auto-stop)
    phantom: str          # "beads" | "somata"
    n_objects: int
    radius: float
    photons: float        # peak scale
    background: float     # per-voxel uniform background as a fraction of `photons`


# BASELINE.json configs; PSF sizes are the survey's proposals (the paper gives none).
CONFIGS = {
    "tiny": Config("tiny", 3, 33, 33, 3, 9, 1, 1.0, 0.6, 1.0, 10, "beads", 3, 1.5, 200.0, 0.0),
    "c2": Config("c2", 11, 319, 319, 21, 99, 4, 1.5, 0.9, 1.5, 8, "beads", 12, 2.0, 200.0, 0.0),
    "c3": Config("c3", 15, 1005, 1005, 51, 165, 5, 2.0, 0.95, 2.0, 0, "somata", 400, 3.0, 50.0,
                 0.05 * 9 / 51),
    "c4": Config("c4", 15, 2025, 2025, 101, 225, 7, 2.0, 0.6, 2.0, 0, "somata", 1600, 3.0, 50.0,
                 0.05 * 9 / 101),
    # scaled N=15 geometry the oracle can run to auto-stop in seconds (SURVEY App. A4 regime)
    "s15": Config("s15", 15, 225, 225, 9, 75, 2, 2.0, 1.5, 3.0, 0, "somata", 25, 3.0, 50.0, 0.05),
}

# 20x / 0.5 NA water objective, d_ML = 150 um, lambda = 0.52 um (zebrafish-like)
OPTICS = dict(wavelength_um=0.52, na=0.5, mla_pitch_um=150.0, magnification=20.0)


def support_radius(cfg: Config, z: int) -> int:
    """r(z) = round(r_max*|z - zc|/zc); K(z) = N*(2 r(z) + 1) <= K_max."""
    zc = (cfg.nz - 1) / 2.0
    if zc == 0:
        return 0
    return int(round(cfg.r_max * abs(z - zc) / zc))


def plane_support(cfg: Config, z: int) -> int:
    """K(z), the odd side of plane z's non-zero support (centred in the K_max array)."""
    return min(cfg.nnum * (2 * support_radius(cfg, z) + 1), cfg.k_max)


def psf_factors(cfg: Config, dtype=np.float64):
    """1-D factors g[z][a][i] (rows) -- the PSF is h[z][a][b][i][j] = g[z][a][i] * g[z][b][j]."""
    N, K, nz = cfg.nnum, cfg.k_max, cfg.nz
    zc = (nz - 1) / 2.0
    c = (N - 1) / 2.0
    kc = (K - 1) // 2
    idx = np.arange(K, dtype=np.float64)
    g = np.zeros((nz, N, K), np.float64)
    for z in range(nz):
        sigma = cfg.sigma0 + cfg.slope * abs(z - zc)
        half = (plane_support(cfg, z) - 1) // 2
        inside = np.abs(idx - kc) <= half
        for a in range(N):
            centre = kc + cfg.shear * (z - zc) * (a - c) / N
            v = np.exp(-0.5 * ((idx - centre) / sigma) ** 2) * inside
            g[z, a] = v / v.sum()
    return g.astype(dtype)


def gen_psf(cfg: Config, dtype=np.float32):
    """h[z][a][b][i][j] (page order (z*N + a)*N + b), each kernel summing to 1 (reading C7)."""
    g = psf_factors(cfg, np.float64)
    N, K = cfg.nnum, cfg.k_max
    h = np.empty((cfg.nz, N, N, K, K), dtype)
    for z in range(cfg.nz):      # plane by plane keeps the fp64 temporary small (c4: 4.6 GB fp32 total)
        h[z] = (g[z][:, None, :, None] * g[z][None, :, None, :]).astype(dtype)
    return h


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def gen_beads(cfg: Config, seed: int, dtype=np.float64):
    """Hard-sphere beads: value `photons` inside, 0 outside, non-overlapping."""
    rng = _rng(seed)
    nz, H, W = cfg.nz, cfg.height, cfg.width
    vol = np.zeros((nz, H, W), np.float64)
    r = cfg.radius
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(H), np.arange(W), indexing="ij")
    centres = []
    tries = 0
    while len(centres) < cfg.n_objects and tries < 10000:
        tries += 1
        cz = rng.uniform(0, nz - 1)
        cy = rng.uniform(r, H - 1 - r)
        cx = rng.uniform(r, W - 1 - r)
        if all((cz - a) ** 2 + (cy - b) ** 2 + (cx - d) ** 2 > (2 * r + 1) ** 2 for a, b, d in centres):
            centres.append((cz, cy, cx))
    for cz, cy, cx in centres:
        vol[(zz - cz) ** 2 + (yy - cy) ** 2 + (xx - cx) ** 2 <= r * r] = cfg.photons
    vol += cfg.background * cfg.photons
    return vol.astype(dtype)


def gen_somata(cfg: Config, seed: int, dtype=np.float64, modulation=None):
    """Neuron-like sparse ellipsoids + uniform background.  `modulation` (optional,
    length n_objects) scales each soma's intensity (time-lapse frames)."""
    rng = _rng(seed)
    nz, H, W = cfg.nz, cfg.height, cfg.width
    vol = np.full((nz, H, W), cfg.background * cfg.photons, np.float64)
    n = cfg.n_objects
    cz = rng.uniform(0, nz - 1, n)
    cy = rng.uniform(8, H - 9, n)
    cx = rng.uniform(8, W - 9, n)
    rad = cfg.radius * rng.uniform(0.6, 1.4, n)
    inten = rng.uniform(0.3, 1.0, n) * cfg.photons
    if modulation is not None:
        inten = inten * np.asarray(modulation, dtype=np.float64)
    thick = 1.5
    for k in range(n):
        r = rad[k]
        z0, z1 = max(0, int(np.floor(cz[k] - thick))), min(nz - 1, int(np.ceil(cz[k] + thick)))
        y0, y1 = max(0, int(np.floor(cy[k] - r))), min(H - 1, int(np.ceil(cy[k] + r)))
        x0, x1 = max(0, int(np.floor(cx[k] - r))), min(W - 1, int(np.ceil(cx[k] + r)))
        zz, yy, xx = np.meshgrid(np.arange(z0, z1 + 1), np.arange(y0, y1 + 1), np.arange(x0, x1 + 1),
                                 indexing="ij")
        inside = ((zz - cz[k]) / thick) ** 2 + ((yy - cy[k]) / r) ** 2 + ((xx - cx[k]) / r) ** 2 <= 1.0
        sub = vol[z0:z1 + 1, y0:y1 + 1, x0:x1 + 1]
        sub[inside] = np.maximum(sub[inside], inten[k] + cfg.background * cfg.photons)
    return vol.astype(dtype)


def gen_volume(cfg: Config, seed: int, dtype=np.float64):
    if cfg.phantom == "beads":
        return gen_beads(cfg, seed, dtype)
    return gen_somata(cfg, seed, dtype)


def poisson(image, seed: int):
    """Pixel-wise Poisson sample with the image as mean; integer counts as float."""
    img = np.asarray(image, dtype=np.float64)
    if np.any(img < 0):
        raise ValueError("negative mean")
    return _rng(seed).poisson(img).astype(np.float64)


def lf_like(cfg: Config, seed: int, dtype=np.float64):
    """Model-free positive image with lenslet-periodic structure (no projector involved): smooth
    random blobs modulated by an N-periodic sub-aperture pattern, plus background, Poisson sampled.
    Used by full-size parity tests that must not take y from either projector."""
    rng = _rng(seed)
    H, W, N = cfg.height, cfg.width, cfg.nnum
    yy, xx = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    img = np.full((H, W), 5.0)
    for _ in range(24):
        cy, cx = rng.uniform(0, H), rng.uniform(0, W)
        s = rng.uniform(0.02, 0.08) * min(H, W)
        img += rng.uniform(20, 80) * np.exp(-0.5 * (((yy - cy) / s) ** 2 + ((xx - cx) / s) ** 2))
    a = (np.arange(H) % N - (N - 1) / 2.0) / max(N, 1)
    b = (np.arange(W) % N - (N - 1) / 2.0) / max(N, 1)
    lens = np.exp(-2.0 * (a[:, None] ** 2 + b[None, :] ** 2))
    return rng.poisson(img * lens).astype(dtype)

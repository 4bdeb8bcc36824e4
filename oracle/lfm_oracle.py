"""TEST INFRASTRUCTURE ONLY -- fp64 CPU oracle of the AutoDeconJ hot path (arXiv 2208.11422).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import this module.  It shares no code with the CUDA product path
(``paper_2208_11422_b200``); neither imports the other.

Citations: ``P:n`` = PAPER.md line n (the paper, arXiv 2208.11422), ``S:n`` = SPEC.md line n.
Readings of silent / garbled passages are numbered C1..C18 as in SURVEY.md §8(c) and DESIGN.md §3.

Contents, in the paper's order:
  * projections  -- direct fp64 spatial convolution in C (lfm_oracle.c): forward H,
                    backward H^T, normalizer H^T 1
  * RL iteration -- classical Richardson-Lucy update (§1 names RL; the update formula is not
                    printed -> reading C1): x <- x * H^T(y / (Hx+eps)) / max(H^T 1, eps)
  * metric       -- z max-projection, orthonormal DCT-II (Eqs. 1-4), Shannon entropy
                    (Eq. 5), cutoff region (Eqs. 6-11), DCT entropy (Eq. 12)
  * stop rule    -- "stop iteration when the DCT entropy value shows a decreasing trend",
                    best = argmax (Fig. 2d); reading C15.

Pins for every function live in tests/test_oracle_*.py (marked ``not gpu``).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblfm_oracle.so")
_SRC = os.path.join(_HERE, "lfm_oracle.c")

EPS = 1e-6   # reading C3: absolute guard 1e-6 in both oracle and GPU path


# ----------------------------------------------------------------------------------------------
# build / load the C half (building the checker is not using it)
# ----------------------------------------------------------------------------------------------
def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared",
                               "-std=c99", _SRC, "-o", _SO])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        i = ctypes.c_int
        lib.lfmo_forward.argtypes = [dp, dp, i, i, i, i, i, i, i, i, i, i, dp]
        lib.lfmo_backward.argtypes = [dp, dp, i, i, i, i, i, i, i, i, ctypes.c_long, ctypes.c_long, dp]
        lib.lfmo_forward_points.argtypes = [dp, dp, i, i, i, i, i, i, ip, ip, i, dp]
        lib.lfmo_backward_points.argtypes = [dp, dp, i, i, i, i, i, i, ip, ip, ip, i, dp]
        for f in (lib.lfmo_forward, lib.lfmo_backward, lib.lfmo_forward_points, lib.lfmo_backward_points):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _psf_dims(h):
    nz, n1, n2, kh, kw = h.shape
    if n1 != n2:
        raise ValueError("PSF must be [nz][N][N][kh][kw]")
    if kh % 2 == 0 or kw % 2 == 0:
        raise ValueError("kernel sizes must be odd (S:192)")
    return nz, n1, kh, kw


# ----------------------------------------------------------------------------------------------
# projections
# ----------------------------------------------------------------------------------------------
def forward_project(x, h, units=None, rows=None):
    """H x: y(s,t) = sum_z sum_{p,q} x(z,p,q) h[z][p%N][q%N](s-p+ch, t-q+cw), 'same' size,
    zero padding (reading C4/C5).  ``units`` = [u0,u1) restricts to units u=z*N*N+a*N+b;
    ``rows`` = [r0,r1) computes only those output rows (others 0)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    h = np.ascontiguousarray(h, dtype=np.float64)
    nz, N, kh, kw = _psf_dims(h)
    if x.ndim != 3 or x.shape[0] != nz:
        raise ValueError("x must be [nz][H][W] with nz matching the PSF")
    _, H, W = x.shape
    u0, u1 = (0, nz * N * N) if units is None else units
    r0, r1 = (0, H) if rows is None else rows
    y = np.zeros((H, W), np.float64)
    rc = _load().lfmo_forward(_dp(x), _dp(h), nz, N, kh, kw, H, W, u0, u1, r0, r1, _dp(y))
    if rc:
        raise ValueError(f"lfmo_forward rejected dims (rc={rc}): H,W must be divisible by N (S:188)")
    return y


def backward_project(r, h, units=None, planes=None):
    """H^T r: xhat(z,p,q) = sum_{s,t} r(s,t) h[z][p%N][q%N](s-p+ch, t-q+cw)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    h = np.ascontiguousarray(h, dtype=np.float64)
    nz, N, kh, kw = _psf_dims(h)
    H, W = r.shape
    u0, u1 = (0, nz * N * N) if units is None else units
    z0, z1 = (0, nz) if planes is None else planes
    xh = np.zeros((nz, H, W), np.float64)
    rc = _load().lfmo_backward(_dp(r), _dp(h), nz, N, kh, kw, H, W, u0, u1, z0 * H, z1 * H, _dp(xh))
    if rc:
        raise ValueError(f"lfmo_backward rejected dims (rc={rc})")
    return xh


def forward_points(x, h, s_idx, t_idx):
    """(H x)(s_k, t_k) for a list of pixels -- same sum as forward_project, one output at a time."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    h = np.ascontiguousarray(h, dtype=np.float64)
    nz, N, kh, kw = _psf_dims(h)
    _, H, W = x.shape
    s = np.ascontiguousarray(s_idx, dtype=np.int32)
    t = np.ascontiguousarray(t_idx, dtype=np.int32)
    out = np.zeros(len(s), np.float64)
    rc = _load().lfmo_forward_points(_dp(x), _dp(h), nz, N, kh, kw, H, W, _ip(s), _ip(t), len(s), _dp(out))
    if rc:
        raise ValueError(f"lfmo_forward_points rc={rc}")
    return out


def backward_points(r, h, z_idx, p_idx, q_idx):
    """(H^T r)(z_k, p_k, q_k) for a list of voxels."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    h = np.ascontiguousarray(h, dtype=np.float64)
    nz, N, kh, kw = _psf_dims(h)
    H, W = r.shape
    z = np.ascontiguousarray(z_idx, dtype=np.int32)
    p = np.ascontiguousarray(p_idx, dtype=np.int32)
    q = np.ascontiguousarray(q_idx, dtype=np.int32)
    out = np.zeros(len(z), np.float64)
    rc = _load().lfmo_backward_points(_dp(r), _dp(h), nz, N, kh, kw, H, W, _ip(z), _ip(p), _ip(q), len(z), _dp(out))
    if rc:
        raise ValueError(f"lfmo_backward_points rc={rc}")
    return out


def backward_project_ht(r, ht):
    """MATLAB-lineage backward with a supplied transposed PSF (reading C6):
    xhat(z,p,q) = sum_{s,t} r(s,t) Ht[z][p%N][q%N](p-s+ch, q-t+cw).  Since Ht(p-s+c) = rot180(Ht)(s-p+c), this is
    the adjoint formula of S:208 evaluated with the kernel bank rot180(Ht)."""
    return backward_project(r, np.ascontiguousarray(np.asarray(ht, dtype=np.float64)[:, :, :, ::-1, ::-1]))


def compute_normalizer(h, H, W, units=None):
    """H^T 1: backward projection of the all-ones image; the RL denominator."""
    return backward_project(np.ones((H, W)), h, units=units)


# ----------------------------------------------------------------------------------------------
# RL iteration (§1; update form = reading C1)
# ----------------------------------------------------------------------------------------------
def initial_volume(y, h, nz, H, W):
    """Reading C2: uniform x0 = c0 with c0 = sum(y) / sum(H 1_vol), i.e. the forward
    projection of x0 has the same total as y."""
    total_h1 = forward_project(np.ones((nz, H, W)), h).sum()
    if total_h1 <= 0:
        raise ValueError("PSF projects nothing")
    return np.full((nz, H, W), y.sum() / total_h1)


def ratio_image(y, yhat, eps=EPS):
    """r = y / (yhat + eps) (reading C3 for eps).  yhat = H x is a sum of non-negative products
    here, so it is >= 0 exactly; the GPU's clamp against FFT round-off (reading C19) has no counterpart."""
    return y / (yhat + eps)


def rl_step(x, y, h, norm, eps=EPS):
    """x_{k+1} = x_k * H^T(y / (H x_k + eps)) / max(H^T 1, eps)   (reading C1/C3).
    Returns (x_{k+1}, H x_k)."""
    yhat = forward_project(x, h)
    bp = backward_project(ratio_image(y, yhat, eps), h)
    return x * bp / np.maximum(norm, eps), yhat


def isra_step(x, y, h, hty, eps=EPS):
    """MATLAB-lineage ISRA form x * H^T y / H^T H x (reading C1).  Not on the default path."""
    yhat = forward_project(x, h)
    return x * hty / np.maximum(backward_project(yhat, h), eps), yhat


def poisson_loglik(y, yhat):
    """sum[y log(Hx) - Hx]: the EM objective RL never decreases."""
    m = y > 0
    return float(np.sum(y[m] * np.log(yhat[m])) - np.sum(yhat))


# ----------------------------------------------------------------------------------------------
# metric (§2.2)
# ----------------------------------------------------------------------------------------------
def max_project_z(vol):
    """"We only take the maximum projection along the z-axis for each iterative result"."""
    return np.max(vol, axis=0)


def dct_basis(Z, count=None):
    """C[u][x] = c(u,Z) cos((2x+1) pi u / 2Z), c = 1/sqrt(Z) for u=0 else sqrt(2/Z)  (Eqs. 2-4).
    Rows u < count (default all Z)."""
    count = Z if count is None else count
    u = np.arange(count, dtype=np.float64)[:, None]
    xx = np.arange(Z, dtype=np.float64)[None, :]
    c = np.where(u == 0, 1.0 / math.sqrt(Z), math.sqrt(2.0 / Z))
    return c * np.cos((2.0 * xx + 1.0) * math.pi * u / (2.0 * Z))


def dct2(f, rows=None, cols=None):
    """F_c(u,v) = sum_{x,y} f(x,y) C_u(x,M) C_v(y,N)  (Eq. 1), orthonormal DCT-II.
    f is [M][N] = [height][width]; u indexes the height axis, v the width axis (reading C8).
    ``rows``/``cols`` return only the top-left rows x cols corner (same definition, truncated)."""
    f = np.asarray(f, dtype=np.float64)
    M, N = f.shape
    return dct_basis(M, rows) @ f @ dct_basis(N, cols).T


def idct2(F):
    """Inverse of the orthonormal dct2 (test plumbing)."""
    M, N = F.shape
    return dct_basis(M).T @ F @ dct_basis(N)


def shannon_entropy(p):
    """F_entropy = -sum p_i log2 p_i  (Eq. 5), with 0 log 0 = 0."""
    p = np.asarray(p, dtype=np.float64)
    if np.any(p < 0):
        raise ValueError("probabilities must be >= 0")
    nz = p[p > 0]
    return -math.fsum((nz * np.log2(nz)).tolist())


def sample_pitch(mla_pitch_um, magnification, nnum):
    """P_u = d_ML / (Q * Nnum)  (Eq. 7)."""
    return mla_pitch_um / (magnification * nnum)


def resolution_limit(wavelength_um, na, nnum):
    """d_psf = 1.22 lambda Nnum / NA  (Eq. 11)."""
    return 1.22 * wavelength_um * nnum / na


@dataclass
class Optics:
    wavelength_um: float
    na: float
    mla_pitch_um: float
    magnification: float
    nnum: int

    def validate(self):
        if min(self.wavelength_um, self.na, self.mla_pitch_um, self.magnification) <= 0:
            raise ValueError("optics fields must be > 0 (S:25)")
        if self.nnum < 1 or self.nnum % 2 == 0:
            raise ValueError("nnum must be odd (S:26)")
        if self.na > 1.6:
            raise ValueError("na <= 1.6 (S:27)")


@dataclass
class CutoffRegion:
    x_s: int
    y_s: int
    g_s: float
    members: list = field(default_factory=list)     # (u, v): u row (height) index, v column index
    p_x: float = 0.0
    p_y: float = 0.0


def cutoff_region(optics: Optics, height, width, shape="triangle"):
    """Eqs. (6)-(11).  X_S = P_u*N/d_psf (Eq. 9), Y_S = P_u*M/d_psf (Eq. 10), rounded up
    and clamped to [1, dim] (reading C10).  Triangle T = {(u,v): u*X_S + v*Y_S < X_S*Y_S} with u the
    height index (< Y_S) and v the width index (< X_S) (reading C11; G_S = X_S*Y_S/2, Eq. 6); the
    'rectangle' variant follows Eq. 12's literal bounds u < X_S, v < Y_S mapped to the same axes.
    P (Eq. 8) is reported per axis only (reading C9)."""
    optics.validate()
    if height < 2 or width < 2:
        raise ValueError("image must be at least 2x2 (S:60)")
    pu = sample_pitch(optics.mla_pitch_um, optics.magnification, optics.nnum)
    dpsf = resolution_limit(optics.wavelength_um, optics.na, optics.nnum)
    x_s = int(min(max(math.ceil(pu * width / dpsf), 1), width))
    y_s = int(min(max(math.ceil(pu * height / dpsf), 1), height))
    if shape == "triangle":
        mem = [(u, v) for u in range(y_s) for v in range(x_s) if u * x_s + v * y_s < x_s * y_s]
    elif shape == "rectangle":
        mem = [(u, v) for u in range(y_s) for v in range(x_s)]
    else:
        raise ValueError("shape must be triangle or rectangle")
    return CutoffRegion(x_s, y_s, x_s * y_s / 2.0, mem, dpsf / pu * width, dpsf / pu * height)


def dct_entropy(img, region: CutoffRegion):
    """DCT entropy, Eq. (12): (2/(X_S*Y_S)) * sum_{(u,v) in T} -w log2 w,
    w = |F_c(u,v)| / L2(F_c) with the L2 norm over the FULL coefficient matrix (reading C13),
    prefactor 2/S^2 read as 1/G_S = 2/(X_S*Y_S) (reading C12); 0 log 0 = 0; all-zero image -> 0."""
    F = dct2(img)
    L = math.sqrt(math.fsum((F.ravel() ** 2).tolist()))
    if L == 0.0:
        return 0.0
    terms = []
    for (u, v) in region.members:
        w = abs(F[u, v]) / L
        if w > 0.0:
            terms.append(-w * math.log2(w))
    return 2.0 / (region.x_s * region.y_s) * math.fsum(terms)


def evaluate_iteration(vol, region):
    """E_k = dct_entropy(max_project_z(x_k))  (P:63 + Eq. 12)."""
    return dct_entropy(max_project_z(vol), region)


# ----------------------------------------------------------------------------------------------
# stop rule (reading C15) and the deconvolution loop
# ----------------------------------------------------------------------------------------------
@dataclass
class Policy:
    mode: str = "auto"        # "auto" | "fixed"
    n_iters: int = 10         # fixed mode
    max_iters: int = 50       # Fig. 2d sweeps 1..50
    min_iters: int = 2
    patience: int = 1
    eps: float = EPS

    def validate(self):
        if self.mode not in ("auto", "fixed"):
            raise ValueError("mode")
        if self.min_iters < 1 or self.min_iters > self.max_iters or self.patience < 1:
            raise ValueError("invalid policy (S:254)")
        if self.mode == "fixed" and self.n_iters < 1:
            raise ValueError("n_iters >= 1")


class StopRule:
    """After each E_k (k >= 1): best = argmax E (ties -> smallest k); in auto mode stop at the first
    k >= min_iters after `patience` consecutive strict decreases ("stop iteration when the DCT
    entropy value shows a decreasing trend"), else at max_iters; fixed mode runs n_iters."""

    def __init__(self, policy: Policy):
        policy.validate()
        self.p = policy
        self.series = []
        self.best_iter = 0
        self.best = -math.inf
        self.decreases = 0

    def update(self, e):
        """Record E_k; returns (improved, stop)."""
        k = len(self.series) + 1
        if self.series and e < self.series[-1]:
            self.decreases += 1
        else:
            self.decreases = 0
        self.series.append(e)
        improved = e > self.best
        if improved:
            self.best, self.best_iter = e, k
        if self.p.mode == "fixed":
            stop = k >= self.p.n_iters
        else:
            stop = (k >= self.p.min_iters and self.decreases >= self.p.patience) or k >= self.p.max_iters
        return improved, stop


@dataclass
class DeconvResult:
    volume: np.ndarray
    best_iter: int
    stop_iter: int
    series: list
    iterates: list = field(default_factory=list)


def deconvolve(y, h, optics: Optics, policy: Policy, x0=None, region_shape="triangle",
               keep_iterates=False, update="rl"):
    """RL loop with the DCT-entropy stop rule.  Rejects all-zero y.
    update="isra": the MATLAB-lineage form x * H^T y / H^T H x starting from x0 = H^T y (reading C1)."""
    y = np.asarray(y, dtype=np.float64)
    if np.any(y < 0):
        raise ValueError("negative measurement")
    if not np.any(y > 0):
        raise ValueError("all-zero measurement (S:288)")
    nz, N, kh, kw = _psf_dims(np.asarray(h))
    H, W = y.shape
    region = cutoff_region(optics, H, W, region_shape)
    if update == "isra":
        hty = backward_project(y, h)
        x = hty.copy() if x0 is None else np.array(x0, dtype=np.float64)
    else:
        norm = compute_normalizer(h, H, W)
        x = initial_volume(y, h, nz, H, W) if x0 is None else np.array(x0, dtype=np.float64)
    rule = StopRule(policy)
    best = x.copy()
    iterates = []
    while True:
        if update == "isra":
            x, _ = isra_step(x, y, h, hty, policy.eps)
        else:
            x, _ = rl_step(x, y, h, norm, policy.eps)
        if keep_iterates:
            iterates.append(x.copy())
        improved, stop = rule.update(evaluate_iteration(x, region))
        if improved:
            best = x.copy()
        if stop:
            break
    return DeconvResult(best, rule.best_iter, len(rule.series), list(rule.series), iterates)

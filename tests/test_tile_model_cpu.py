"""CPU check of the overlap-save index algebra of the tiled frequency path, independent of the CUDA
code: a numpy model with the same window origins (forward tile*T - dmax, adjoint tile*T + dmin), the same valid output
offsets and the same wrapped coarse-kernel placement reproduces the oracle's forward and backward projections to
rounding.  It pins the geometry the kernels implement (tap range from the kernel size, L = T + dmax - dmin); the GPU
parity of the kernels themselves is tests/test_gpu_tiles.py."""
import math

import numpy as np
import pytest

from oracle import lfm_oracle as O


def tap_range(N, k):
    c = (k - 1) // 2
    return math.ceil((-(N - 1) - c) / N), math.floor((k - 1 + (N - 1) - c) / N)


def model(h, x, r, N, L):
    nz, _, _, kh, kw = h.shape
    H, W = x.shape[1:]
    nh, nw = H // N, W // N
    ch, cw = (kh - 1) // 2, (kw - 1) // 2
    (d1a, d1b), (d2a, d2b) = tap_range(N, kh), tap_range(N, kw)
    T1, T2 = L - (d1b - d1a), L - (d2b - d2a)
    nty, ntx = -(-nh // T1), -(-nw // T2)
    units = [(z, a1, a2) for z in range(nz) for a1 in range(N) for a2 in range(N)]
    bps = [(b1, b2) for b1 in range(N) for b2 in range(N)]
    M = np.zeros((L, L, len(bps), len(units)), complex)
    for ui, (z, a1, a2) in enumerate(units):
        for bi, (b1, b2) in enumerate(bps):
            k = np.zeros((L, L))
            for d1 in range(d1a, d1b + 1):
                k1 = b1 - a1 + ch + N * d1
                for d2 in range(d2a, d2b + 1):
                    k2 = b2 - a2 + cw + N * d2
                    if 0 <= k1 < kh and 0 <= k2 < kw:
                        k[d1 % L, d2 % L] += h[z, a1, a2, k1, k2]
            M[:, :, bi, ui] = np.fft.fft2(k)

    def win(img, s1, s2):
        w = np.zeros((L, L))
        i0, j0 = max(0, -s1), max(0, -s2)
        i1, j1 = min(L, img.shape[0] - s1), min(L, img.shape[1] - s2)
        if i1 > i0 and j1 > j0:
            w[i0:i1, j0:j1] = img[s1 + i0:s1 + i1, s2 + j0:s2 + j1]
        return w

    y = np.zeros((H, W))
    xb = np.zeros((nz, H, W))
    for ty in range(nty):
        for tx in range(ntx):
            G = np.stack([np.fft.fft2(win(x[z, a1::N, a2::N], ty * T1 - d1b, tx * T2 - d2b)) for (z, a1, a2) in units], -1)
            Y = np.einsum("ijbu,iju->ijb", M, G)
            R = np.stack([np.fft.fft2(win(r[b1::N, b2::N], ty * T1 + d1a, tx * T2 + d2a)) for (b1, b2) in bps], -1)
            X = np.einsum("ijbu,ijb->iju", M.conj(), R)
            m1 = np.arange(ty * T1, min(nh, (ty + 1) * T1))
            m2 = np.arange(tx * T2, min(nw, (tx + 1) * T2))
            for bi, (b1, b2) in enumerate(bps):
                zt = np.fft.ifft2(Y[:, :, bi]).real
                y[np.ix_(b1 + N * m1, b2 + N * m2)] = zt[np.ix_(d1b + m1 - ty * T1, d2b + m2 - tx * T2)]
            for ui, (z, a1, a2) in enumerate(units):
                zt = np.fft.ifft2(X[:, :, ui]).real
                xb[z][np.ix_(a1 + N * m1, a2 + N * m2)] = zt[np.ix_(-d1a + m1 - ty * T1, -d2a + m2 - tx * T2)]
    return y, xb, nty * ntx


@pytest.mark.parametrize("case", [(2, 3, 27, 33, 9, 9, 8), (2, 3, 30, 24, 9, 15, 12), (1, 5, 45, 40, 15, 25, 9)],
                         ids=["3x3-tiles", "unequal-spans", "N5"])
def test_overlap_save_model_matches_oracle(case):
    nz, N, H, W, kh, kw, L = case
    rng = np.random.default_rng(sum(case))
    h = rng.uniform(0, 1, (nz, N, N, kh, kw))
    x = rng.uniform(0, 1, (nz, H, W))
    r = rng.uniform(0.5, 1.5, (H, W))
    y, xb, ntiles = model(h, x, r, N, L)
    assert ntiles >= 2
    yo, xo = O.forward_project(x, h), O.backward_project(r, h)
    assert np.linalg.norm(y - yo) <= 1e-12 * np.linalg.norm(yo)
    assert np.linalg.norm(xb - xo) <= 1e-12 * np.linalg.norm(xo)


def test_c3_tap_range_and_window():
    """c3 (N = 15, K_max = 165): coarse taps in [-6, 6]; L = 27 gives T = 15 and 5 x 5 tiles over 67 coarse pixels."""
    assert tap_range(15, 165) == (-6, 6)
    T = 27 - 12
    assert T == 15 and -(-67 // T) == 5


def _lib():
    from paper_2208_11422_b200 import lfm
    return lfm


@pytest.mark.parametrize("args,expect", [
    ((15, 1005, 1005, -6, 6, -6, 6), (27, 15, 15, 25)),     # c3, r = 5 planes (taps +-6)
    ((15, 1005, 1005, -3, 3, -3, 3), (20, 14, 14, 25)),     # c3, r = 2 planes
    ((15, 2025, 2025, -8, 8, -8, 8), (45, 29, 29, 25)),     # c4, the widest planes
    ((11, 319, 319, -5, 5, -5, 5), (20, 10, 10, 9)),        # c2
    ((3, 33, 33, -2, 2, -2, 2), (0, 0, 0, 0)),              # tiny: a single window would cover the image
])
def test_tile_model_choices(args, expect):
    """lfm_tile_model is the planner's own choice (host-only, no GPU): window size, valid outputs and tile count at
    the BASELINE geometries; the window spans the taps (L = T + d1b - d1a) and 2-32 tiles cover the coarse image."""
    m = _lib().lfm_tile_model(*args)
    assert (m["L"], m["T1"], m["T2"], m["ntile"]) == expect
    if m["L"]:
        nnum, h, w, d1a, d1b, d2a, d2b = args
        assert m["L"] == m["T1"] + d1b - d1a == m["T2"] + d2b - d2a
        assert 2 <= m["ntile"] == -(-(h // nnum) // m["T1"]) * -(-(w // nnum) // m["T2"]) <= 32
        assert 0 < m["cost_unit"] < m["cost_whole"]


def test_tile_model_flags_and_errors():
    L = _lib()
    assert L.lfm_tile_model(15, 1005, 1005, -6, 6, -6, 6, flags=L.LFM_PLAN_NO_TILES)["L"] == 0
    assert L.lfm_tile_model(15, 1005, 1005, -6, 6, -6, 6, flags=L.LFM_PLAN_FRAMES)["L"] == 0
    with pytest.raises(L.LfmError) as e:
        L.lfm_tile_model(15, 1005, 1005, 6, -6, -6, 6)
    assert e.value.status == L.LFM_EINVAL
    with pytest.raises(L.LfmError) as e:
        L.lfm_tile_model(15, 1000, 1005, -6, 6, -6, 6)   # 1000 is not a multiple of N = 15
    assert e.value.status == L.LFM_EDIM

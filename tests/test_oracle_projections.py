"""Pins of the oracle's projections (not gpu).  Each test states what fixes the expected value
independently of the oracle: a dense operator built entry by entry, a library routine, a closed form,
or an invariant of the mathematics (SURVEY §8(c) pin table)."""
import numpy as np
import pytest
import scipy.signal

from lfm_inputs import CONFIGS, gen_psf
from oracle import lfm_oracle as O


def rand_psf(rng, nz, N, kh, kw, normalise=False):
    h = rng.uniform(0.0, 1.0, (nz, N, N, kh, kw))
    if normalise:
        h /= h.sum(axis=(3, 4), keepdims=True)
    return h


def dense_operator(h, H, W):
    """Materialise H entry by entry from the element definition:
    A[(s,t), (z,p,q)] = h[z][p%N][q%N][s-p+ch][t-q+cw] when inside the kernel, else 0.
    Pure-python loops, independent of the C oracle's loop structure."""
    nz, N, _, kh, kw = h.shape
    ch, cw = (kh - 1) // 2, (kw - 1) // 2
    A = np.zeros((H * W, nz * H * W))
    for z in range(nz):
        for p in range(H):
            for q in range(W):
                col = (z * H + p) * W + q
                for s in range(H):
                    i = s - p + ch
                    if not 0 <= i < kh:
                        continue
                    for t in range(W):
                        j = t - q + cw
                        if 0 <= j < kw:
                            A[s * W + t, col] = h[z, p % N, q % N, i, j]
    return A


@pytest.mark.parametrize("nz,N,H,W,kh,kw", [(2, 3, 9, 9, 3, 3), (3, 3, 9, 12, 5, 7), (2, 1, 6, 5, 3, 5)])
def test_dense_operator_bruteforce(nz, N, H, W, kh, kw):
    """S:204 / S:593: forward equals the materialised operator (1e-12); backward equals its transpose;
    normalizer equals its column sums."""
    rng = np.random.default_rng(1)
    h = rand_psf(rng, nz, N, kh, kw)
    A = dense_operator(h, H, W)
    x = rng.uniform(0, 1, (nz, H, W))
    r = rng.uniform(0, 1, (H, W))
    y = O.forward_project(x, h)
    np.testing.assert_allclose(y.ravel(), A @ x.ravel(), rtol=1e-12, atol=1e-13)
    xb = O.backward_project(r, h)
    np.testing.assert_allclose(xb.ravel(), A.T @ r.ravel(), rtol=1e-12, atol=1e-13)
    nrm = O.compute_normalizer(h, H, W)
    np.testing.assert_allclose(nrm.ravel(), A.sum(axis=0), rtol=1e-12, atol=1e-13)
    # point evaluators are the same sums one output at a time
    s, t = np.nonzero(np.ones((H, W)))
    np.testing.assert_allclose(O.forward_points(x, h, s, t), y.ravel(), rtol=1e-12, atol=1e-13)
    zz, pp, qq = np.nonzero(np.ones((nz, H, W)))
    np.testing.assert_allclose(O.backward_points(r, h, zz, pp, qq), xb.ravel(), rtol=1e-12, atol=1e-13)


def test_adjoint_dot_test():
    """<Hx, y> = <x, H^T y> on 100 random instances at nz=3, N=3, 9x9, 3x3 kernels,
    plus larger shapes; tolerance 1e-12 * |Hx| |y|."""
    rng = np.random.default_rng(2)
    for k in range(100):
        h = rand_psf(rng, 3, 3, 3, 3)
        x = rng.normal(size=(3, 9, 9))
        y = rng.normal(size=(9, 9))
        hx = O.forward_project(x, h)
        lhs = np.vdot(hx, y)
        rhs = np.vdot(x, O.backward_project(y, h))
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(hx) * np.linalg.norm(y)
    for (nz, N, H, kh) in [(2, 5, 30, 11), (3, 3, 33, 9)]:
        h = rand_psf(rng, nz, N, kh, kh)
        x = rng.normal(size=(nz, H, H))
        y = rng.normal(size=(H, H))
        hx = O.forward_project(x, h)
        assert abs(np.vdot(hx, y) - np.vdot(x, O.backward_project(y, h))) <= 1e-12 * np.linalg.norm(hx) * np.linalg.norm(y)


def test_delta_psf_identity():
    """Closed form: h = delta at the kernel centre for every (z,a,b) => H x = sum_z x_z exactly, and
    H^T r = r on every plane (SURVEY §8(c) pin 'delta PSF')."""
    rng = np.random.default_rng(3)
    nz, N, K, H = 4, 3, 5, 12
    h = np.zeros((nz, N, N, K, K))
    h[:, :, :, K // 2, K // 2] = 1.0
    x = rng.uniform(0, 5, (nz, H, H))
    assert np.array_equal(O.forward_project(x, h), x.sum(axis=0))
    r = rng.uniform(0, 5, (H, H))
    assert np.array_equal(O.backward_project(r, h), np.broadcast_to(r, (nz, H, H)))


def test_shifted_delta_permutation():
    """Closed form: h[z][a][b] = delta at (ch + di(z,a), cw + dj(z,b)) moves voxel (z,p,q) to pixel
    (p + di, q + dj) (when inside).  Pins the kernel centre, convolution orientation and that the
    kernel is chosen by the INPUT voxel's phase (p mod N, q mod N) -- readings C5/C6."""
    rng = np.random.default_rng(4)
    nz, N, K, H, W = 2, 3, 7, 12, 15
    c = K // 2
    di = rng.integers(-c, c + 1, (nz, N))
    dj = rng.integers(-c, c + 1, (nz, N))
    h = np.zeros((nz, N, N, K, K))
    for z in range(nz):
        for a in range(N):
            for b in range(N):
                h[z, a, b, c + di[z, a], c + dj[z, b]] = 1.0
    x = rng.uniform(0, 1, (nz, H, W))
    expect = np.zeros((H, W))
    for z in range(nz):
        for p in range(H):
            for q in range(W):
                s, t = p + di[z, p % N], q + dj[z, q % N]
                if 0 <= s < H and 0 <= t < W:
                    expect[s, t] += x[z, p, q]
    np.testing.assert_allclose(O.forward_project(x, h), expect, rtol=0, atol=1e-14)


def test_single_phase_is_scipy_convolution():
    """Library routine: N = 1, nz = 1 => forward is scipy.signal.convolve2d(mode='same') and backward is
    scipy.signal.correlate2d(mode='same')."""
    rng = np.random.default_rng(5)
    for (H, W, kh, kw) in [(17, 23, 5, 7), (9, 9, 9, 3), (30, 20, 11, 11)]:
        ker = rng.uniform(0, 1, (kh, kw))
        h = ker[None, None, None]
        x = rng.uniform(0, 1, (1, H, W))
        np.testing.assert_allclose(O.forward_project(x, h), scipy.signal.convolve2d(x[0], ker, mode="same"),
                                   rtol=1e-12, atol=1e-13)
        r = rng.uniform(0, 1, (H, W))
        np.testing.assert_allclose(O.backward_project(r, h)[0], scipy.signal.correlate2d(r, ker, mode="same"),
                                   rtol=1e-12, atol=1e-13)


def test_impulse_response_linearity_nonnegativity():
    """S:203 impulse stamps h[z0][p%N][q%N] centred at (p,q); S:225 linearity; S:227 non-negativity."""
    rng = np.random.default_rng(6)
    nz, N, K, H = 2, 3, 5, 15
    h = rand_psf(rng, nz, N, K, K)
    x = np.zeros((nz, H, H))
    z0, p, q = 1, 7, 4
    x[z0, p, q] = 1.0
    y = O.forward_project(x, h)
    expect = np.zeros((H, H))
    c = K // 2
    expect[p - c:p + c + 1, q - c:q + c + 1] = h[z0, p % N, q % N]
    assert np.array_equal(y, expect)
    x1, x2 = rng.uniform(0, 1, (2, nz, H, H))
    np.testing.assert_allclose(O.forward_project(2.5 * x1 - 0.5 * x2, h),
                               2.5 * O.forward_project(x1, h) - 0.5 * O.forward_project(x2, h), rtol=1e-10, atol=1e-12)
    assert O.forward_project(x1, h).min() >= 0 and O.backward_project(x1[0], h).min() >= 0


def test_lattice_shift_equivariance():
    """translating x by (N, N) translates y by (N, N) in the interior."""
    rng = np.random.default_rng(7)
    nz, N, K, H = 2, 3, 5, 27
    h = rand_psf(rng, nz, N, K, K)
    x = np.zeros((nz, H, H))
    x[:, 6:15, 6:15] = rng.uniform(0, 1, (nz, 9, 9))
    xs = np.roll(x, (N, N), axis=(1, 2))
    y, ys = O.forward_project(x, h), O.forward_project(xs, h)
    np.testing.assert_allclose(ys[N:, N:], y[:-N, :-N], rtol=1e-13, atol=1e-14)


def test_flux_conservation_and_normalizer_interior():
    """Per-kernel-normalised PSF (reading C7): sum(Hx) = sum(x) when x is zero within c of the border,
    and the normalizer H^T 1 is exactly 1 in the interior."""
    cfg = CONFIGS["tiny"]
    h = gen_psf(cfg, np.float64)
    rng = np.random.default_rng(8)
    c = cfg.k_max // 2
    x = np.zeros((cfg.nz, cfg.height, cfg.width))
    x[:, c:-c, c:-c] = rng.uniform(0, 1, (cfg.nz, cfg.height - 2 * c, cfg.width - 2 * c))
    assert abs(O.forward_project(x, h).sum() - x.sum()) <= 1e-12 * x.sum()
    nrm = O.compute_normalizer(h, cfg.height, cfg.width)
    np.testing.assert_allclose(nrm[:, c:-c, c:-c], 1.0, rtol=0, atol=1e-12)
    assert nrm.max() <= 1.0 + 1e-12 and nrm.min() > 0


def test_unit_partition_sums_to_full():
    """S:235 / S:352: forward over a partition of units sums to the full forward; backward restricted to
    a unit range equals the full backward on those units and zero elsewhere."""
    rng = np.random.default_rng(9)
    nz, N, K, H = 3, 3, 5, 12
    h = rand_psf(rng, nz, N, K, K)
    x = rng.uniform(0, 1, (nz, H, H))
    nu = nz * N * N
    cuts = [0, 5, 13, 20, nu]
    parts = sum(O.forward_project(x, h, units=(cuts[i], cuts[i + 1])) for i in range(len(cuts) - 1))
    np.testing.assert_allclose(parts, O.forward_project(x, h), rtol=1e-13, atol=1e-14)
    r = rng.uniform(0, 1, (H, H))
    full = O.backward_project(r, h)
    part = O.backward_project(r, h, units=(5, 13))
    z, p, q = np.meshgrid(np.arange(nz), np.arange(H), np.arange(H), indexing="ij")
    u = (z * N + p % N) * N + q % N
    own = (u >= 5) & (u < 13)
    assert np.array_equal(part[own], full[own]) and not part[~own].any()


def test_rejects_bad_dims():
    h = np.ones((1, 3, 3, 3, 3))
    with pytest.raises(ValueError):
        O.forward_project(np.ones((1, 10, 9)), h)       # H not divisible by N
    with pytest.raises(ValueError):
        O.forward_project(np.ones((1, 9, 9)), np.ones((1, 3, 3, 4, 3)))   # even kernel


def test_ht_backward_bruteforce():
    """f3: the Ht backward equals the operator built entry by entry from its definition
    xhat(z,p,q) = sum_{s,t} r(s,t) Ht[z][p%N][q%N](p-s+ch, q-t+cw); with Ht = rot180(h) it is the exact adjoint."""
    rng = np.random.default_rng(12)
    nz, N, H, W, kh, kw = 2, 3, 9, 12, 5, 3
    ht = rng.uniform(0, 1, (nz, N, N, kh, kw))
    ch, cw = kh // 2, kw // 2
    B = np.zeros((nz * H * W, H * W))
    for z in range(nz):
        for p in range(H):
            for q in range(W):
                for s in range(H):
                    i = p - s + ch
                    if not 0 <= i < kh:
                        continue
                    for t in range(W):
                        j = q - t + cw
                        if 0 <= j < kw:
                            B[(z * H + p) * W + q, s * W + t] = ht[z, p % N, q % N, i, j]
    r = rng.uniform(0, 1, (H, W))
    np.testing.assert_allclose(O.backward_project_ht(r, ht).ravel(), B @ r.ravel(), rtol=1e-12, atol=1e-13)
    h = rng.uniform(0, 1, (nz, N, N, kh, kw))
    np.testing.assert_allclose(O.backward_project_ht(r, h[:, :, :, ::-1, ::-1]), O.backward_project(r, h), rtol=1e-13)

"""Pins of the oracle's RL iteration (not gpu): closed forms and invariants of Richardson-Lucy
(P:29 names RL, reading C1 fixes the classical update)."""
import numpy as np
import pytest

from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson
from oracle import lfm_oracle as O


def small_problem(seed=0, nz=3, N=3, H=15, K=5):
    rng = np.random.default_rng(seed)
    h = rng.uniform(0, 1, (nz, N, N, K, K))
    h /= h.sum(axis=(3, 4), keepdims=True)
    xt = rng.uniform(0, 10, (nz, H, H))
    y = rng.poisson(O.forward_project(xt, h)).astype(float)
    return h, y


def test_flux_identity():
    """Exact identity of the update: sum_v x1(v) max(norm(v),eps) = <H x0, r> = sum_s y yhat/(yhat+eps),
    for any PSF (holds to 12 digits)."""
    for seed in range(5):
        h, y = small_problem(seed)
        nz, _, _, _, _ = h.shape
        H, W = y.shape
        norm = O.compute_normalizer(h, H, W)
        x0 = O.initial_volume(y, h, nz, H, W)
        x1, yhat = O.rl_step(x0, y, h, norm)
        lhs = np.sum(x1 * np.maximum(norm, O.EPS))
        rhs = np.sum(y * yhat / (yhat + O.EPS))
        assert abs(lhs - rhs) <= 1e-12 * rhs


def test_initial_volume_matches_flux():
    """Reading C2: the forward projection of x0 has the same total as y."""
    h, y = small_problem(1)
    x0 = O.initial_volume(y, h, h.shape[0], *y.shape)
    assert abs(O.forward_project(x0, h).sum() - y.sum()) <= 1e-12 * y.sum()
    assert np.ptp(x0) == 0


def test_delta_psf_closed_form():
    """Closed form: delta PSF, nz planes, uniform init c0 = sum(y)/(nz H W) (since sum H1 = nz H W)
    => x1 = c0 * y / (nz c0 + eps) on every plane."""
    rng = np.random.default_rng(2)
    nz, N, K, H = 3, 3, 3, 9
    h = np.zeros((nz, N, N, K, K))
    h[:, :, :, 1, 1] = 1.0
    y = rng.poisson(20, (H, H)).astype(float)
    norm = O.compute_normalizer(h, H, H)
    x0 = O.initial_volume(y, h, nz, H, H)
    c0 = y.sum() / (nz * H * H)
    assert np.allclose(x0, c0, rtol=1e-15)
    x1, _ = O.rl_step(x0, y, h, norm)
    np.testing.assert_allclose(x1, np.broadcast_to(c0 * y / (nz * c0 + O.EPS), x1.shape), rtol=1e-14)


def test_exact_data_fixed_point_and_zeros():
    """y = H x*, x_k = x* => x_{k+1} = x* (up to the eps guard); S:273 zeros stay zero; iterates >= 0."""
    rng = np.random.default_rng(3)
    nz, N, K, H = 2, 3, 5, 12
    h = rng.uniform(0, 1, (nz, N, N, K, K))
    xs = rng.uniform(1, 2, (nz, H, H))
    xs[0, 3, 4] = 0.0
    y = O.forward_project(xs, h)
    norm = O.compute_normalizer(h, H, H)
    x1, _ = O.rl_step(xs, y, h, norm)
    np.testing.assert_allclose(x1, xs, rtol=1e-6)
    assert x1[0, 3, 4] == 0.0 and x1.min() >= 0
    z, _ = O.rl_step(np.zeros_like(xs), y, h, norm)
    assert not z.any()


def test_poisson_loglik_nondecreasing():
    """EM property of RL: sum[y log Hx - Hx] never decreases over 20 iterations on random
    nz=3, N=3, 15x15 instances (round-off tolerance 1e-10 relative)."""
    for seed in range(20):
        h, y = small_problem(seed)
        nz = h.shape[0]
        H, W = y.shape
        norm = O.compute_normalizer(h, H, W)
        x = O.initial_volume(y, h, nz, H, W)
        prev = -np.inf
        for k in range(20):
            xn, yhat = O.rl_step(x, y, h, norm)
            ll = O.poisson_loglik(y, yhat)
            assert ll >= prev - 1e-10 * abs(ll)
            prev = ll
            x = xn
            assert x.min() >= 0


def test_isra_residual_nonincreasing():
    """f3 variant: ISRA x * H^T y / H^T H x never increases ||y - Hx||^2 (Daube-Witherspoon & Muehllehner)."""
    h, y = small_problem(4)
    nz = h.shape[0]
    H, W = y.shape
    hty = O.backward_project(y, h)
    x = O.initial_volume(y, h, nz, H, W)
    prev = np.inf
    for k in range(15):
        xn, yhat = O.isra_step(x, y, h, hty)
        res = float(np.sum((y - yhat) ** 2))
        assert res <= prev * (1 + 1e-12)
        prev, x = res, xn


def test_deconvolve_tiny_runs_and_stops():
    """End-to-end oracle loop on the tiny BASELINE config: fixed 10 iterations (BASELINE configs[0]);
    best = argmax of the series; volume non-negative; the auto loop obeys the stop rule."""
    cfg = CONFIGS["tiny"]
    h = gen_psf(cfg, np.float64)
    xt = gen_volume(cfg, 1)
    y = poisson(O.forward_project(xt, h), 101)
    optics = O.Optics(nnum=cfg.nnum, **OPTICS)
    res = O.deconvolve(y, h, optics, O.Policy(mode="fixed", n_iters=10))
    assert res.stop_iter == 10 and len(res.series) == 10
    assert res.best_iter == int(np.argmax(res.series)) + 1
    assert res.volume.min() >= 0
    res2 = O.deconvolve(y, h, optics, O.Policy(mode="auto", max_iters=30))
    s = res2.series
    if res2.stop_iter < 30:
        assert s[-1] < s[-2]
    # no strict decrease before the stop (patience 1, min_iters 2)
    assert all(not (s[k] < s[k - 1]) for k in range(1, len(s) - 1))


def test_deconvolve_rejects_zero_measurement():
    h = np.ones((1, 3, 3, 3, 3)) / 9
    with pytest.raises(ValueError):
        O.deconvolve(np.zeros((9, 9)), h, O.Optics(nnum=3, **OPTICS), O.Policy())


def test_deconvolve_returns_best_snapshot():
    """S:299 snapshot correctness: the returned volume equals, bit for bit, the iterate obtained by re-running the
    update best_iter times from the same init (here chained by hand from initial_volume and rl_step, outside the
    loop's bookkeeping), and it is not the last iterate when the run went on past the best one."""
    cfg = CONFIGS["tiny"]
    h = gen_psf(cfg, np.float64)
    optics = O.Optics(nnum=cfg.nnum, **OPTICS)
    checked = 0
    for seed in (1, 2, 3):
        y = poisson(O.forward_project(gen_volume(cfg, seed), h), 100 + seed)
        res = O.deconvolve(y, h, optics, O.Policy(mode="auto", max_iters=30))
        norm = O.compute_normalizer(h, cfg.height, cfg.width)
        x = O.initial_volume(y, h, cfg.nz, cfg.height, cfg.width)
        chain = []
        for _ in range(res.stop_iter):
            x, _ = O.rl_step(x, y, h, norm)
            chain.append(x)
        assert np.array_equal(res.volume, chain[res.best_iter - 1])
        if res.best_iter < res.stop_iter:
            assert not np.array_equal(res.volume, chain[-1])
            checked += 1
    assert checked > 0


def test_isra_start_closed_form():
    """ISRA starts from x0 = H^T y (reading C23).  Closed form with two planes of delta PSFs of weights 1 and 2
    (H x = x_0 + 2 x_1, H^T r = (r, 2 r)): x0 = (y, 2y), H x0 = 5y, H^T H x0 = (5y, 10y), so
    x1 = x0 H^T y / H^T H x0 = (y/5, 2y/5).  A uniform start c would give (y/3, y/3) instead."""
    rng = np.random.default_rng(7)
    N, K, H = 3, 3, 12
    h = np.zeros((2, N, N, K, K))
    h[0, :, :, 1, 1] = 1.0
    h[1, :, :, 1, 1] = 2.0
    y = rng.poisson(20, (H, H)).astype(float) + 1.0
    res = O.deconvolve(y, h, O.Optics(nnum=N, **OPTICS), O.Policy(mode="fixed", n_iters=1), update="isra")
    np.testing.assert_allclose(res.volume[0], y / 5, rtol=1e-14)
    np.testing.assert_allclose(res.volume[1], 2 * y / 5, rtol=1e-14)

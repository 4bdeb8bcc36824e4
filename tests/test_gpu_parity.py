"""GPU parity (marked gpu): the CUDA path, called through the C ABI, against the fp64 oracle on the
same seeded inputs.  Tolerances: operators rel-L2 <= 2e-6 and max-abs <= 1e-5 * max|ref| on
the CUDA-core paths (fp32 FFT + fp32 MAC over nz N^2 terms, measured ~1e-7); <= 1e-5 rel-L2 / 2e-5 max-abs
when planes run on the tcgen05 direct path (2xFP16 split, 3 products; its fp32 accumulation truncates: bias up to ~3e-6
relative over ~250 chained MMAs); RL rel-L2 <= 1e-4 after 1 iteration and
<= 1e-3 after 30 (BASELINE.json north star); identical stop / best iteration unless the decision margin is
within 10x the observed entropy error (reading C16)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from lfm_inputs import CONFIGS, OPTICS, Config, gen_psf, gen_volume, lf_like, poisson  # noqa: E402
from oracle import lfm_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

OPT = O.Optics(nnum=0, **OPTICS)


def L():
    from paper_2208_11422_b200 import lfm
    return lfm


def dev(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def optics(nnum):
    return L().make_optics(**OPTICS)


def op_tol(info):
    """(rel-L2, max-abs/max) operator tolerance: CUDA-core paths 2e-6 / 1e-5; tcgen05 planes (2xFP16 split) 1e-5 / 2e-5."""
    return (1e-5, 2e-5) if info.get("tc_planes", 0) > 0 else (2e-6, 1e-5)


def rand_case(seed, nz, N, H, W, kh, kw):
    rng = np.random.default_rng(seed)
    h = rng.uniform(0, 1, (nz, N, N, kh, kw)).astype(np.float32)
    h /= h.sum(axis=(3, 4), keepdims=True)
    x = rng.uniform(0, 1, (nz, H, W)).astype(np.float32)
    r = rng.uniform(0.5, 1.5, (H, W)).astype(np.float32)
    return h, x, r


OP_CASES = [  # (nz, N, H, W, kh, kw): tiny, ragged units, non-square, radix 2/3/5 mixes, N=1, kernel > image
    (3, 3, 33, 33, 9, 9),
    (2, 3, 27, 36, 7, 11),
    (4, 5, 45, 45, 15, 15),
    (2, 1, 20, 24, 5, 7),
    (2, 3, 9, 9, 21, 21),
    (5, 7, 63, 49, 29, 21),
]


@pytest.mark.parametrize("flags", [0, 2, 4, 18, 64], ids=["hybrid", "direct", "fft", "direct-tc", "hybrid-notc"])
@pytest.mark.parametrize("case", OP_CASES, ids=[str(c) for c in OP_CASES])
def test_projections_match_oracle(case, flags):
    nz, N, H, W, kh, kw = case
    h, x, r = rand_case(sum(case), *case)
    hd = h.astype(np.float64)
    with L().Plan(h, N, H, W, optics=optics(N), flags=flags) as plan:
        y_d = torch.zeros((H, W), device="cuda")
        plan.forward(dev(x), y_d)
        xb_d = torch.zeros((nz, H, W), device="cuda")
        plan.backward(dev(r), xb_d)
        nrm_d = torch.zeros((nz, H, W), device="cuda")
        plan.normalizer(nrm_d)
        torch.cuda.synchronize()
        info = plan.info()
    y_ref = O.forward_project(x.astype(np.float64), hd)
    xb_ref = O.backward_project(r.astype(np.float64), hd)
    nrm_ref = O.compute_normalizer(hd, H, W)
    tol, mtol = op_tol(info)
    for got, ref in [(y_d, y_ref), (xb_d, xb_ref), (nrm_d, nrm_ref)]:
        g = got.cpu().numpy()
        assert rel(g, ref) <= tol, (rel(g, ref), info)
        assert np.abs(g - ref).max() <= mtol * np.abs(ref).max()
    if flags == 4:
        assert info["fft_h"] >= info["lc_min_h"] and info["fft_w"] >= info["lc_min_w"]
        assert info["direct_planes"] == 0 and info["fft_units"] == nz * N * N
    if flags & 2:
        assert info["direct_planes"] == nz and info["fft_units"] == 0


def test_adjoint_on_gpu():
    """<Hx, y> = <x, H^T y> for the GPU operators (fp32: 1e-5 relative)."""
    h, x, r = rand_case(7, 3, 5, 45, 45, 15, 15)
    with L().Plan(h, 5, 45, 45, optics=optics(5)) as plan:
        y_d = torch.zeros((45, 45), device="cuda")
        plan.forward(dev(x), y_d)
        xb_d = torch.zeros((3, 45, 45), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
    lhs = np.vdot(y_d.cpu().numpy().astype(np.float64), r)
    rhs = np.vdot(x.astype(np.float64), xb_d.cpu().numpy())
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


@pytest.mark.parametrize("flags", [0, 18], ids=["hybrid", "direct-tc"])
def test_c2_operators_match_oracle(flags):
    """BASELINE configs[1] geometry (N=11, 319^2, 21 planes, K=99): full-image operator parity."""
    cfg = CONFIGS["c2"]
    h = gen_psf(cfg, np.float32)
    x = gen_volume(cfg, 1, np.float32)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
        tol = op_tol(plan.info())[0]
        y_d = torch.zeros((cfg.height, cfg.width), device="cuda")
        plan.forward(dev(x), y_d)
        torch.cuda.synchronize()
        y_ref = O.forward_project(x.astype(np.float64), h.astype(np.float64))
        assert rel(y_d.cpu().numpy(), y_ref) <= tol
        r = (y_ref + 1.0) / (y_ref.mean() + 1.0)
        xb_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
    xb_ref = O.backward_project(r.astype(np.float32).astype(np.float64), h.astype(np.float64))
    assert rel(xb_d.cpu().numpy(), xb_ref) <= tol


@pytest.mark.gpu
def test_memory_aware_planning():
    """A capped device (lfm_set_memory_limit) makes the hybrid planner move planes off the frequency path until the
    transfer matrices fit; the operators still match the oracle.  An impossible cap fails with LFM_ENOMEM naming the
    limiting term.  PSF bank: two wide planes (per-pair tap box D = 13: the frequency path is faster, the tensor-core
    taps need less memory than their transfer matrices) and two narrow ones (D = 1)."""
    L_ = L()
    N, H, W, K = 11, 319, 319, 143
    rng = np.random.default_rng(11)
    h = np.zeros((4, N, N, K, K), np.float32)
    h[:2] = rng.uniform(0, 1, (2, N, N, K, K))
    c = K // 2
    h[2:, :, :, c - 5:c + 6, c - 5:c + 6] = rng.uniform(0, 1, (2, N, N, 11, 11))
    h /= h.sum(axis=(3, 4), keepdims=True)
    x = rng.uniform(0, 1, (4, H, W)).astype(np.float32)
    nt = L_.LFM_PLAN_NO_TILES   # whole-image transfer matrices (the estimate's model; tiles need far less memory)
    try:
        with L_.Plan(h, N, H, W, optics=optics(N), flags=nt) as free:
            assert free.info()["fft_units"] > 0
        with L_.Plan(h, N, H, W, optics=optics(N), flags=L_.LFM_PLAN_FFT_ONLY | nt) as full:
            m_all = full.info()["transfer_bytes"]
        est, _ = L_.lfm_plan_estimate(N, 4, K, K, H, W)   # all-frequency-path estimate: transfer + the rest
        L_.lfm_set_memory_limit(int(est - m_all + 0.45 * m_all))   # fits only after moving the wide planes
        with L_.Plan(h, N, H, W, optics=optics(N), flags=nt) as plan:
            info = plan.info()
            assert info["planes_moved_for_memory"] > 0
            tol = op_tol(info)[0]
            y_d = torch.zeros((H, W), device="cuda")
            plan.forward(dev(x), y_d)
            torch.cuda.synchronize()
            y_ref = O.forward_project(x.astype(np.float64), h.astype(np.float64))
            assert rel(y_d.cpu().numpy(), y_ref) <= tol
            r = (y_ref + 1.0) / (y_ref.mean() + 1.0)
            xb_d = torch.zeros((4, H, W), device="cuda")
            plan.backward(dev(r), xb_d)
            torch.cuda.synchronize()
        xb_ref = O.backward_project(r.astype(np.float32).astype(np.float64), h.astype(np.float64))
        assert rel(xb_d.cpu().numpy(), xb_ref) <= tol
        L_.lfm_set_memory_limit(1 << 20)
        with pytest.raises(L_.LfmError) as e:
            L_.Plan(h, N, H, W, optics=optics(N))
        assert "LFM_ENOMEM" in str(e.value) and "limiting term" in str(e.value)
    finally:
        L_.lfm_set_memory_limit(0)


def tiny_problem(name="tiny", seed=1):
    cfg = CONFIGS[name]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    xt = gen_volume(cfg, seed)
    y = poisson(O.forward_project(xt, hd), 100 + seed)
    return cfg, h, hd, y


def oracle_iterates(y, hd, cfg, n):
    norm = O.compute_normalizer(hd, cfg.height, cfg.width)
    x = O.initial_volume(y, hd, cfg.nz, cfg.height, cfg.width)
    reg = O.cutoff_region(O.Optics(nnum=cfg.nnum, **OPTICS), cfg.height, cfg.width)
    out, es = [], []
    for _ in range(n):
        x, _ = O.rl_step(x, y, hd, norm)
        out.append(x.copy())
        es.append(O.evaluate_iteration(x, reg))
    return out, es


@pytest.mark.parametrize("flags", [0, 2, 4, 18], ids=["hybrid", "direct", "fft", "direct-tc"])
def test_rl_tiny_1_and_30_iterations(flags):
    """North star: rel-L2 <= 1e-4 after 1 iteration, <= 1e-3 after 30; E_k within 1e-4 relative."""
    cfg, h, hd, y = tiny_problem()
    xs, es = oracle_iterates(y, hd, cfg, 30)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
        y_d = dev(y)
        for n, tol in [(1, 1e-4), (10, 1e-3), (30, 1e-3)]:
            x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
            res = plan.rl_iterate(y_d, x_d, L().make_policy(mode="fixed", n_iters=n))
            assert res["stop_iter"] == n
            # fixed mode returns the argmax-E iterate; compare against the oracle's same iterate
            assert res["best_iter"] == int(np.argmax(es[:n])) + 1
            assert rel(x_d.cpu().numpy(), xs[res["best_iter"] - 1]) <= tol
            np.testing.assert_allclose(res["series"], es[:n], rtol=1e-4)


def test_rl_step_matches_oracle_step_by_step():
    """lfm_rl_step: each GPU step from the oracle's own iterate stays within 1e-5 of the oracle's next."""
    cfg, h, hd, y = tiny_problem(seed=2)
    xs, es = oracle_iterates(y, hd, cfg, 5)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum)) as plan:
        y_d = dev(y)
        for k in range(4):
            xo = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
            yh = torch.zeros((cfg.height, cfg.width), device="cuda")
            e = plan.rl_step(y_d, dev(xs[k]), xo, yhat_out=yh)
            assert rel(xo.cpu().numpy(), xs[k + 1]) <= 1e-5
            assert abs(e - es[k + 1]) <= 1e-5 * abs(es[k + 1])
            assert rel(yh.cpu().numpy(), O.forward_project(xs[k].astype(np.float32).astype(np.float64), hd)) <= 2e-6


def stop_parity(cfg, h, hd, y, max_iters=50, flags=0):
    res_o = O.deconvolve(y, hd, O.Optics(nnum=cfg.nnum, **OPTICS), O.Policy(mode="auto", max_iters=max_iters))
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="auto", max_iters=max_iters))
        torch.cuda.synchronize()
    n = min(len(res["series"]), len(res_o.series))
    err = max(abs(a - b) / abs(b) for a, b in zip(res["series"][:n], res_o.series[:n]))
    s = res_o.series
    k = res_o.stop_iter
    margin = min(abs(s[i] - s[i - 1]) / abs(s[i]) for i in range(1, k)) if k > 1 else 1.0
    return res, res_o, err, margin, x_d


@pytest.mark.parametrize("name,seed,flags", [("tiny", 1, 0), ("tiny", 3, 0), ("s15", 1, 0), ("s15", 1, 18)])
def test_auto_stop_identical(name, seed, flags):
    """Identical stop_iter and best_iter vs the oracle (P:99 stop rule) unless tie-ambiguous (C16)."""
    cfg, h, hd, y = tiny_problem(name, seed)
    res, res_o, err, margin, x_d = stop_parity(cfg, h, hd, y, flags=flags)
    assert err <= 1e-4
    if margin <= 10 * err:
        pytest.skip(f"tie-ambiguous: decision margin {margin:.2e} <= 10 x entropy error {err:.2e} (C16)")
    assert (res["stop_iter"], res["best_iter"]) == (res_o.stop_iter, res_o.best_iter)
    assert rel(x_d.cpu().numpy(), res_o.volume) <= 1e-3


def test_c2_rl_8_iterations():
    """BASELINE configs[1]: N=11, 319^2, 21 planes, 8 RL iterations (fixed)."""
    cfg, h, hd, y = tiny_problem("c2", 1)
    xs, es = oracle_iterates(y, hd, cfg, 8)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum)) as plan:
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=8))
        torch.cuda.synchronize()
    assert res["best_iter"] == int(np.argmax(es)) + 1
    assert rel(x_d.cpu().numpy(), xs[res["best_iter"] - 1]) <= 1e-3
    np.testing.assert_allclose(res["series"], es, rtol=1e-4)
    x1 = xs[0]
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum)) as plan:
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=1))
        assert rel(x_d.cpu().numpy(), x1) <= 1e-4


def test_dct_entropy_standalone():
    """Eq. (12) on the GPU (fp64) vs the oracle on full-size images, triangle and rectangle."""
    for (H, W, N) in [(1005, 1005, 15), (319, 319, 11), (33, 33, 3), (225, 300, 15)]:
        img = lf_like(Config("t", N, H, W, 1, 1, 0, 1, 0, 0, 0, "beads", 0, 1, 1, 0), 5).astype(np.float32)
        for shape, code in [("triangle", 0), ("rectangle", 1)]:
            e, xs, ys = L().lfm_dct_entropy(dev(img), N, optics(N), code)
            reg = O.cutoff_region(O.Optics(nnum=N, **OPTICS), H, W, shape)
            assert (xs, ys) == (reg.x_s, reg.y_s)
            assert e == pytest.approx(O.dct_entropy(img.astype(np.float64), reg), rel=1e-10)


def test_virtual_shards_partition():
    """S:352 depth/phase sharding: NO_COMM plans of rank r/world own contiguous unit ranges; their partial
    forwards sum to the full forward and their backwards cover disjoint units (world 2, 3, 4)."""
    L_ = L()
    h, x, r = rand_case(11, 4, 3, 27, 27, 9, 9)
    hd = h.astype(np.float64)
    y_ref = O.forward_project(x.astype(np.float64), hd)
    xb_ref = O.backward_project(r.astype(np.float64), hd)
    for world in (2, 3, 4):
        tot = np.zeros_like(y_ref)
        cover = np.zeros((4, 27, 27))
        xb_acc = np.zeros_like(xb_ref)
        for rank in range(world):
            with L_.Plan(h, 3, 27, 27, optics=optics(3), rank=rank, world=world, flags=L_.LFM_PLAN_NO_COMM) as plan:
                info = plan.info()
                assert plan.owned() == L_.lfm_shard_units_balanced(h, 3, 27, 27, world, rank)[:2] == (
                    info["unit_begin"], info["unit_end"])
                y_d = torch.zeros((27, 27), device="cuda")
                plan.forward(dev(x), y_d)
                xb_d = torch.full((4, 27, 27), -1.0, device="cuda")
                plan.backward(dev(r), xb_d)
                torch.cuda.synchronize()
                tot += y_d.cpu().numpy()
                xb = xb_d.cpu().numpy()
                own = xb != -1.0
                cover += own
                xb_acc[own] = xb[own]
                nu = 4 * 9
                assert info["unit_begin"] == rank * (nu // world) + min(rank, nu % world)
        assert rel(tot, y_ref) <= 2e-6
        assert (cover == 1).all()
        assert rel(xb_acc, xb_ref) <= 2e-6


def test_error_statuses():
    L_ = L()
    h, x, r = rand_case(1, 2, 3, 9, 9, 3, 3)
    with pytest.raises(L_.LfmError) as e:
        L_.Plan(h, 3, 10, 9)
    assert e.value.status == L_.LFM_EDIM
    hn = h.copy()
    hn[0, 0, 0, 0, 0] = -1
    with pytest.raises(L_.LfmError) as e:
        L_.Plan(hn, 3, 9, 9)
    assert e.value.status == L_.LFM_ENEG
    h0 = h.copy()
    h0[1] = 0.0   # at least one nonzero kernel per plane
    with pytest.raises(L_.LfmError) as e:
        L_.Plan(h0, 3, 9, 9)
    assert e.value.status == L_.LFM_EZERO and "z=1" in str(e.value)
    hs = np.zeros((1, 3, 3, 21, 21), np.float32)   # every kernel's only tap lies 10 pixels off-centre: on a 9x9
    hs[0, :, :, 0, 0] = 1.0                        # image no voxel reaches a pixel, sum H^T 1 = 0
    with pytest.raises(L_.LfmError) as e:
        L_.Plan(hs, 3, 9, 9)
    assert e.value.status == L_.LFM_EZERO and "projects nothing" in str(e.value)
    with L_.Plan(h, 3, 9, 9, optics=optics(3)) as plan:
        x_d = torch.zeros((2, 9, 9), device="cuda")
        with pytest.raises(L_.LfmError) as e:
            plan.rl_iterate(torch.zeros((9, 9), device="cuda"), x_d, L_.make_policy())
        assert e.value.status == L_.LFM_EZERO
        yneg = torch.ones((9, 9), device="cuda")
        yneg[1, 1] = -2
        with pytest.raises(L_.LfmError) as e:
            plan.rl_iterate(yneg, x_d, L_.make_policy())
        assert e.value.status == L_.LFM_ENEG
        with pytest.raises(L_.LfmError) as e:
            plan.rl_iterate(torch.ones((9, 9), device="cuda"), x_d, L_.make_policy(min_iters=9, max_iters=3))
        assert e.value.status == L_.LFM_EINVAL
        with pytest.raises(L_.LfmError) as e:
            plan.rl_iterate(torch.ones((9, 9), device="cuda"), x_d, L_.make_policy(eps=0.0))
        assert e.value.status == L_.LFM_EINVAL


def test_host_buffer_call_and_quality():
    """lfm_deconvolve_host (the e2e call) equals lfm_rl_iterate; lfm_quality equals the oracle's E."""
    cfg, h, hd, y = tiny_problem(seed=4)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum)) as plan:
        pol = L().make_policy(mode="auto", max_iters=30)
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        r1 = plan.rl_iterate(dev(y), x_d, pol)
        xh = np.zeros((cfg.nz, cfg.height, cfg.width), np.float32)
        r2 = plan.deconvolve_host(np.ascontiguousarray(y, np.float32), xh, pol)
        assert (r1["stop_iter"], r1["best_iter"]) == (r2["stop_iter"], r2["best_iter"])
        assert np.array_equal(xh, x_d.cpu().numpy())
        e = plan.quality(x_d)
    reg = O.cutoff_region(O.Optics(nnum=cfg.nnum, **OPTICS), cfg.height, cfg.width)
    assert e == pytest.approx(O.evaluate_iteration(x_d.cpu().numpy().astype(np.float64), reg), rel=1e-10)
    assert e == pytest.approx(r1["series"][r1["best_iter"] - 1], rel=1e-6)


def _nonzero_rows(h, z):
    nzr = np.nonzero(h[z].reshape(-1, h.shape[3], h.shape[4]).any(axis=(0, 2)))[0]
    return int(nzr.min()), int(nzr.max())


@pytest.fixture(scope="module")
def c3_plan():
    """The c3 workload in the launch configuration bench.py times (frequency path, 75x75, 1 GPU)."""
    cfg = CONFIGS["c3"]
    h = gen_psf(cfg, np.float32)
    plan = L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum))
    yield cfg, h, plan
    plan.close()


def test_c3_forward_backward_sampled(c3_plan):
    """Full-size c3: forward at 64 sampled pixels and backward at 64 sampled voxels (corners, borders, interior,
    all planes) against the oracle's one-output evaluators; |err| <= 1e-5 max|ref|."""
    cfg, h, plan = c3_plan
    hd = h.astype(np.float64)
    rng = np.random.default_rng(0)
    x = gen_volume(cfg, 2, np.float32)
    y_d = torch.zeros((cfg.height, cfg.width), device="cuda")
    plan.forward(dev(x), y_d)
    torch.cuda.synchronize()
    yg = y_d.cpu().numpy()
    H, W = cfg.height, cfg.width
    s = np.concatenate([[0, 0, H - 1, H - 1, 7, H // 2], rng.integers(0, H, 58)])
    t = np.concatenate([[0, W - 1, 0, W - 1, W // 2, 3], rng.integers(0, W, 58)])
    ref = O.forward_points(x.astype(np.float64), hd, s, t)
    assert np.abs(yg[s, t] - ref).max() <= 1e-5 * np.abs(yg).max()
    r = (lf_like(cfg, 3) + 1.0).astype(np.float32)
    r /= r.mean()
    xb_d = torch.zeros((cfg.nz, H, W), device="cuda")
    plan.backward(dev(r), xb_d)
    torch.cuda.synchronize()
    z = np.concatenate([[0, cfg.nz - 1, cfg.nz // 2, 10], rng.integers(0, cfg.nz, 60)])
    p = np.concatenate([[0, H - 1, 500, 14], rng.integers(0, H, 60)])
    q = np.concatenate([[0, W - 1, 501, 1004], rng.integers(0, W, 60)])
    refb = O.backward_points(r.astype(np.float64), hd, z, p, q)
    got = xb_d[torch.from_numpy(z).cuda(), torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()].cpu().numpy()
    assert np.abs(got - refb).max() <= 1e-5 * np.abs(refb).max()


def test_c3_one_rl_step_sampled(c3_plan):
    """Full-size c3, one RL step from a random positive x0 (init_from_x): x1 at 12 sampled voxels of the
    near-focus planes computed by the oracle from its own forward / backward evaluators; 1e-5 relative."""
    cfg, h, plan = c3_plan
    hd = h.astype(np.float64)
    H, W = cfg.height, cfg.width
    rng = np.random.default_rng(5)
    y = lf_like(cfg, 9).astype(np.float32)
    x0 = (rng.uniform(0.5, 1.5, (cfg.nz, H, W)) * (y.mean() / cfg.nz)).astype(np.float32)
    x1_d = torch.zeros((cfg.nz, H, W), device="cuda")
    e = plan.rl_step(dev(y), dev(x0), x1_d)
    torch.cuda.synchronize()
    x1 = x1_d.cpu().numpy()
    x0d = x0.astype(np.float64)
    yd = y.astype(np.float64)
    ch = cfg.k_max // 2
    ones = np.ones((H, W))
    for z in (25, 24, 26, 21):
        i0, i1 = _nonzero_rows(hd, z)
        for _ in range(3):
            p, q = int(rng.integers(0, H)), int(rng.integers(0, W))
            ss = [p + i - ch for i in range(i0, i1 + 1) if 0 <= p + i - ch < H]
            tt = [q + j - ch for j in range(i0, i1 + 1) if 0 <= q + j - ch < W]
            S, T = np.meshgrid(ss, tt, indexing="ij")
            yhat = O.forward_points(x0d, hd, S.ravel(), T.ravel())
            rimg = np.zeros((H, W))
            rimg[S.ravel(), T.ravel()] = yd[S.ravel(), T.ravel()] / (yhat + O.EPS)
            bp = O.backward_points(rimg, hd, [z], [p], [q])[0]
            nrm = O.backward_points(ones, hd, [z], [p], [q])[0]
            ref = x0d[z, p, q] * bp / max(nrm, O.EPS)
            assert abs(x1[z, p, q] - ref) <= 1e-5 * abs(ref), (z, p, q, x1[z, p, q], ref)
    assert e > 0


@pytest.mark.parametrize("flags", [0, 18], ids=["hybrid", "all-tc"])
def test_c4_geometry_sampled(flags):
    """Maximum sizes: the c4 geometry (Nnum 15, 2025^2 image, K = 225) with 6 planes whose per-pair tap boxes span
    D = 3 / 9 / 15 -- on the tensor-core path a 17 x 17 union box (289 taps) over 135 x 151 coarse pixels.  Forward at
    64 sampled pixels and backward at 64 sampled voxels against the oracle's one-output evaluators."""
    import dataclasses
    cfg = dataclasses.replace(CONFIGS["c4"], name="c4_6", nz=6)
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    H, W = cfg.height, cfg.width
    rng = np.random.default_rng(4)
    x = rng.uniform(0, 1, (cfg.nz, H, W)).astype(np.float32)
    with L().Plan(h, cfg.nnum, H, W, optics=optics(cfg.nnum), flags=flags) as plan:
        info = plan.info()
        if flags == 18:
            assert info["tc_planes"] == cfg.nz
        y_d = torch.zeros((H, W), device="cuda")
        plan.forward(dev(x), y_d)
        torch.cuda.synchronize()
        yg = y_d.cpu().numpy()
        s = np.concatenate([[0, 0, H - 1, H - 1, 7, H // 2], rng.integers(0, H, 58)])
        t = np.concatenate([[0, W - 1, 0, W - 1, W // 2, 3], rng.integers(0, W, 58)])
        ref = O.forward_points(x.astype(np.float64), hd, s, t)
        assert np.abs(yg[s, t] - ref).max() <= 1e-5 * np.abs(yg).max()
        r = rng.uniform(0.5, 1.5, (H, W)).astype(np.float32)
        xb_d = torch.zeros((cfg.nz, H, W), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
    z = np.concatenate([[0, cfg.nz - 1, 2, 3], rng.integers(0, cfg.nz, 60)])
    p = np.concatenate([[0, H - 1, 1000, 14], rng.integers(0, H, 60)])
    q = np.concatenate([[0, W - 1, 1001, 2024], rng.integers(0, W, 60)])
    refb = O.backward_points(r.astype(np.float64), hd, z, p, q)
    got = xb_d[torch.from_numpy(z).cuda(), torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()].cpu().numpy()
    assert np.abs(got - refb).max() <= 1e-5 * np.abs(refb).max()


@pytest.mark.parametrize("flags", [0, 2, 4, 18], ids=["hybrid", "direct", "fft", "direct-tc"])
def test_isra_matches_oracle(flags):
    """MATLAB-lineage ISRA update x * H^T y / H^T H x from x0 = H^T y; 1 and 10 iterations."""
    cfg, h, hd, y = tiny_problem(seed=5)
    for n, tol in [(1, 1e-4), (10, 1e-3)]:
        ref = O.deconvolve(y, hd, O.Optics(nnum=cfg.nnum, **OPTICS), O.Policy(mode="fixed", n_iters=n),
                           update="isra", keep_iterates=True)
        with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
            x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
            res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=n, update="isra"))
            torch.cuda.synchronize()
        assert res["best_iter"] == ref.best_iter
        assert rel(x_d.cpu().numpy(), ref.iterates[res["best_iter"] - 1]) <= tol
        np.testing.assert_allclose(res["series"], ref.series, rtol=1e-4)


@pytest.mark.parametrize("flags", [0, 2, 4, 18], ids=["hybrid", "direct", "fft", "direct-tc"])
def test_supplied_ht(flags):
    """f3: a supplied transposed PSF Ht drives the backward (and normalizer); Ht = rot180(H) reproduces the
    exact-adjoint plan; an unrelated Ht matches the oracle's Ht backward."""
    h, x, r = rand_case(21, 3, 3, 27, 33, 9, 9)
    rng = np.random.default_rng(22)
    ht = rng.uniform(0, 1, h.shape).astype(np.float32)
    with L().Plan(h, 3, 27, 33, optics=optics(3), flags=flags, psf_t=ht) as plan:
        xb_d = torch.zeros((3, 27, 33), device="cuda")
        plan.backward(dev(r), xb_d)
        nrm_d = torch.zeros((3, 27, 33), device="cuda")
        plan.normalizer(nrm_d)
        y_d = torch.zeros((27, 33), device="cuda")
        plan.forward(dev(x), y_d)
        torch.cuda.synchronize()
        tol = op_tol(plan.info())[0]
    assert rel(xb_d.cpu().numpy(), O.backward_project_ht(r.astype(np.float64), ht.astype(np.float64))) <= tol
    assert rel(nrm_d.cpu().numpy(), O.backward_project_ht(np.ones((27, 33)), ht.astype(np.float64))) <= tol
    assert rel(y_d.cpu().numpy(), O.forward_project(x.astype(np.float64), h.astype(np.float64))) <= tol
    with L().Plan(h, 3, 27, 33, optics=optics(3), flags=flags, psf_t=np.ascontiguousarray(h[:, :, :, ::-1, ::-1])) as p1, \
            L().Plan(h, 3, 27, 33, optics=optics(3), flags=flags) as p0:
        a_d = torch.zeros((3, 27, 33), device="cuda")
        b_d = torch.zeros((3, 27, 33), device="cuda")
        p1.backward(dev(r), a_d)
        p0.backward(dev(r), b_d)
        torch.cuda.synchronize()
        assert rel(a_d.cpu().numpy(), b_d.cpu().numpy().astype(np.float64)) <= 1e-6


def oracle_frame(y, hd, cfg, max_iters=25):
    """The oracle's auto-stop run of one frame, extended to >= 3 iterates for the fixed-3 comparison."""
    opt = O.Optics(nnum=cfg.nnum, **OPTICS)
    ref = O.deconvolve(y, hd, opt, O.Policy(mode="auto", max_iters=max_iters), keep_iterates=True)
    its = ref.iterates
    if len(its) < 3:
        its = O.deconvolve(y, hd, opt, O.Policy(mode="fixed", n_iters=3), keep_iterates=True).iterates
    return ref, its


@pytest.mark.parametrize("name,F,flags", [("tiny", 4, 0), ("tiny", 2, 4), ("c2", 4, 4), ("s15", 8, 0), ("c2", 16, 4),
                                          ("s15", 16, 4), ("s15", 16, 0)])
def test_batched_frames_match_single_and_oracle(name, F, flags):
    """f1: lockstep frame batching (F = 8 / 16 engage the tcgen05 batched MACs on the frequency-path planes).
    Against the fp64 oracle, frame by frame (every frame; c2 at F = 16: frames 0, 1, F/2, F-1): fixed 3 iterations
    and auto-stop -- identical stop / best iterations (C16 margin rule), E_k within 1e-4, volumes within 1e-3.
    Against the single-frame plan: equal within fp32 re-association (1e-5)."""
    cfg = CONFIGS[name]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    ys = [poisson(O.forward_project(gen_volume(cfg, 1 + f % 3), hd) * (1.0 + 0.1 * f), 300 + f) for f in range(F)]
    check = list(range(F)) if not (name == "c2" and F > 4) else [0, 1, F // 2, F - 1]
    refs = {f: oracle_frame(ys[f], hd, cfg) for f in check}
    # (whole-image transforms: the lockstep batched MACs; tiled plans batch frame by frame, test_gpu_tiles.py)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags | L().LFM_PLAN_NO_TILES) as plan:
        for pol in (L().make_policy(mode="fixed", n_iters=3), L().make_policy(mode="auto", max_iters=25)):
            yb = dev(np.stack(ys))
            xb = torch.zeros((F, cfg.nz, cfg.height, cfg.width), device="cuda")
            rb = plan.rl_iterate_batch(yb, xb, pol)
            for f in range(F):
                x1 = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
                r1 = plan.rl_iterate(dev(ys[f]), x1, pol)
                assert (rb["stop_iter"][f], rb["best_iter"][f]) == (r1["stop_iter"], r1["best_iter"])
                np.testing.assert_allclose(rb["series"][f], r1["series"], rtol=1e-5)
                assert rel(xb[f].cpu().numpy(), x1.cpu().numpy().astype(np.float64)) <= 1e-5
            for f in check:
                ref, its = refs[f]
                got = xb[f].cpu().numpy()
                if pol.mode == L().LFM_MODE_FIXED:
                    es = [O.evaluate_iteration(its[k], O.cutoff_region(O.Optics(nnum=cfg.nnum, **OPTICS), cfg.height,
                                                                        cfg.width)) for k in range(3)]
                    assert rb["best_iter"][f] == int(np.argmax(es)) + 1
                    np.testing.assert_allclose(rb["series"][f], es, rtol=1e-4)
                    assert rel(got, its[rb["best_iter"][f] - 1]) <= 1e-3
                    continue
                n = min(len(ref.series), len(rb["series"][f]))
                err = max(abs(a - b) / abs(b) for a, b in zip(rb["series"][f][:n], ref.series[:n]))
                assert err <= 1e-4, (f, err)
                k = ref.stop_iter
                margin = min(abs(ref.series[i] - ref.series[i - 1]) / abs(ref.series[i]) for i in range(1, k)) if k > 1 else 1.0
                if margin <= 10 * err:
                    continue   # tie-ambiguous frame (C16)
                assert (rb["stop_iter"][f], rb["best_iter"][f]) == (ref.stop_iter, ref.best_iter), f
                assert rel(got, ref.volume) <= 1e-3


@pytest.mark.parametrize("name", ["tiny", "c2"])
def test_graph_replay_identical(name):
    """f4: with LFM_PLAN_GRAPHS each iteration replays a captured CUDA graph; results are bit-identical to the
    eager launches (same kernels, same order) and the replay is not slower."""
    cfg, h, hd, y = tiny_problem(name, 2)
    s = torch.cuda.Stream()
    out = {}
    with torch.cuda.stream(s):
        for flags in (0, L().LFM_PLAN_GRAPHS):
            with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
                x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
                plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=3), stream=s)   # warm / capture
                r = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="auto", max_iters=30), want_ms=True, stream=s)
                s.synchronize()
                out[flags] = (r, x_d.cpu().numpy())
    (r0, x0), (r1, x1) = out[0], out[L().LFM_PLAN_GRAPHS]
    assert (r0["stop_iter"], r0["best_iter"]) == (r1["stop_iter"], r1["best_iter"])
    assert r0["series"] == r1["series"] and np.array_equal(x0, x1)


@pytest.mark.gpu
@pytest.mark.parametrize("name,mode,update", [("tiny", "auto", "rl"), ("s15", "auto", "rl"), ("c2", "fixed", "rl"),
                                              ("tiny", "auto", "isra")])
def test_device_loop_identical(name, mode, update):
    """f4: with LFM_PLAN_DEVICE_LOOP the whole auto-stop loop is one graph launch (conditional WHILE node, stop rule
    and argmax snapshot on the device).  Same kernels in the same order as the host loop, so the series, the stop /
    best iterations and the returned argmax volume are bit-identical."""
    cfg, h, hd, y = tiny_problem(name, 2)
    s = torch.cuda.Stream()
    pol = L().make_policy(mode=mode, max_iters=30, n_iters=8, update=update)
    out = {}
    with torch.cuda.stream(s):
        for flags in (0, L().LFM_PLAN_DEVICE_LOOP):
            with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
                x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
                for _ in range(2):   # second call replays the cached graph
                    r = plan.rl_iterate(dev(y), x_d, pol, want_ms=True, stream=s)
                    s.synchronize()
                out[flags] = (r, x_d.cpu().numpy())
    (r0, x0), (r1, x1) = out[0], out[L().LFM_PLAN_DEVICE_LOOP]
    assert (r0["stop_iter"], r0["best_iter"]) == (r1["stop_iter"], r1["best_iter"])
    assert r0["series"] == r1["series"] and np.array_equal(x0, x1)
    if mode == "fixed":
        assert r1["stop_iter"] == 8
    # and the device-resident loop against the oracle (not only against the host loop)
    ref = O.deconvolve(y, hd, O.Optics(nnum=cfg.nnum, **OPTICS),
                       O.Policy(mode=mode, max_iters=30, n_iters=8), update=update)
    n = min(len(ref.series), len(r1["series"]))
    err = max(abs(a - b) / abs(b) for a, b in zip(r1["series"][:n], ref.series[:n]))
    assert err <= 1e-4, err
    k = ref.stop_iter
    margin = min(abs(ref.series[i] - ref.series[i - 1]) / abs(ref.series[i]) for i in range(1, k)) if k > 1 else 1.0
    if margin > 10 * err:
        assert (r1["stop_iter"], r1["best_iter"]) == (ref.stop_iter, ref.best_iter)
        assert rel(x1, ref.volume) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [0, 32, 128, 1024, 1024 | 32], ids=["eager", "graphs", "device-loop", "symmetric",
                                                                    "symmetric-graphs"])
def test_nccl_one_rank_identical(extra):
    """The sharded path's collectives executed for real over a one-rank NCCL communicator (LFM_PLAN_FORCE_COMM):
    communicator init from lfm_comm_unique_id, allreduce(sum) of yhat, allreduce(max) of the max-projection, the
    broadcast-gather of x_best -- eagerly, inside captured graphs and inside the conditional device loop.  Over one
    rank every collective is an identity, so results are bit-identical to the plan without a communicator."""
    L_ = L()
    cfg, h, hd, y = tiny_problem("c2", 3)
    s = torch.cuda.Stream()
    pol = L_.make_policy(mode="auto", max_iters=20)
    out = {}
    with torch.cuda.stream(s):
        for force in (False, True):
            kw = dict(nccl_id=L_.lfm_comm_unique_id(), flags=extra | L_.LFM_PLAN_FORCE_COMM) if force else \
                dict(flags=extra & ~1024)
            with L_.Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), stream=s, **kw) as plan:
                if force:
                    info_sym = plan.info()
                x = gen_volume(cfg, 2, np.float32)
                yh = torch.zeros((cfg.height, cfg.width), device="cuda")
                plan.forward(dev(x), yh, stream=s)
                xb = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
                plan.backward(dev(y.astype(np.float32)), xb, stream=s)
                x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
                r = plan.rl_iterate(dev(y), x_d, pol, stream=s)
                s.synchronize()
                out[force] = (yh.cpu().numpy(), xb.cpu().numpy(), r, x_d.cpu().numpy())
    a, b = out[False], out[True]
    if extra & 1024:   # C1 through our own kernel over the symmetric window (NVLS multimem where the box offers it)
        assert info_sym["c1_mode"] in (1, 2), info_sym
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert (a[2]["stop_iter"], a[2]["best_iter"], a[2]["series"]) == (b[2]["stop_iter"], b[2]["best_iter"], b[2]["series"])
    assert np.array_equal(a[3], b[3])


def mixed_problem():
    """The c2 geometry (N=11, 319^2) with a bank whose planes need very different tap boxes: 3 wide planes (K = 143,
    D = 13: the frequency path) and 5 narrow ones (D <= 3: the tensor cores), so the default plan holds both kinds."""
    import dataclasses
    cfg = dataclasses.replace(CONFIGS["c2"], name="mixed", nz=8, k_max=143)
    rng = np.random.default_rng(12)
    N, K = cfg.nnum, cfg.k_max
    h = np.zeros((cfg.nz, N, N, K, K), np.float32)
    c = K // 2
    for z in range(cfg.nz):
        half = c if z < 3 else (5 if z < 6 else 16)
        h[z, :, :, c - half:c + half + 1, c - half:c + half + 1] = rng.uniform(0, 1, (N, N, 2 * half + 1, 2 * half + 1))
    h /= h.sum(axis=(3, 4), keepdims=True)
    hd = h.astype(np.float64)
    y = poisson(O.forward_project(gen_volume(cfg, 1), hd), 77)
    return cfg, h, hd, y


@pytest.mark.gpu
@pytest.mark.parametrize("flags", [0, 32], ids=["eager", "graphs"])
def test_sm_partitions_identical(flags, monkeypatch):
    """§5.5: with the tensor-core planes and the frequency-path MAC side by side on disjoint SM partitions (green
    contexts, forced here with LFM_TC_SMS_F / _B) every kernel computes the same sums in the same order as the
    one-after-the-other plan (LFM_SERIAL): projections, the RL series and the volumes are bit-identical, eagerly
    and inside captured graphs."""
    cfg, h, hd, y = mixed_problem()
    x = gen_volume(cfg, 3, np.float32)
    r_img = np.asarray(y, np.float32) / np.float32(max(float(np.max(y)), 1.0)) + np.float32(0.5)
    monkeypatch.setenv("LFM_PLAN_MOVE", "0")   # the same plane assignment in both modes (no partition-aware moves)
    s = torch.cuda.Stream()
    out = {}
    with torch.cuda.stream(s):
        for mode in ("serial", "split"):
            if mode == "serial":
                monkeypatch.setenv("LFM_SERIAL", "1")
            else:
                monkeypatch.delenv("LFM_SERIAL", raising=False)
                monkeypatch.setenv("LFM_TC_SMS_F", "96")
                monkeypatch.setenv("LFM_TC_SMS_B", "104")
            with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
                info = plan.info()
                assert info["tc_planes"] > 0 and info["fft_units"] > 0, info
                y_d = torch.zeros((cfg.height, cfg.width), device="cuda")
                plan.forward(dev(x), y_d, stream=s)
                xb_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
                plan.backward(dev(r_img), xb_d, stream=s)
                x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
                plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=2), stream=s)
                res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=6), stream=s)
                s.synchronize()
                out[mode] = (info["partition_sms"], y_d.cpu().numpy(), xb_d.cpu().numpy(), res["series"],
                             x_d.cpu().numpy())
            monkeypatch.delenv("LFM_TC_SMS_F", raising=False)
            monkeypatch.delenv("LFM_TC_SMS_B", raising=False)
    ps, pp = out["serial"][0], out["split"][0]
    assert ps == [[0, 0], [0, 0]]
    assert pp[0][0] >= 96 and pp[1][0] >= 104 and pp[0][1] > 0 and pp[1][1] > 0
    for a, b in zip(out["serial"][1:], out["split"][1:]):
        if isinstance(a, list):
            assert a == b
        else:
            assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("name,flags", [("s15", 18), ("c2", 0)], ids=["s15-all-tc", "c2-hybrid"])
def test_tc_column_ranges_bit_identical(name, flags, monkeypatch):
    """§5.3 column ranges: every tcgen05 MMA after a drain group's first runs only over its coefficient tile's nonzero
    columns.  The skipped columns would add exact zeros, so projections and RL iterates are bit-identical to the
    full-width MMAs (LFM_TC_EXP=16)."""
    cfg, h, hd, y = tiny_problem(name, 2)
    x = gen_volume(cfg, 3, np.float32)
    r_img = np.asarray(y, np.float32) / np.float32(max(float(np.max(y)), 1.0)) + np.float32(0.5)
    out = {}
    for mode in ("full", "ranged"):
        if mode == "full":
            monkeypatch.setenv("LFM_TC_EXP", "16")
        else:
            monkeypatch.delenv("LFM_TC_EXP", raising=False)
        with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=flags) as plan:
            info = plan.info()
            if info["tc_planes"] == 0:
                pytest.skip("plan has no tensor-core planes")
            y_d = torch.zeros((cfg.height, cfg.width), device="cuda")
            plan.forward(dev(x), y_d)
            xb_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
            plan.backward(dev(r_img), xb_d)
            x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
            res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=4))
            torch.cuda.synchronize()
            out[mode] = (y_d.cpu().numpy(), xb_d.cpu().numpy(), res["series"], x_d.cpu().numpy(),
                         info["tc_flops_executed"])
    a, b = out["full"], out["ranged"]
    for u, v in zip(a[:4], b[:4]):
        if isinstance(u, list):
            assert u == v
        else:
            assert np.array_equal(u, v)
    assert b[4] <= a[4]   # executed tensor flops never grow


@pytest.mark.gpu
@pytest.mark.parametrize("mirror", [0, 1], ids=["final-copy", "mirror"])
@pytest.mark.parametrize("name,mode", [("tiny", "auto"), ("c2", "auto"), ("s15", "fixed")])
def test_host_call_pinned_mirror(name, mode, mirror, monkeypatch):
    """lfm_deconvolve_host into page-locked memory, with the single final copy (default) and with LFM_HOST_MIRROR
    (improving iterates converted and copied on a side stream while the next iteration runs; the call then skips its
    final copy).  The returned volume, series and stop / best iterations equal the device call's."""
    if mirror:
        monkeypatch.setenv("LFM_HOST_MIRROR", "1")
    cfg, h, hd, y = tiny_problem(name, 5)
    pol = L().make_policy(mode=mode, max_iters=30, n_iters=6)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum)) as plan:
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        r1 = plan.rl_iterate(dev(y), x_d, pol)
        torch.cuda.synchronize()
        xh_t = torch.full((cfg.nz, cfg.height, cfg.width), -1.0, dtype=torch.float32).pin_memory()
        r2 = plan.deconvolve_host(np.ascontiguousarray(y, np.float32), xh_t.numpy(), pol)
        assert (r1["stop_iter"], r1["best_iter"]) == (r2["stop_iter"], r2["best_iter"])
        assert r1["series"] == r2["series"]
        assert np.array_equal(xh_t.numpy(), x_d.cpu().numpy())


@pytest.mark.gpu
def test_batched_tc_macs_repeatable():
    """Race guard for the frame-batched tcgen05 MACs (compute-sanitizer is closed on this pool): every kernel of the
    batched path is deterministic, so 12 repetitions of the same F = 16 batch (s15, all planes through the batched
    forward and backward MACs, ring stages shared by the prep groups) must give bit-identical volumes and series; a
    prep group reading a half-filled tile (the r01 fault) would show up as a mismatch or a trap."""
    cfg = CONFIGS["s15"]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    F = 16
    ys = [poisson(O.forward_project(gen_volume(cfg, 1 + f % 3), hd) * (1.0 + 0.05 * f), 500 + f) for f in range(F)]
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum),
                  flags=L().LFM_PLAN_FFT_ONLY | L().LFM_PLAN_NO_TILES) as plan:
        yb = dev(np.stack(ys))
        ref = None
        for rep in range(12):
            xb = torch.zeros((F, cfg.nz, cfg.height, cfg.width), device="cuda")
            r = plan.rl_iterate_batch(yb, xb, L().make_policy(mode="fixed", n_iters=3))
            torch.cuda.synchronize()
            got = (xb.cpu().numpy(), r["series"])
            if ref is None:
                ref = got
            else:
                assert np.array_equal(got[0], ref[0]) and got[1] == ref[1], f"repetition {rep} differs"


@pytest.mark.gpu
@pytest.mark.parametrize("name,F", [("s15", 8), ("s15", 32), ("c2", 16)])
def test_frames_plan_matches_oracle(name, F):
    """LFM_PLAN_FRAMES (f1): the transfer matrices stored split into scaled fp16 hi / lo rows plus a split transposed
    copy; both batched passes on tcgen05 kind::f16.  Frames 0, 1, F/2, F-1 against the oracle: identical stop / best
    (C16 margin rule), series within 1e-4, volumes within 1e-3 (fixed 3 and auto); single-frame calls are refused."""
    cfg = CONFIGS[name]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    ys = [poisson(O.forward_project(gen_volume(cfg, 1 + f % 3), hd) * (1.0 + 0.05 * f), 700 + f) for f in range(F)]
    check = [0, 1, F // 2, F - 1]
    refs = {f: oracle_frame(ys[f], hd, cfg) for f in check}
    reg = O.cutoff_region(O.Optics(nnum=cfg.nnum, **OPTICS), cfg.height, cfg.width)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=optics(cfg.nnum), flags=L().LFM_PLAN_FRAMES) as plan:
        with pytest.raises(L().LfmError) as e:
            plan.forward(torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda"),
                         torch.zeros((cfg.height, cfg.width), device="cuda"))
        assert e.value.status == L().LFM_EUNSUPPORTED
        yb = dev(np.stack(ys))
        for pol in (L().make_policy(mode="fixed", n_iters=3), L().make_policy(mode="auto", max_iters=25)):
            xb = torch.zeros((F, cfg.nz, cfg.height, cfg.width), device="cuda")
            rb = plan.rl_iterate_batch(yb, xb, pol)
            for f in check:
                ref, its = refs[f]
                got = xb[f].cpu().numpy()
                if pol.mode == L().LFM_MODE_FIXED:
                    es = [O.evaluate_iteration(its[k], reg) for k in range(3)]
                    np.testing.assert_allclose(rb["series"][f], es, rtol=1e-4)
                    assert rb["best_iter"][f] == int(np.argmax(es)) + 1
                    assert rel(got, its[rb["best_iter"][f] - 1]) <= 1e-3
                    continue
                n = min(len(ref.series), len(rb["series"][f]))
                err = max(abs(a - b) / abs(b) for a, b in zip(rb["series"][f][:n], ref.series[:n]))
                assert err <= 1e-4, (f, err)
                k = ref.stop_iter
                margin = min(abs(ref.series[i] - ref.series[i - 1]) / abs(ref.series[i]) for i in range(1, k)) if k > 1 else 1.0
                if margin > 10 * err:
                    assert (rb["stop_iter"][f], rb["best_iter"][f]) == (ref.stop_iter, ref.best_iter), f
                    assert rel(got, ref.volume) <= 1e-3


@pytest.mark.gpu
def test_frames_plan_with_supplied_ht():
    """LFM_PLAN_FRAMES with a supplied transposed PSF (f3): the transposed split copy is built from the Ht matrices, so
    the batched frames equal the single-frame plan with the same Ht (itself oracle-tested, test_supplied_ht) within
    the fp32 / 2xFP16 re-association bound."""
    h, x, r = rand_case(31, 3, 3, 27, 33, 9, 9)
    rng = np.random.default_rng(32)
    ht = rng.uniform(0, 1, h.shape).astype(np.float32)
    F = 8
    ys = [np.ascontiguousarray(rng.uniform(5, 50, (27, 33)).astype(np.float32)) for _ in range(F)]
    pol = L().make_policy(mode="fixed", n_iters=4)
    with L().Plan(h, 3, 27, 33, optics=optics(3), flags=L().LFM_PLAN_FFT_ONLY, psf_t=ht) as p1:
        singles = []
        for f in range(F):
            x1 = torch.zeros((3, 27, 33), device="cuda")
            r1 = p1.rl_iterate(dev(ys[f]), x1, pol)
            singles.append((r1, x1.cpu().numpy()))
    with L().Plan(h, 3, 27, 33, optics=optics(3), flags=L().LFM_PLAN_FRAMES, psf_t=ht) as pf:
        xb = torch.zeros((F, 3, 27, 33), device="cuda")
        rb = pf.rl_iterate_batch(dev(np.stack(ys)), xb, pol)
    for f in range(F):
        r1, x1 = singles[f]
        assert rb["best_iter"][f] == r1["best_iter"]
        np.testing.assert_allclose(rb["series"][f], r1["series"], rtol=1e-5)
        assert rel(xb[f].cpu().numpy(), x1.astype(np.float64)) <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("flags", [4, 2048], ids=["fft", "frames"])
def test_whole_image_75_point_transforms(flags):
    """Whole-image coarse transforms of 75 points (the c3 / c5 size, kernels_fft_fast.cu) at a small geometry: N = 3,
    213 x 213 (71 coarse pixels, kernel 13: alias-free minimum 73 -> 75).  Operators against the oracle (fft plan) and
    batched RL frames against the oracle's iterations (frames plan)."""
    h, x, r = rand_case(75, 2, 3, 213, 213, 13, 13)
    hd = h.astype(np.float64)
    if flags == 4:
        with L().Plan(h, 3, 213, 213, optics=optics(3), flags=4 | L().LFM_PLAN_NO_TILES) as plan:
            assert plan.info()["fft_h"] == 75 and plan.info()["tiles"] == 0
            y_d = torch.zeros((213, 213), device="cuda")
            plan.forward(dev(x), y_d)
            xb_d = torch.zeros((2, 213, 213), device="cuda")
            plan.backward(dev(r), xb_d)
            nrm_d = torch.zeros((2, 213, 213), device="cuda")
            plan.normalizer(nrm_d)
            torch.cuda.synchronize()
        for got, ref in [(y_d, O.forward_project(x.astype(np.float64), hd)),
                         (xb_d, O.backward_project(r.astype(np.float64), hd)),
                         (nrm_d, O.compute_normalizer(hd, 213, 213))]:
            g = got.cpu().numpy()
            assert rel(g, ref) <= 2e-6, rel(g, ref)
            assert np.abs(g - ref).max() <= 1e-5 * np.abs(ref).max()
        return
    rng = np.random.default_rng(76)
    F = 8
    ys = [np.maximum(O.forward_project(rng.uniform(0, 1, (2, 213, 213)), hd), 0.0) + 1.0 for _ in range(F)]
    opt = O.Optics(nnum=3, **OPTICS)
    with L().Plan(h, 3, 213, 213, optics=optics(3), flags=L().LFM_PLAN_FRAMES) as plan:
        assert plan.info()["fft_h"] == 75
        xb = torch.zeros((F, 2, 213, 213), device="cuda")
        rb = plan.rl_iterate_batch(dev(np.stack(ys).astype(np.float32)), xb, L().make_policy(mode="fixed", n_iters=2))
        torch.cuda.synchronize()
    for f in (0, F - 1):
        ref = O.deconvolve(ys[f], hd, opt, O.Policy(mode="fixed", n_iters=2), keep_iterates=True)
        got = xb[f].cpu().numpy()
        assert rel(got, ref.iterates[rb["best_iter"][f] - 1]) <= 1e-4
        np.testing.assert_allclose(rb["series"][f], ref.series, rtol=1e-4)

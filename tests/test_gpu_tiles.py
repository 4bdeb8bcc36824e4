"""GPU parity of the overlap-save tiled frequency path (LFM_PLAN_TILES) against the fp64 oracle
(marked gpu), through the C ABI.  The tiles run their MACs on tcgen05 kind::f16 with the 2xFP16 split of the
direct path (3 products), so the operator bar is the tensor-core one: rel-L2 <= 1e-5, max-abs <=
2e-5 max|ref|; RL as the north star (1e-4 after one iteration, identical stop / best under reading C16)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson  # noqa: E402
from oracle import lfm_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def L():
    from paper_2208_11422_b200 import lfm
    return lfm


def dev(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def rand_case(seed, nz, N, H, W, kh, kw):
    rng = np.random.default_rng(seed)
    h = rng.uniform(0, 1, (nz, N, N, kh, kw)).astype(np.float32)
    h /= h.sum(axis=(3, 4), keepdims=True)
    x = rng.uniform(0, 1, (nz, H, W)).astype(np.float32)
    r = rng.uniform(0.5, 1.5, (H, W)).astype(np.float32)
    return h, x, r


# (nz, N, H, W, kh, kw): 3x3 tiles, ragged last tiles and unequal tap spans, N=5, N=1 (large span), N=7 non-square
TILE_CASES = [
    (3, 3, 99, 99, 9, 9),
    (2, 3, 96, 105, 9, 15),
    (3, 5, 150, 150, 25, 25),
    (2, 1, 64, 80, 9, 9),
    (2, 7, 210, 140, 29, 21),
]


@pytest.mark.parametrize("flags", [4, 0], ids=["fft", "hybrid"])
@pytest.mark.parametrize("case", TILE_CASES, ids=[str(c) for c in TILE_CASES])
def test_tiled_projections_match_oracle(case, flags):
    nz, N, H, W, kh, kw = case
    h, x, r = rand_case(sum(case) + 5, *case)
    hd = h.astype(np.float64)
    with L().Plan(h, N, H, W, optics=L().make_optics(**OPTICS), flags=flags | L().LFM_PLAN_TILES) as plan:
        info = plan.info()
        assert info["tiles"] >= 2 or info["fft_units"] == 0, info   # (hybrid: small kernels may all go direct)
        y_d = torch.zeros((H, W), device="cuda")
        plan.forward(dev(x), y_d)
        xb_d = torch.zeros((nz, H, W), device="cuda")
        plan.backward(dev(r), xb_d)
        nrm_d = torch.zeros((nz, H, W), device="cuda")
        plan.normalizer(nrm_d)
        torch.cuda.synchronize()
    y_ref = O.forward_project(x.astype(np.float64), hd)
    xb_ref = O.backward_project(r.astype(np.float64), hd)
    nrm_ref = O.compute_normalizer(hd, H, W)
    for got, ref in [(y_d, y_ref), (xb_d, xb_ref), (nrm_d, nrm_ref)]:
        g = got.cpu().numpy()
        assert rel(g, ref) <= 1e-5, (rel(g, ref), info)
        assert np.abs(g - ref).max() <= 2e-5 * np.abs(ref).max(), info


@pytest.mark.parametrize("L", [45, 20, 32], ids=["warp-kernels", "register-kernels", "register-wide-tiles"])
def test_tiled_window_sizes(L, monkeypatch):
    """Forced window sizes (LFM_TILE_L, dev): L = 45 runs the warp-per-transform tile kernels (c4's size), L = 20 the
    register-resident ones, L = 32 the register kernels with tiles wider than 16 outputs (the C2R epilogue's one-row-
    per-warp lane mapping); all match the oracle."""
    monkeypatch.setenv("LFM_TILE_L", str(L))
    h, x, r = rand_case(97, 2, 3, 120, 99, 27, 21)
    hd = h.astype(np.float64)
    with L_().Plan(h, 3, 120, 99, flags=L_().LFM_PLAN_TILES | L_().LFM_PLAN_FFT_ONLY) as plan:
        info = plan.info()
        assert info["tiles"] >= 2 and info["fft_h"] == L, info
        if L == 32:
            assert info["tile_T2"] > 16, info
        y_d = torch.zeros((120, 99), device="cuda")
        plan.forward(dev(x), y_d)
        xb_d = torch.zeros((2, 120, 99), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
    assert rel(y_d.cpu().numpy(), O.forward_project(x.astype(np.float64), hd)) <= 1e-5
    assert rel(xb_d.cpu().numpy(), O.backward_project(r.astype(np.float64), hd)) <= 1e-5


def L_():
    return L()


def test_tiled_off_centre_psf():
    """A PSF whose support lies on one side of the kernel centre (coarse taps not straddling 0): the tile windows
    keep the centre in their tap range; forward and backward match the oracle."""
    rng = np.random.default_rng(103)
    h = np.zeros((2, 3, 3, 15, 15), np.float32)
    h[:, :, :, 12:15, 11:15] = rng.uniform(0, 1, (2, 3, 3, 3, 4))   # rows / columns >= 4 right of the centre (7):
    # every coarse tap d >= 1 on both axes
    h /= h.sum(axis=(3, 4), keepdims=True)
    x = rng.uniform(0, 1, (2, 120, 99)).astype(np.float32)
    r = rng.uniform(0.5, 1.5, (120, 99)).astype(np.float32)
    hd = h.astype(np.float64)
    with L().Plan(h, 3, 120, 99, flags=L().LFM_PLAN_TILES | L().LFM_PLAN_FFT_ONLY) as plan:
        assert plan.info()["tiles"] >= 2
        y_d = torch.zeros((120, 99), device="cuda")
        plan.forward(dev(x), y_d)
        xb_d = torch.zeros((2, 120, 99), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
    assert rel(y_d.cpu().numpy(), O.forward_project(x.astype(np.float64), hd)) <= 1e-5
    assert rel(xb_d.cpu().numpy(), O.backward_project(r.astype(np.float64), hd)) <= 1e-5


def test_tiled_signed_inputs():
    """lfm_forward / lfm_backward of sign-changing inputs: the per-tile fp16 scale is bounded by sum |window|, not by
    the (non-negative-source) DC term."""
    h, x, r = rand_case(91, 3, 3, 99, 99, 9, 9)
    rng = np.random.default_rng(92)
    x = (x - 0.5).astype(np.float32)
    r = rng.normal(0, 1, r.shape).astype(np.float32)
    hd = h.astype(np.float64)
    with L().Plan(h, 3, 99, 99, flags=L().LFM_PLAN_TILES | L().LFM_PLAN_FFT_ONLY) as plan:
        y_d = torch.zeros((99, 99), device="cuda")
        plan.forward(dev(x), y_d)
        xb_d = torch.zeros((3, 99, 99), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
    assert rel(y_d.cpu().numpy(), O.forward_project(x.astype(np.float64), hd)) <= 2e-5
    assert rel(xb_d.cpu().numpy(), O.backward_project(r.astype(np.float64), hd)) <= 2e-5


def test_tiled_supplied_ht():
    """f3 on a tiled plan: the transposed split copy is built from the supplied Ht."""
    h, x, r = rand_case(93, 3, 3, 99, 99, 9, 9)
    ht = np.random.default_rng(94).uniform(0, 1, h.shape).astype(np.float32)
    with L().Plan(h, 3, 99, 99, flags=L().LFM_PLAN_TILES | L().LFM_PLAN_FFT_ONLY, psf_t=ht) as plan:
        xb_d = torch.zeros((3, 99, 99), device="cuda")
        plan.backward(dev(r), xb_d)
        y_d = torch.zeros((99, 99), device="cuda")
        plan.forward(dev(x), y_d)
        torch.cuda.synchronize()
    assert rel(xb_d.cpu().numpy(), O.backward_project_ht(r.astype(np.float64), ht.astype(np.float64))) <= 1e-5
    assert rel(y_d.cpu().numpy(), O.forward_project(x.astype(np.float64), h.astype(np.float64))) <= 1e-5


@pytest.mark.parametrize("flags", [4, 0], ids=["fft", "hybrid"])
def test_tiled_c2_operators(flags):
    """BASELINE configs[1] geometry (N=11, 319^2, 21 planes, K=99) on tiles: full-image operator parity."""
    cfg = CONFIGS["c2"]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    x = gen_volume(cfg, 1, np.float32)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, flags=flags | L().LFM_PLAN_TILES) as plan:
        info = plan.info()
        assert info["tiles"] >= 2
        y_d = torch.zeros((cfg.height, cfg.width), device="cuda")
        plan.forward(dev(x), y_d)
        torch.cuda.synchronize()
        y_ref = O.forward_project(x.astype(np.float64), hd)
        r = ((y_ref + 1.0) / (y_ref.mean() + 1.0)).astype(np.float32)
        xb_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
    assert rel(y_d.cpu().numpy(), y_ref) <= 1e-5, info
    assert rel(xb_d.cpu().numpy(), O.backward_project(r.astype(np.float64), hd)) <= 1e-5, info


@pytest.mark.parametrize("name,flags", [("s15", 4), ("s15", 4 | 32), ("c2", 0)], ids=["s15-fft", "s15-fft-graphs", "c2-hybrid"])
def test_tiled_rl_auto_stop(name, flags):
    """Auto-stop RL with a tiled plan (s15: every plane on tiles, eager and graph replay; c2: tiles beside tcgen05
    planes): series within 1e-4, identical stop / best (C16), x_best within 1e-3 of the oracle's."""
    cfg = CONFIGS[name]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    y = poisson(O.forward_project(gen_volume(cfg, 1), hd), 77)
    pol_o = O.Policy(mode="auto", max_iters=25)
    ref = O.deconvolve(y, hd, O.Optics(nnum=cfg.nnum, **OPTICS), pol_o)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st), L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L().make_optics(**OPTICS),
                                         flags=flags | L().LFM_PLAN_TILES, stream=st) as plan:
        assert plan.info()["tiles"] >= 2
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="auto", max_iters=25), stream=st)
        st.synchronize()
    n = min(len(res["series"]), len(ref.series))
    err = max(abs(a - b) / abs(b) for a, b in zip(res["series"][:n], ref.series[:n]))
    assert err <= 1e-4, err
    k = ref.stop_iter
    margin = min(abs(ref.series[i] - ref.series[i - 1]) / abs(ref.series[i]) for i in range(1, k)) if k > 1 else 1.0
    if margin > 10 * err:
        assert (res["stop_iter"], res["best_iter"]) == (ref.stop_iter, ref.best_iter)
    assert rel(x_d.cpu().numpy(), ref.volume) <= 1e-3


def test_tiled_plan_batches_frame_by_frame():
    """lfm_rl_iterate_batch on a tiled plan runs the frames one after the other through the single-frame loop: every
    frame identical to its own lfm_rl_iterate call."""
    cfg = CONFIGS["s15"]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    F = 4
    ys = np.stack([poisson(O.forward_project(gen_volume(cfg, 1 + f), hd), 300 + f) for f in range(F)]).astype(np.float32)
    pol = L().make_policy(mode="auto", max_iters=12)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L().make_optics(**OPTICS),
                  flags=L().LFM_PLAN_TILES | L().LFM_PLAN_FFT_ONLY) as plan:
        assert plan.info()["tiles"] >= 2
        xb = torch.zeros((F, cfg.nz, cfg.height, cfg.width), device="cuda")
        rb = plan.rl_iterate_batch(dev(ys), xb, pol)
        for f in range(F):
            x1 = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
            r1 = plan.rl_iterate(dev(ys[f]), x1, pol)
            torch.cuda.synchronize()
            assert (rb["best_iter"][f], rb["stop_iter"][f]) == (r1["best_iter"], r1["stop_iter"])
            assert np.array_equal(np.asarray(rb["series"][f]), np.asarray(r1["series"]))
            assert torch.equal(xb[f], x1)


def test_tiled_virtual_shards():
    """Depth / phase sharding on tiled plans: NO_COMM plans of rank r / world own contiguous unit ranges (a
    rank may hold part of a plane: its tile groups hold only its units); partial forwards sum to the oracle's forward,
    the backwards cover disjoint units."""
    h, x, r = rand_case(98, 3, 3, 99, 99, 9, 9)
    h[2] = 0.0
    h[2, :, :, 3:6, 3:6] = np.random.default_rng(99).uniform(0, 1, (3, 3, 3, 3))   # a narrower plane: 2 tile groups
    h /= h.sum(axis=(3, 4), keepdims=True)
    hd = h.astype(np.float64)
    y_ref = O.forward_project(x.astype(np.float64), hd)
    xb_ref = O.backward_project(r.astype(np.float64), hd)
    for world in (2, 3):
        tot = np.zeros_like(y_ref)
        cover = np.zeros((3, 99, 99))
        xb_acc = np.zeros_like(xb_ref)
        for rank in range(world):
            with L().Plan(h, 3, 99, 99, rank=rank, world=world,
                          flags=L().LFM_PLAN_NO_COMM | L().LFM_PLAN_TILES | L().LFM_PLAN_FFT_ONLY) as plan:
                assert plan.info()["tiles"] >= 2
                y_d = torch.zeros((99, 99), device="cuda")
                plan.forward(dev(x), y_d)
                xb_d = torch.full((3, 99, 99), -1.0, device="cuda")
                plan.backward(dev(r), xb_d)
                torch.cuda.synchronize()
                tot += y_d.cpu().numpy()
                xb = xb_d.cpu().numpy()
                own = xb != -1.0
                cover += own
                xb_acc[own] = xb[own]
        assert rel(tot, y_ref) <= 1e-5
        assert (cover == 1).all()
        assert rel(xb_acc, xb_ref) <= 1e-5


def test_tiled_isra_and_groups():
    """ISRA (f3) on a tiled plan whose planes need two window geometries (tile groups): 1 and 5 iterations against
    the oracle's ISRA."""
    h, _, _ = rand_case(100, 3, 3, 99, 99, 9, 9)
    h[0] = 0.0
    h[0, :, :, 3:6, 3:6] = np.random.default_rng(101).uniform(0, 1, (3, 3, 3, 3))
    h /= h.sum(axis=(3, 4), keepdims=True)
    hd = h.astype(np.float64)
    y = O.forward_project(np.random.default_rng(102).uniform(0, 1, (3, 99, 99)), hd) + 0.5
    opt = O.Optics(nnum=3, **OPTICS)
    with L().Plan(h, 3, 99, 99, optics=L().make_optics(**OPTICS),
                  flags=L().LFM_PLAN_TILES | L().LFM_PLAN_FFT_ONLY) as plan:
        info = plan.info()
        assert info["tile_groups"] == 2, info
        for n, tol in [(1, 1e-4), (5, 1e-3)]:
            ref = O.deconvolve(y, hd, opt, O.Policy(mode="fixed", n_iters=n), update="isra", keep_iterates=True)
            x_d = torch.zeros((3, 99, 99), device="cuda")
            res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="fixed", n_iters=n, update="isra"))
            torch.cuda.synchronize()
            assert res["best_iter"] == ref.best_iter
            assert rel(x_d.cpu().numpy(), ref.iterates[res["best_iter"] - 1]) <= tol
            np.testing.assert_allclose(res["series"], ref.series, rtol=1e-4)

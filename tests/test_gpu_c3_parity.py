"""GPU parity at the benchmarked configuration (marked gpu): c3 (BASELINE.json configs[2]: Nnum=15, 1005x1005,
51 planes) in the launch configuration bench.py times -- the default hybrid plan, tcgen05 planes and frequency-path
planes side by side on SM partitions -- against the fp64 oracle, through the C ABI.

* auto-stop RL vs tests/golden/c3_auto.json (written by scripts/make_golden_c3.py from oracle/ only): identical
  stop_iter / best_iter (P:99 stop rule, reading C15; guarded by C16's margin rule), E_k within 1e-4 relative,
  x_best's per-plane and per-(z,a)-unit sums and ~14k sampled voxels;
* 30 RL iterations on the c3 geometry with 13 planes (a bank that mixes tcgen05 and frequency-path planes) vs
  tests/golden/c3g13_30.json: the north-star gates rel-L2 <= 1e-4 after 1 iteration and <= 1e-3 after 30;
* full-image forward and full-volume backward element-wise against the oracle run live (~40 s each on 16 cores).
"""
import dataclasses
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, lf_like  # noqa: E402
from oracle import lfm_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def L():
    from paper_2208_11422_b200 import lfm
    return lfm


def dev(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def load_golden(name, yname):
    with open(os.path.join(GOLD, name)) as f:
        g = json.load(f)
    y = np.load(os.path.join(GOLD, yname))["y"].astype(np.float64)
    assert hashlib.sha256(y.tobytes()).hexdigest() == g["y_sha256"], "stored y does not match its recorded digest"
    return g, y


def check_volume(x, rec, z, p, q, N, tol_samples, tol_units):
    """x [nz][H][W] (GPU result) against a golden record: per-plane sums, per-(z,a) unit sums, sampled voxels."""
    nz, H, W = x.shape
    xd = x.astype(np.float64)
    planes = xd.reshape(nz, -1).sum(axis=1)
    assert rel(planes, rec["plane_sums"]) <= tol_units, rel(planes, rec["plane_sums"])
    np.testing.assert_allclose(planes, rec["plane_sums"], rtol=10 * tol_units)
    units = xd.reshape(nz, H // N, N, W // N, N).sum(axis=(1, 3)).reshape(nz, N * N)
    ref_units = np.asarray(rec["unit_sums"])
    assert rel(units, ref_units) <= tol_units, rel(units, ref_units)
    np.testing.assert_allclose(units, ref_units, rtol=10 * tol_units)
    got = x[z, p, q]
    assert rel(got, rec["x"]) <= tol_samples, rel(got, rec["x"])


def test_c3_auto_stop_matches_golden():
    """The benchmarked c3 plan (flags 0: hybrid tcgen05 + frequency path on SM partitions), auto-stop from the
    uniform start: stop / best iterations identical to the oracle's, E_k within 1e-4 relative, x_best within 1e-3
    (samples) and 1e-4 (per-plane and per-unit sums)."""
    g, y = load_golden("c3_auto.json", "c3_y.npz")
    cfg = CONFIGS["c3"]
    h = gen_psf(cfg, np.float32)
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L().make_optics(**OPTICS)) as plan:
        info = plan.info()
        assert info["tc_planes"] > 0 and info["fft_units"] > 0
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        res = plan.rl_iterate(dev(y), x_d, L().make_policy(mode="auto", max_iters=50))
        torch.cuda.synchronize()
        print(f"c3 plan: {info['tc_planes']} tcgen05 planes, {info['fft_units']} frequency-path units, "
              f"partitions {info['partition_sms']}; gpu stop {res['stop_iter']} best {res['best_iter']}, "
              f"oracle stop {g['stop_iter']} best {g['best_iter']}")
    s_o = g["series"]
    n = min(len(res["series"]), len(s_o))
    err = max(abs(a - b) / abs(b) for a, b in zip(res["series"][:n], s_o[:n]))
    assert err <= 1e-4, err
    margin = g["decision_margin"]
    assert margin > 10 * err, f"tie-ambiguous at c3 (C16): margin {margin:.2e} vs entropy error {err:.2e}"
    assert (res["stop_iter"], res["best_iter"]) == (g["stop_iter"], g["best_iter"])
    sm = g["samples"]
    z, p, q = (np.asarray(sm[k]) for k in ("z", "p", "q"))
    rec = {"plane_sums": g["plane_sums"], "unit_sums": g["unit_sums"], "x": sm["x"]}
    check_volume(x_d.cpu().numpy(), rec, z, p, q, cfg.nnum, 1e-3, 1e-4)


def c3g13():
    return dataclasses.replace(CONFIGS["c3"], name="c3g13", nz=13, n_objects=100, background=0.05 * 9 / 13)


@pytest.mark.parametrize("flags", [0, 32], ids=["eager", "graphs"])
def test_c3g13_1_and_30_iterations(flags, monkeypatch):
    """North-star gates on the c3 geometry (1005x1005, Nnum=15, c3 PSF recipe) with 13 planes: the default plan holds
    tcgen05 planes and frequency-path planes, run side by side on forced SM partitions.  x_1 within 1e-4, the argmax
    iterate of 30 within 1e-3, the series within 1e-4; x_30 (chained lfm_rl_step calls) within 1e-3."""
    g, y = load_golden("c3g13_30.json", "c3g13_y.npz")
    cfg = c3g13()
    h = gen_psf(cfg, np.float32)
    monkeypatch.setenv("LFM_TC_SMS_F", "96")
    monkeypatch.setenv("LFM_TC_SMS_B", "104")
    sm = g["samples"]
    z, p, q = (np.asarray(sm[k]) for k in ("z", "p", "q"))
    st = torch.cuda.Stream()   # graph capture needs a non-default stream
    with torch.cuda.stream(st), \
            L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L().make_optics(**OPTICS), flags=flags, stream=st) as plan:
        info = plan.info()
        assert info["tc_planes"] > 0 and info["fft_units"] > 0, info
        assert info["partition_sms"][0][0] == 96 and info["partition_sms"][1][0] == 104
        y_d = dev(y)
        x_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        r1 = plan.rl_iterate(y_d, x_d, L().make_policy(mode="fixed", n_iters=1), stream=st)
        st.synchronize()
        check_volume(x_d.cpu().numpy(), g["x1"], z, p, q, cfg.nnum, 1e-4, 1e-4)
        assert abs(r1["series"][0] - g["series"][0]) <= 1e-4 * abs(g["series"][0])
        r30 = plan.rl_iterate(y_d, x_d, L().make_policy(mode="fixed", n_iters=30), stream=st)
        st.synchronize()
        np.testing.assert_allclose(r30["series"], g["series"], rtol=1e-4)
        assert r30["best_iter"] == g["best_iter"]
        check_volume(x_d.cpu().numpy(), g["x_best"], z, p, q, cfg.nnum, 1e-3, 1e-4)
        if flags == 0:   # x_30 itself through lfm_rl_step (the one-step ABI call), from the uniform start
            c0 = float(y.sum()) / plan_forward_total(plan, cfg)
            xa = torch.full((cfg.nz, cfg.height, cfg.width), c0, device="cuda")
            xb = torch.zeros_like(xa)
            for _ in range(30):
                plan.rl_step(y_d, xa, xb, entropy=False)
                xa, xb = xb, xa
            torch.cuda.synchronize()
            check_volume(xa.cpu().numpy(), g["x30"], z, p, q, cfg.nnum, 1e-3, 1e-4)


def plan_forward_total(plan, cfg):
    """sum H 1_vol through the product's forward projection (reading C2's c0 denominator)."""
    ones = torch.ones((cfg.nz, cfg.height, cfg.width), device="cuda")
    yo = torch.zeros((cfg.height, cfg.width), device="cuda")
    plan.forward(ones, yo)
    torch.cuda.synchronize()
    return float(yo.double().sum())


def test_c3_full_image_forward_backward():
    """Element-wise full-size operator parity on the benchmarked c3 plan: the whole 1005x1005 forward image and the
    whole 51x1005x1005 backward volume against the oracle (fp64 direct convolution, run live).  Tolerances as the
    tcgen05 operator bar: rel-L2 <= 1e-5, max-abs <= 2e-5 max|ref|; per plane rel-L2 <= 2e-5."""
    cfg = CONFIGS["c3"]
    h = gen_psf(cfg, np.float32)
    hd = h.astype(np.float64)
    x = gen_volume(cfg, 2, np.float32)
    r = (lf_like(cfg, 3) + 1.0).astype(np.float32)
    r /= np.float32(r.mean())
    with L().Plan(h, cfg.nnum, cfg.height, cfg.width, optics=L().make_optics(**OPTICS)) as plan:
        info = plan.info()
        y_d = torch.zeros((cfg.height, cfg.width), device="cuda")
        plan.forward(dev(x), y_d)
        xb_d = torch.zeros((cfg.nz, cfg.height, cfg.width), device="cuda")
        plan.backward(dev(r), xb_d)
        torch.cuda.synchronize()
        yg, xbg = y_d.cpu().numpy(), xb_d.cpu().numpy()
    del h
    y_ref = O.forward_project(x.astype(np.float64), hd)
    assert rel(yg, y_ref) <= 1e-5, rel(yg, y_ref)
    assert np.abs(yg - y_ref).max() <= 2e-5 * np.abs(y_ref).max()
    xb_ref = O.backward_project(r.astype(np.float64), hd)
    assert rel(xbg, xb_ref) <= 1e-5, rel(xbg, xb_ref)
    assert np.abs(xbg - xb_ref).max() <= 2e-5 * np.abs(xb_ref).max()
    per_plane = [rel(xbg[k], xb_ref[k]) for k in range(cfg.nz)]
    assert max(per_plane) <= 2e-5, (int(np.argmax(per_plane)), max(per_plane), info["tc_planes"])

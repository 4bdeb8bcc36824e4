"""Pins of the oracle's metric and stop rule (not gpu): worked examples (tests/golden, cited), a
library routine (scipy.fft.dctn), closed forms and invariants (§2.2)."""
import itertools
import math

import numpy as np
import pytest
import scipy.fft

from conftest import golden
from oracle import lfm_oracle as O


def _kv(tokens):
    return {k: float(v) for k, v in (t.split("=") for t in tokens)}


def test_optics_worked_examples():
    """Eqs. (7), (11), (9)-(10), (6): worked values (golden/optics_examples.txt)."""
    for row in golden("optics_examples.txt"):
        kind, rest = row[0], row[1:]
        if kind == "sample_pitch":
            a = _kv(rest[:3])
            assert O.sample_pitch(a["d_ml"], a["q"], int(a["nnum"])) == pytest.approx(float(rest[3]), rel=1e-15)
        elif kind == "resolution":
            a = _kv(rest[:3])
            assert O.resolution_limit(a["lam"], a["na"], int(a["nnum"])) == pytest.approx(float(rest[3]), rel=1e-12)
        else:
            a = _kv(rest[:7])
            e = _kv(rest[7:])
            reg = O.cutoff_region(O.Optics(a["lam"], a["na"], a["d_ml"], a["q"], int(a["nnum"])), int(a["m"]), int(a["n"]))
            assert (reg.x_s, reg.y_s, reg.g_s) == (int(e["x_s"]), int(e["y_s"]), e["g_s"])


def test_region_properties():
    """brute-force member count, downward closure, (0,0) member, |T| ~ G_S within X_S+Y_S;
    increasing d_psf never grows the region; homogeneity of Eqs. 7 and 11."""
    for lam in (0.4, 0.52, 0.7):
        for na in (0.3, 0.5, 0.8, 1.0):
            for (M, N) in [(64, 64), (45, 60), (300, 200)]:
                reg = O.cutoff_region(O.Optics(lam, na, 150.0, 20.0, 15), M, N)
                mem = set(reg.members)
                brute = {(u, v) for u in range(M) for v in range(N)
                         if u < reg.y_s and v < reg.x_s and u * reg.x_s + v * reg.y_s < reg.x_s * reg.y_s}
                assert mem == brute and (0, 0) in mem
                assert abs(len(mem) - reg.g_s) <= reg.x_s + reg.y_s
                for (u, v) in mem:
                    assert all((uu, vv) in mem for uu in range(u + 1) for vv in range(v + 1))
                bigger = O.cutoff_region(O.Optics(lam * 1.3, na, 150.0, 20.0, 15), M, N)
                assert bigger.x_s <= reg.x_s and bigger.y_s <= reg.y_s
    assert O.sample_pitch(300.0, 20, 15) == 2 * O.sample_pitch(150.0, 20, 15)
    assert O.resolution_limit(1.04, 0.5, 15) == 2 * O.resolution_limit(0.52, 0.5, 15)
    with pytest.raises(ValueError):
        O.Optics(0.52, 0.5, 150, 20, 14).validate()      # even Nnum
    with pytest.raises(ValueError):
        O.Optics(0.52, 1.7, 150, 20, 15).validate()      # NA > 1.6


def test_dct_worked_examples():
    """Eqs. (1)-(4): golden/dct_examples.txt."""
    for row in golden("dct_examples.txt"):
        M, N = int(row[0]), int(row[1])
        bar = [i for i, t in enumerate(row) if t == "|"]
        img = np.array([float(t) for t in row[bar[0] + 1:bar[1]]]).reshape(M, N)
        exp = np.array([float(t) for t in row[bar[1] + 1:]]).reshape(M, N)
        np.testing.assert_allclose(O.dct2(img), exp, atol=1e-15)


def test_dct_matches_scipy_and_parseval():
    """Library routine: scipy.fft.dctn(type=2, norm='ortho') is the orthonormal DCT-II of Eqs. (1)-(4);
    Parseval within 1e-9; idct2 inverts; the corner variant is the same matrix."""
    rng = np.random.default_rng(0)
    for (M, N) in [(1, 1), (2, 3), (17, 23), (64, 64), (128, 96), (33, 33)]:
        f = rng.normal(size=(M, N))
        F = O.dct2(f)
        np.testing.assert_allclose(F, scipy.fft.dctn(f, type=2, norm="ortho"), rtol=1e-10, atol=1e-12)
        assert abs(np.linalg.norm(F) - np.linalg.norm(f)) <= 1e-9 * np.linalg.norm(f)
        np.testing.assert_allclose(O.idct2(F), f, atol=1e-9)
        r, c = max(1, M // 3), max(1, N // 4)
        np.testing.assert_allclose(O.dct2(f, rows=r, cols=c), F[:r, :c], rtol=1e-13, atol=1e-13)
    # single DC coefficient sqrt(MN) v -> constant image v
    F = np.zeros((5, 7))
    F[0, 0] = math.sqrt(35) * 2.5
    np.testing.assert_allclose(O.idct2(F), 2.5, rtol=1e-14)


def test_shannon_worked_examples():
    """Eq. (5): golden/entropy_examples.txt."""
    for row in golden("entropy_examples.txt"):
        exp = float(row[0])
        p = [float(t) for t in row[2:]]
        assert O.shannon_entropy(p) == pytest.approx(exp, abs=1e-15)
    with pytest.raises(ValueError):
        O.shannon_entropy([0.5, -0.1])


def _optics15():
    return O.Optics(0.52, 0.5, 150.0, 20.0, 15)


def test_dct_entropy_closed_forms():
    """Eq. (12) closed forms: constant image -> 0; a single DCT basis image inside T -> 0;
    two equal-amplitude basis images inside T -> w = 1/sqrt2 each, E = (2/(X_S Y_S)) * 2 * (0.5/sqrt2);
    all-zero image -> 0; scale invariance."""
    M = N = 225
    reg = O.cutoff_region(_optics15(), M, N)       # X_S = Y_S = 6
    assert (reg.x_s, reg.y_s) == (6, 6)
    assert O.dct_entropy(np.full((M, N), 3.7), reg) == pytest.approx(0.0, abs=1e-12)
    assert O.dct_entropy(np.zeros((M, N)), reg) == 0.0
    Bm, Bn = O.dct_basis(M), O.dct_basis(N)
    one = np.outer(Bm[2], Bn[1])                   # F = delta at (2,1), inside T (2*6+1*6 < 36)
    assert O.dct_entropy(one, reg) == pytest.approx(0.0, abs=1e-12)
    two = 4.0 * (np.outer(Bm[2], Bn[1]) + np.outer(Bm[0], Bn[3]))
    expect = 2.0 / 36 * 2 * (0.5 / math.sqrt(2))
    assert O.dct_entropy(two, reg) == pytest.approx(expect, rel=1e-12)
    outside = 4.0 * (np.outer(Bm[2], Bn[1]) + np.outer(Bm[5], Bn[5]))   # (5,5) not in T
    assert O.dct_entropy(outside, reg) == pytest.approx(2.0 / 36 * (0.5 / math.sqrt(2)), rel=1e-12)
    rng = np.random.default_rng(1)
    f = rng.uniform(0, 1, (M, N))
    e = O.dct_entropy(f, reg)
    assert e > 0
    for a in (2.0, 10.0, 1000.0):
        assert O.dct_entropy(a * f, reg) == pytest.approx(e, rel=1e-12)


def test_dct_entropy_bruteforce():
    """S:150 / S:592: 50 random 16x16 images with random regions vs enumeration of the triangle using
    scipy's DCT (independent transform) -- 1e-12."""
    rng = np.random.default_rng(2)
    for k in range(50):
        f = rng.uniform(0, 1, (16, 16))
        lam = rng.uniform(0.1, 0.3)
        reg = O.cutoff_region(O.Optics(lam, 0.9, 150.0, 20.0, 3), 16, 16)
        F = scipy.fft.dctn(f, norm="ortho")
        L = np.sqrt(np.sum(F * F))
        tot = 0.0
        for u, v in itertools.product(range(16), range(16)):
            if u * reg.x_s + v * reg.y_s < reg.x_s * reg.y_s:
                w = abs(F[u, v]) / L
                tot += -w * math.log2(w) if w > 0 else 0.0
        assert O.dct_entropy(f, reg) == pytest.approx(2.0 / (reg.x_s * reg.y_s) * tot, rel=1e-12, abs=1e-14)


def test_rectangle_region_contains_triangle():
    reg_t = O.cutoff_region(_optics15(), 225, 225, "triangle")
    reg_r = O.cutoff_region(_optics15(), 225, 225, "rectangle")
    assert set(reg_t.members) < set(reg_r.members) and len(reg_r.members) == 36


def test_max_projection():
    """per-pixel max over z."""
    v = np.array([1.0, 5.0, 3.0]).reshape(3, 1, 1)
    assert O.max_project_z(v)[0, 0] == 5.0
    rng = np.random.default_rng(3)
    vol = rng.uniform(0, 1, (3, 8, 8))
    ref = np.array([[max(vol[z, i, j] for z in range(3)) for j in range(8)] for i in range(8)])
    assert np.array_equal(O.max_project_z(vol), ref)


def test_stop_rule_worked_examples():
    """P:99 + Fig. 2d, reading C15: golden/stop_examples.txt (first row = S:290)."""
    for row in golden("stop_examples.txt"):
        bar = [i for i, t in enumerate(row) if t == "|"]
        mode, a, mn, pat = row[0], int(row[1]), int(row[2]), int(row[3])
        series = [float(t) for t in row[bar[0] + 1:bar[1]]]
        stop_exp, best_exp = int(row[bar[1] + 1]), int(row[bar[1] + 2])
        pol = O.Policy(mode=mode, n_iters=a, max_iters=max(a, 1), min_iters=mn, patience=pat) if mode == "fixed" \
            else O.Policy(mode=mode, max_iters=a, min_iters=mn, patience=pat)
        rule = O.StopRule(pol)
        for e in series:
            _, stop = rule.update(e)
            if stop:
                break
        assert (len(rule.series), rule.best_iter) == (stop_exp, best_exp), row
    with pytest.raises(ValueError):
        O.StopRule(O.Policy(min_iters=5, max_iters=3))
    with pytest.raises(ValueError):
        O.StopRule(O.Policy(patience=0))

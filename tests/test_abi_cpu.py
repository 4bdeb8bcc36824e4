"""Host-only checks of the C-ABI library (not gpu): it loads, exports every symbol include/lfm.h
declares, and its pure-host entry points (policy defaults, memory estimate, errors) behave."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lfm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lfm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2208_11422_b200 import lfm as L
    lib = ctypes.CDLL(L.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(L.EXPORTED) == syms


def test_policy_default_and_version():
    from paper_2208_11422_b200 import lfm as L
    p = L.lfm_policy_default()
    assert (p.mode, p.max_iters, p.min_iters, p.patience, p.region, p.init_from_x, p.update) == (1, 50, 2, 1, 0, 0, 0)
    assert abs(p.eps - 1e-6) < 1e-12
    assert "sm_100a" in L.lfm_version()


def test_plan_estimate_and_budget():
    """P:49 memory estimate: c3 on one GPU needs ~59 GB of transfer matrices; c4 does not
    fit a 180 GB budget on one GPU and names the transfer matrices as the limiting term."""
    from paper_2208_11422_b200 import lfm as L
    b, term = L.lfm_plan_estimate(15, 51, 165, 165, 1005, 1005)
    assert 58e9 < b < 62e9 and term.startswith("transfer matrices")
    with pytest.raises(L.LfmError) as ei:
        L.lfm_plan_estimate(15, 101, 225, 225, 2025, 2025, world=1, budget_bytes=180 * 10 ** 9)
    assert ei.value.status == L.LFM_ENOMEM and "transfer matrices" in str(ei.value)
    b8, _ = L.lfm_plan_estimate(15, 101, 225, 225, 2025, 2025, world=8)
    assert b8 < 70e9
    bd, termd = L.lfm_plan_estimate(3, 3, 9, 9, 33, 33, flags=L.LFM_PLAN_DIRECT)
    assert bd < 10 ** 7


def test_plan_estimate_rejects_bad_dims():
    from paper_2208_11422_b200 import lfm as L
    for args, st in [((15, 51, 165, 165, 1000, 1005), L.LFM_EDIM),   # H % N != 0
                     ((15, 51, 164, 165, 1005, 1005), L.LFM_EDIM),   # even kernel
                     ((14, 51, 165, 165, 1008, 1008), L.LFM_EDIM)]:  # even N
        with pytest.raises(L.LfmError) as ei:
            L.lfm_plan_estimate(*args)
        assert ei.value.status == st


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle or numpy-based projections (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2208_11422_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith(".py"):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in src.replace("no oracle", ""), f


def test_host_buffer_checks():
    """lfm_deconvolve_host takes raw host pointers: the binding rejects wrong dtype, shape or layout before the call
    (the library would read H*W and write nz*H*W float32 values)."""
    import numpy as np
    from paper_2208_11422_b200 import lfm as L
    L._check_host(np.zeros((9, 9), np.float32), (9, 9), "y")
    with pytest.raises(TypeError):
        L._check_host(np.zeros((9, 9), np.float64), (9, 9), "y")
    with pytest.raises(ValueError):
        L._check_host(np.zeros((2, 9, 8), np.float32), (2, 9, 9), "x")
    with pytest.raises(TypeError):
        L._check_host(np.zeros((9, 18), np.float32)[:, ::2], (9, 9), "y")

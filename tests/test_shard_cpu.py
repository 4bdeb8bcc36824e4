"""Cost-balanced sharding (include/lfm.h lfm_shard_units_balanced): host-only, no GPU.

Invariants checked on the c2 / s15 PSF banks for world 2..5:
  * the ranges are contiguous, ordered and cover every unit exactly once;
  * the per-rank cost estimates add up to the unsharded estimate -- a tensor-core plane (whose cost does not shrink
    with the owned fraction) is therefore never split between ranks;
  * the slowest rank is no slower than under the even split, and strictly faster where the per-plane costs differ.
"""
import numpy as np
import pytest

from lfm_inputs import CONFIGS, gen_psf


def L():
    from paper_2208_11422_b200 import lfm
    return lfm


@pytest.mark.parametrize("name", ["c2", "s15"])
def test_balanced_partition(name):
    lib = L()
    cfg = CONFIGS[name]
    h = gen_psf(cfg, np.float32)
    N2 = cfg.nnum ** 2
    _, _, total = lib.lfm_shard_units_balanced(h, cfg.nnum, cfg.height, cfg.width, 1, 0)
    assert total > 0
    for world in (2, 3, 4, 5):
        bal = [lib.lfm_shard_units_balanced(h, cfg.nnum, cfg.height, cfg.width, world, r) for r in range(world)]
        even = [lib.lfm_shard_units_balanced(h, cfg.nnum, cfg.height, cfg.width, world, r, lib.LFM_PLAN_EVEN_SHARDS)
                for r in range(world)]
        assert bal[0][0] == 0 and bal[-1][1] == cfg.nz * N2
        for r in range(world - 1):
            assert bal[r][1] == bal[r + 1][0] and bal[r][0] <= bal[r][1]
        assert [(b, e) for b, e, _ in even] == [lib.lfm_shard_units(cfg.nz, cfg.nnum, world, r) for r in range(world)]
        assert abs(sum(t for _, _, t in bal) - total) <= 1e-9 * total
        assert max(t for _, _, t in bal) <= max(t for _, _, t in even) * (1 + 1e-12)


def test_balanced_beats_even_on_mixed_costs():
    """Half the planes narrow (cheap on the tensor cores), half wide (frequency path): the even split puts all the
    expensive planes on one rank, the balanced split does not."""
    lib = L()
    N, H, W, K, nz = 11, 319, 319, 143, 8
    rng = np.random.default_rng(3)
    h = np.zeros((nz, N, N, K, K), np.float32)
    c = K // 2
    h[: nz // 2, :, :, c - 5:c + 6, c - 5:c + 6] = rng.uniform(0, 1, (nz // 2, N, N, 11, 11))
    h[nz // 2:] = rng.uniform(0, 1, (nz // 2, N, N, K, K))
    h /= h.sum(axis=(3, 4), keepdims=True)
    bal = [lib.lfm_shard_units_balanced(h, N, H, W, 2, r)[2] for r in range(2)]
    even = [lib.lfm_shard_units_balanced(h, N, H, W, 2, r, lib.LFM_PLAN_EVEN_SHARDS)[2] for r in range(2)]
    assert max(bal) < 0.9 * max(even)

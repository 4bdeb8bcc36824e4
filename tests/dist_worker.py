"""World-size-N CPU (gloo) rehearsal of the sharded RL iteration the GPU path runs over NCCL
(DESIGN.md §7): each rank owns the units the product's partition gives it (cost-balanced, as lfm_plan_create
uses by default, or the even split with LFM_TEST_EVEN_SHARDS=1), computes its partial forward
projection, C1 = allreduce(sum) of yhat, a local backward projection + update of its own units,
C2 = allreduce(max) of its partial z max-projection, the metric on the reduced projection, and a
final gather.  The arithmetic is the oracle's (this is test infrastructure); the partition and the
unique-id exchange are the product's.  Every rank checks the result against the unsharded oracle."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from lfm_inputs import CONFIGS, OPTICS, gen_psf, gen_volume, poisson  # noqa: E402
from oracle import lfm_oracle as O  # noqa: E402
from paper_2208_11422_b200 import lfm as L  # noqa: E402


def allreduce(a, op):
    t = torch.from_numpy(np.ascontiguousarray(a))
    dist.all_reduce(t, op=op)
    return t.numpy()


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    # NCCL unique id produced by the library on rank 0 and broadcast by the caller (lfm.h, lfm_dist)
    obj = [L.lfm_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ids = [None] * world
    dist.all_gather_object(ids, obj[0])
    assert len(obj[0]) == 128 and all(i == ids[0] for i in ids)

    cfg = CONFIGS["tiny"]
    h = gen_psf(cfg, np.float64)
    y = poisson(O.forward_project(gen_volume(cfg, 1), h), 101)
    nz, N, H, W = cfg.nz, cfg.nnum, cfg.height, cfg.width
    if os.environ.get("LFM_TEST_EVEN_SHARDS") == "1":
        u0, u1 = L.lfm_shard_units(nz, N, world, rank)
    else:
        u0, u1, _ = L.lfm_shard_units_balanced(h.astype(np.float32), N, H, W, world, rank)
    zz, pp, qq = np.meshgrid(np.arange(nz), np.arange(H), np.arange(W), indexing="ij")
    unit = (zz * N + pp % N) * N + qq % N
    own = (unit >= u0) & (unit < u1)
    cover = allreduce(own.astype(np.int32), dist.ReduceOp.SUM)
    assert (cover == 1).all(), "shards must partition the units"

    reg = O.cutoff_region(O.Optics(nnum=N, **OPTICS), H, W)
    norm = O.compute_normalizer(h, H, W, units=(u0, u1))
    c0 = y.sum() / allreduce(np.array([norm.sum()]), dist.ReduceOp.SUM)[0]   # sum H1 = sum H^T 1
    x = np.where(own, c0, 0.0)
    series = []
    for k in range(4):
        yhat = allreduce(O.forward_project(x, h, units=(u0, u1)), dist.ReduceOp.SUM)          # C1
        bp = O.backward_project(O.ratio_image(y, yhat), h, units=(u0, u1))
        x = np.where(own, x * bp / np.maximum(norm, O.EPS), 0.0)
        m = allreduce(np.where(own, x, 0.0).max(axis=0), dist.ReduceOp.MAX)                  # C2
        series.append(O.dct_entropy(m, reg))
    xfull = allreduce(x, dist.ReduceOp.SUM)                                                  # gather

    ref = O.deconvolve(y, h, O.Optics(nnum=N, **OPTICS), O.Policy(mode="fixed", n_iters=4), keep_iterates=True)
    np.testing.assert_allclose(xfull, ref.iterates[-1], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(series, ref.series, rtol=1e-12)
    print(f"rank {rank}/{world} units [{u0},{u1}) ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

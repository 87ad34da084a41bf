"""Multi-rank sharding logic on CPU: world_size 2 over gloo, oracle executor.

The same ShardedIteration that drives the GPUs over NCCL (bench.py under
torchrun) partitions rows/frames and composes the all-reduces/all-gathers;
here each rank runs the CPU oracle on its shard and the assembled result is
compared with the unsharded oracle iteration.
"""

from __future__ import annotations

import os
import socket
from dataclasses import dataclass

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pxst_oracle as orc
from paper_2003_12726_b200.sharding import ShardedIteration, partition_frames, partition_rows


@dataclass
class Cfg:
    half_ss: int = 2
    half_fs: int = 2
    subpixel_grid: float | None = None
    refine: bool = True
    update_translations: bool = True
    t_half_ss: int = 1
    t_half_fs: int = 1
    t_subpixel_grid: float | None = None
    sigma: float = 0.0
    integrate: bool = False


def test_partition_rows_balanced():
    work = np.array([10, 0, 0, 10, 10, 10, 5, 5])
    bands = partition_rows(work, 3, 2)
    assert bands[0][0] == 3 and bands[-1][1] == 11
    assert all(a <= b for a, b in bands)
    sums = [work[a - 3:b - 3].sum() for a, b in bands]
    assert abs(sums[0] - sums[1]) <= 10
    assert partition_frames(7, 3) == [(0, 2), (2, 5), (5, 7)]
    assert partition_rows(np.ones(3, int), 0, 5)[-1] == (3, 3)   # more ranks than rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, cfg):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from scan_helpers import OracleExecutor, tiny_scan
        sc, w, m, u, t = tiny_scan(seed=21, n=7, ss=20, fs=24)
        good = np.ones(7, bool)
        good[3] = False
        ex = OracleExecutor(sc.frames, good, w.w, m.mask)
        it = ShardedIteration(ex, rank, world)
        u_n, di_n, dj_n = it.iteration(torch.as_tensor(u.u), torch.as_tensor(t.di),
                                       torch.as_tensor(t.dj), cfg)
        if rank == 0:
            out.update(u=u_n.numpy(), di=di_n.numpy(), dj=dj_n.numpy(),
                       total=it.metrics.total, per_frame=it.metrics.per_frame.numpy(),
                       per_pixel=it.metrics.per_pixel.numpy(),
                       plane=it.metrics.reference_plane.numpy(), rows=it.rows, frames=it.frames)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [Cfg(), Cfg(sigma=1.0, integrate=True)],
                         ids=["plain", "regularised"])
def test_two_rank_iteration_matches_unsharded(cfg):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from scan_helpers import tiny_scan
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, cfg), nprocs=world, join=True)
    assert len(out["rows"]) == 2 and out["rows"][0][1] == out["rows"][1][0]

    sc, w, m, u, t = tiny_scan(seed=21, n=7, ss=20, fs=24)
    good = np.ones(7, bool)
    good[3] = False
    ref = orc.make_object_map(sc.frames, good, w.w, m.mask, u.u, t.di, t.dj)
    u1, _, stack = orc.update_pixel_map(sc.frames, good, w.w, m.mask, *ref, u.u, t.di, t.dj,
                                        cfg.half_ss, cfg.half_fs, return_stack=True,
                                        sigma=cfg.sigma, integrate=cfg.integrate)
    di1, dj1 = orc.update_translations(sc.frames, good, w.w, m.mask, *ref, u1, t.di, t.dj,
                                       cfg.t_half_ss, cfg.t_half_fs)
    d = orc.calc_error(sc.frames, good, w.w, m.mask, *ref, u1, di1, dj1)
    # object maps differ only in float64 summation order across ranks, so
    # compare maps on pixels whose argmin is unique
    P = stack.shape[-1]
    part = np.partition(stack.reshape(-1, P), 1, axis=0)
    uniq = ((part[1] - part[0]) > 1e-9 * np.abs(part[0])).reshape(w.w.shape)
    if cfg.sigma > 0 or cfg.integrate:      # coupling stages: every argmin must agree
        assert uniq.all()
        uniq = np.ones_like(uniq)
    np.testing.assert_allclose(out["u"][:, uniq], u1[:, uniq], rtol=0, atol=1e-9)
    np.testing.assert_allclose(out["di"], di1, atol=1e-9)
    np.testing.assert_allclose(out["dj"], dj1, atol=1e-9)
    np.testing.assert_allclose(out["total"], d["total"], rtol=1e-10)
    np.testing.assert_allclose(out["per_frame"], d["per_frame"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(out["per_pixel"], d["per_pixel"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(out["plane"], d["reference_plane"], rtol=1e-9, atol=1e-12)
    assert out["per_frame"][3] == 0.0

"""Multi-GPU sharding of one PXST iteration.

One process per GPU (torchrun), ``torch.distributed`` over NCCL for the
exchanges.  The frame stack is replicated on every GPU (<= 8 GB vs 180 GB
HBM), so no data moves between phases except the small exchange tensors:

=====================  =================  ====================================
phase                  partition          exchange after it
=====================  =================  ====================================
K1 object formation    good frames        all-reduce(sum) of the int64
                                          fixed-point num/den (exact), max of
                                          the touched flags
K2 pixel-map search    detector rows,     all-gather of the u rows (exact)
                       balanced by work
                       pixel count
K3 translation search  good frames        all-gather of (di, dj) (exact)
K4 error maps          detector rows      all-reduce of the per-frame sums
                                          (float64) and of the int64 plane
                                          num/den (exact); all-gather of the
                                          per-pixel rows (exact)
=====================  =================  ====================================

The grid bbox is computed redundantly from the replicated u and t.  Row
shards need no halo (sigma = 0, integrate = False: pixels are independent,
recon.py:221-315).  The object map and the reference plane are integer sums
(fixsplat.cuh), so they are bit-identical for any number of GPUs; the
all-gathers are exact, so u and t then match the single-GPU result bit for
bit too; only the per-frame error sums differ, in float64 summation order.

The logic talks to an *executor* (``DeviceExecutor`` here; tests supply a
CPU one built on the oracle and run it under gloo), so the partitioning and
collective composition are exercised without GPUs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def partition_rows(row_work: np.ndarray, r0: int, world: int) -> list[tuple[int, int]]:
    """Split ROI rows [r0, r0 + len(row_work)) into `world` contiguous bands
    with (nearly) equal work-pixel counts."""
    n = len(row_work)
    cum = np.concatenate([[0], np.cumsum(row_work, dtype=np.int64)])
    total = cum[-1]
    cuts = [0]
    for k in range(1, world):
        target = total * k / world
        cut = int(np.searchsorted(cum, target, side="left"))
        cuts.append(min(max(cut, cuts[-1]), n))
    cuts.append(n)
    return [(r0 + cuts[k], r0 + cuts[k + 1]) for k in range(world)]


def partition_frames(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous blocks of the good-frame list."""
    edges = [round(n * k / world) for k in range(world + 1)]
    return [(edges[k], edges[k + 1]) for k in range(world)]


@dataclass
class ShardedMetrics:
    total_t: torch.Tensor          # [1] sum of per_frame over good frames (no host sync)
    per_frame: torch.Tensor
    per_pixel: torch.Tensor
    reference_plane: torch.Tensor

    @property
    def total(self) -> float:
        return float(self.total_t.item())


class ShardedIteration:
    """Runs object map -> pixel map -> (translations) -> error maps with the
    work split across the ranks of `group`."""

    def __init__(self, ex, rank: int, world: int, group=None):
        self.ex = ex
        self.rank = rank
        self.world = world
        self.group = group
        r0, r1, _, _ = ex.roi
        self.rows = partition_rows(ex.row_work_counts(), r0, world)
        self.frames = partition_frames(ex.n_good, world)
        self.max_rows = max(hi - lo for lo, hi in self.rows)
        self.max_frames = max(hi - lo for lo, hi in self.frames)

    # ----------------------------------------------------------- collectives
    def _host_staged(self, t: torch.Tensor) -> bool:
        """gloo groups over device tensors (multi-rank tests on one GPU) go
        through host copies; NCCL takes device tensors directly."""
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def _all_reduce(self, t: torch.Tensor, op=dist.ReduceOp.SUM) -> torch.Tensor:
        if self._host_staged(t):
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
            return t
        dist.all_reduce(t, op=op, group=self.group)
        return t

    def _all_reduce_acc(self, acc) -> None:
        """Splat accumulators of the ranks' frame / row shares: int64 sums
        (exact) and touched flags (max)."""
        self._all_reduce(acc.data)
        if getattr(acc, "touched", None) is not None:
            self._all_reduce(acc.touched, op=dist.ReduceOp.MAX)

    def _all_gather(self, out: torch.Tensor, buf: torch.Tensor) -> None:
        if self._host_staged(buf):
            h = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather_into_tensor(h, buf.cpu(), group=self.group)
            out.copy_(h)
            return
        dist.all_gather_into_tensor(out, buf, group=self.group)

    def _gather_rows(self, u_local: torch.Tensor) -> torch.Tensor:
        """Assemble a full [C, SS, FS] plane from each rank's row band (exact);
        rows outside every band keep u_local's values."""
        c, ss, fs = u_local.shape
        lo, hi = self.rows[self.rank]
        buf = torch.zeros((c, self.max_rows, fs), dtype=u_local.dtype, device=u_local.device)
        buf[:, : hi - lo] = u_local[:, lo:hi]
        out = torch.empty((self.world * c, self.max_rows, fs), dtype=u_local.dtype,
                          device=u_local.device)
        self._all_gather(out, buf.contiguous())
        out = out.view(self.world, c, self.max_rows, fs)
        u = u_local.clone()
        for k, (a, b) in enumerate(self.rows):
            u[:, a:b] = out[k, :, : b - a]
        return u

    def _gather_frames(self, di: torch.Tensor, dj: torch.Tensor):
        """Assemble translations searched on each rank's frame block (exact)."""
        good = self.ex.good_index_tensor()
        lo, hi = self.frames[self.rank]
        buf = torch.zeros((2, self.max_frames), dtype=di.dtype, device=di.device)
        idx = good[lo:hi]
        buf[0, : hi - lo] = di[idx]
        buf[1, : hi - lo] = dj[idx]
        out = torch.empty((self.world * 2, self.max_frames), dtype=di.dtype, device=di.device)
        self._all_gather(out, buf)
        out = out.view(self.world, 2, self.max_frames)
        di_o, dj_o = di.clone(), dj.clone()
        for k, (a, b) in enumerate(self.frames):
            di_o[good[a:b]] = out[k, 0, : b - a]
            dj_o[good[a:b]] = out[k, 1, : b - a]
        return di_o, dj_o

    # ---------------------------------------------------------------- phases
    def object_map(self, u, di, dj, geom=None):
        n0, m0, shape = geom.bbox() if geom is not None else self.ex.bbox(u, di, dj)
        lo, hi = self.frames[self.rank]
        acc = self.ex.object_splat(u, di, dj, n0, m0, shape, lo, hi)
        self._all_reduce_acc(acc)
        return self.ex.object_finish(acc, (n0, m0), shape)

    def pixel_map(self, ref, u, di, dj, half_ss, half_fs, sub=None, refine=True, opts=None,
                  geom=None):
        u_local = self.ex.pixel_map_search(ref, u, di, dj, half_ss, half_fs, sub, refine,
                                           rows=self.rows[self.rank], geom=geom)
        u_full = self._gather_rows(u_local)
        # sigma smoothing / irrotational projection (recon.py:298-311) couple all
        # pixels; they are small [SS, FS] planes, so every rank runs them on the
        # gathered map (deterministic kernels: the ranks stay identical)
        if opts is not None and (getattr(opts, "sigma", 0.0) > 0 or
                                 getattr(opts, "integrate", False)):
            u_full = self.ex.regularise(u_full, opts)
        return u_full

    def translations(self, ref, u, di, dj, half_ss, half_fs, sub=None):
        lo, hi = self.frames[self.rank]
        di_l, dj_l = self.ex.translation_search(ref, u, di, dj, half_ss, half_fs, sub, lo, hi)
        return self._gather_frames(di_l, dj_l)

    def error_maps(self, ref, u, di, dj) -> ShardedMetrics:
        per_frame, per_pixel, acc = self.ex.error_partials(ref, u, di, dj,
                                                           rows=self.rows[self.rank])
        # per-frame sums add; the per-pixel map is row-local (gathered); the
        # plane accumulators add exactly
        self._all_reduce(per_frame)
        per_pixel = self._gather_rows(per_pixel.reshape(1, *per_pixel.shape))[0]
        self._all_reduce_acc(acc)
        plane = self.ex.error_finish(acc, ref)
        good = self.ex.good_index_tensor()
        total = per_frame[good].sum().reshape(1) if len(good) else per_frame.new_zeros(1)
        return ShardedMetrics(total, per_frame, per_pixel, plane)

    def iteration(self, u, di, dj, cfg, ev=None, geom=None):
        """One full iteration with the reference's ordering (recon.py:511-516).
        `geom` = this iteration's geometry future (GeometryFuture, optional);
        the next one is left in self.next_geom (computed on every rank from
        the gathered u and translations, overlapping the error maps)."""
        ref = self.object_map(u, di, dj, geom)
        if ev:
            ev[0].record(torch.cuda.current_stream())
        u_new = self.pixel_map(ref, u, di, dj, cfg.half_ss, cfg.half_fs, cfg.subpixel_grid,
                               cfg.refine, opts=cfg, geom=geom)
        if ev:
            ev[1].record(torch.cuda.current_stream())
        di_new, dj_new = di, dj
        if cfg.update_translations:
            di_new, dj_new = self.translations(ref, u_new, di, dj, cfg.t_half_ss, cfg.t_half_fs,
                                               cfg.t_subpixel_grid)
        self.next_geom = self.ex.geometry_async(u_new, di_new, dj_new)
        self.metrics = self.error_maps(ref, u_new, di_new, dj_new)
        return u_new, di_new, dj_new


class DeviceExecutor:
    """Executor over a DeviceScan (the GPU kernels)."""

    def __init__(self, ds):
        self.ds = ds
        self.roi = ds.roi
        self.n_good = ds.n_good
        self._good = torch.as_tensor(ds.good_idx.astype(np.int64), device=ds.device)

    def row_work_counts(self) -> np.ndarray:
        r0, r1, c0, c1 = self.roi
        work = self.ds.work.view(self.ds.ss, self.ds.fs)[r0:r1, c0:c1]
        return work.sum(dim=1).cpu().numpy()

    def good_index_tensor(self) -> torch.Tensor:
        return self._good

    def bbox(self, u, di, dj):
        return self.ds.bbox(u, di, dj)

    def object_splat(self, u, di, dj, n0, m0, shape, lo, hi):
        return self.ds.object_splat(u, di, dj, n0, m0, shape, lo, hi)

    def object_finish(self, acc, origin, shape):
        return self.ds.object_finish(acc, origin, shape)

    def pixel_map_search(self, ref, u, di, dj, half_ss, half_fs, sub, refine, rows, geom=None):
        band = self.ds.band(*rows)
        u_out, _ = band.pixel_map_search(ref, u, di, dj, half_ss, half_fs, sub, refine,
                                         geom=geom)
        return u_out

    def geometry_async(self, u, di, dj):
        return self.ds.geometry_async(u, di, dj)

    def translation_search(self, ref, u, di, dj, half_ss, half_fs, sub, lo, hi):
        return self.ds.translation_search(ref, u, di, dj, half_ss, half_fs, sub, lo, hi)

    def error_partials(self, ref, u, di, dj, rows):
        return self.ds.band(*rows).error_partials(ref, u, di, dj)

    def error_finish(self, acc, ref):
        return self.ds.plane_finish(acc, ref.shape)

    def regularise(self, u, opts):
        return self.ds.regularise(u, opts)

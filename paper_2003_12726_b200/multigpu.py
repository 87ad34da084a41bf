"""Single-process multi-GPU PXST iteration.

``Devices([0, 1, ..., 7])`` runs the hot path on several GPUs from ONE
process -- no torchrun -- behind the drop-in ``run_main_loop(...,
devices=...)``.  Every GPU holds a ``DeviceScan`` of the scan (the frame
stack is replicated: <= 8 GB of 180 GB HBM) and the current u and
translations; the work splits as in ``sharding.py``:

=====================  ==================  ===================================
phase                  partition           exchange (peer copies over NVLink /
                                           NVSwitch + library add kernels)
=====================  ==================  ===================================
K1 object formation    good-frame blocks   int64 fixed-point num/den, touched:
                                           ONE kernel per device reads every
                                           peer's terms in place (P2P loads),
                                           adds them (exact: the object is
                                           bit-identical for any device
                                           count), normalises its slice of the
                                           cells and stores it into every
                                           peer's images (P2P stores):
                                           ``pxst_object_finish_peers``
K2 pixel-map search    detector-row bands  u rows gathered on every device
K3 translation search  good-frame blocks   (di, dj) of each block gathered
K4 error maps          detector-row bands  per-frame sums added in device
                                           order; per-pixel rows gathered;
                                           plane: the same fused peer finish
=====================  ==================  ===================================

A device id may repeat (``Devices([0, 0])``): two shares of the work on one
GPU, the functional check this one-GPU pool can run.  Cross-device copies
are ``Tensor.copy_`` between devices (cudaMemcpyPeerAsync, ordered against
both devices' current streams); the sums are the library's
``pxst_add_i64`` / ``pxst_add_f64`` / ``pxst_or_u8`` kernels.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _native
from ._native import check, stream_ptr
from .engine import DeviceScan
from .sharding import partition_frames, partition_rows


class Devices:
    """The GPUs one process drives (``pxst_ctx_create(n_dev, dev_ids)`` of
    SURVEY 8(b), as a Python context)."""

    def __init__(self, ids):
        ids = [int(i) for i in ids]
        if not ids:
            raise ValueError("Devices needs at least one device id")
        n = torch.cuda.device_count()
        for i in ids:
            if not 0 <= i < n:
                raise ValueError(f"no CUDA device {i} (visible: {n})")
        self.ids = ids

    def __len__(self) -> int:
        return len(self.ids)

    def __repr__(self) -> str:
        return f"Devices({self.ids})"


class MultiScan:
    """One scan resident on several GPUs, with the sharded phases."""

    def __init__(self, scan, w, m, roi, devices: Devices):
        self.devices = devices
        self.scans: list[DeviceScan] = []
        first_on: dict[int, DeviceScan] = {}
        for d in devices.ids:
            with torch.cuda.device(d):
                prev = first_on.get(d)
                if prev is None:
                    ds = DeviceScan(scan.frames, scan.good_frames, w.w, m.mask, roi)
                    first_on[d] = ds
                else:         # a repeated id shares the uploaded stack
                    ds = DeviceScan(scan.frames, scan.good_frames, w.w, m.mask, roi,
                                    frames_dev=prev.frames, frames_upload=prev._upload)
            self.scans.append(ds)
        d0 = self.scans[0]
        self.n_frames, self.empty = d0.n_frames, d0.empty
        r0, r1, c0, c1 = d0.roi
        work = d0.work.view(d0.ss, d0.fs)[r0:r1, c0:c1]
        self.rows = partition_rows(work.sum(dim=1).cpu().numpy(), r0, len(devices))
        self.frames = partition_frames(d0.n_good, len(devices))
        self.good = [torch.as_tensor(d0.good_idx.astype(np.int64), device=ds.device)
                     for ds in self.scans]
        self.lib = _native.lib()
        # the accumulators' all-reduce fused with their normalisation over peer
        # memory (PXST_MULTI_FUSED=0: peer copies + add kernels + per-device finish)
        self.fused_finish = os.environ.get("PXST_MULTI_FUSED", "1") != "0" and \
            len(devices) <= 16
        self._enable_peer_access()

    def _enable_peer_access(self):
        """Kernels of device a dereference pointers of device b: make torch
        enable peer access for every ordered pair of distinct devices (it does
        so on the first cross-device copy)."""
        ids = sorted(set(self.devices.ids))
        for a in ids:
            for b in ids:
                if a != b:
                    torch.empty(1, device=f"cuda:{a}").copy_(torch.empty(1, device=f"cuda:{b}"))

    # ------------------------------------------------------------ plumbing
    def on(self, k):
        return torch.cuda.device(self.devices.ids[k])

    def upload(self, u, di, dj):
        """Replicate (u, di, dj) on every device."""
        out = []
        for k, ds in enumerate(self.scans):
            with self.on(k):
                out.append((ds.upload_u(u), *ds.upload_t(di, dj)))
        return [list(x) for x in zip(*out)]

    def _add_peers_i64(self, ts):
        """ts[k] (int64, device k) += every peer's (exact)."""
        W = len(ts)
        copies = []
        for k in range(W):
            with self.on(k):
                copies.append([torch.empty_like(ts[k]).copy_(ts[j], non_blocking=True)
                               for j in range(W) if j != k])
        for k in range(W):
            with self.on(k):
                for c in copies[k]:
                    check(self.lib.pxst_add_i64(ts[k].data_ptr(), c.data_ptr(), ts[k].numel(),
                                                stream_ptr()))

    def _finish_peers(self, accs, shape, origin=None):
        """The all-reduce of the shards' fixed-point accumulators fused with the
        normalisation (``pxst_object_finish_peers``): device k reads every
        peer's int64 terms in place (P2P loads), adds them exactly, normalises
        its 1/W slice of the cells and stores the results into every peer's
        output images (P2P stores).  origin given: DeviceRefs (object map);
        None: reference planes (float64).  Same bits as adding the peers'
        accumulators and finishing on each device."""
        W = len(accs)
        os_, of = shape
        n = os_ * of
        outs = []
        for k, ds in enumerate(self.scans):
            with self.on(k):
                i_ref = torch.empty(n, dtype=torch.float64, device=ds.device)
                if origin is None:
                    outs.append((i_ref, None, None, None))
                else:
                    outs.append((i_ref, torch.empty(n, dtype=torch.float64, device=ds.device),
                                 torch.empty(n, dtype=torch.float32, device=ds.device),
                                 torch.empty(n, dtype=torch.uint8, device=ds.device)))
        ready = []
        for k in range(W):                 # the peers' splats, in each device's stream order
            with self.on(k):
                ev = torch.cuda.Event()
                ev.record()
                ready.append(ev)
        c_accs = (_native.PxstAccum * W)(*[a.c() for a in accs])

        def ptrs(idx):
            if outs[0][idx] is None:
                return None
            return (ctypes.c_void_p * W)(*[o[idx].data_ptr() for o in outs])
        arrs = [ptrs(i) for i in range(4)]
        bounds = [n * k // W for k in range(W + 1)]
        done = []
        for k in range(W):
            with self.on(k):
                st = torch.cuda.current_stream()
                for j in range(W):
                    if j != k:
                        st.wait_event(ready[j])
                check(self.lib.pxst_object_finish_peers(c_accs, W, bounds[k], bounds[k + 1],
                                                        *arrs, stream_ptr()))
                ev = torch.cuda.Event()
                ev.record()
                done.append(ev)
        for k in range(W):                 # a device's images are complete once every peer's
            with self.on(k):               # slice has landed
                st = torch.cuda.current_stream()
                for j in range(W):
                    if j != k:
                        st.wait_event(done[j])
        if origin is None:
            return [o[0].view(os_, of) for o in outs]
        from .engine import DeviceRef
        return [DeviceRef(o[0].view(os_, of), o[1].view(os_, of), o[2].view(os_, of),
                          o[3].view(os_, of), (int(origin[0]), int(origin[1]))) for o in outs]

    def _or_peers_u8(self, ts):
        W = len(ts)
        copies = []
        for k in range(W):
            with self.on(k):
                copies.append([torch.empty_like(ts[k]).copy_(ts[j], non_blocking=True)
                               for j in range(W) if j != k])
        for k in range(W):
            with self.on(k):
                for c in copies[k]:
                    check(self.lib.pxst_or_u8(ts[k].data_ptr(), c.data_ptr(), ts[k].numel(),
                                              stream_ptr()))

    def _sum_f64_ordered(self, ts):
        """Every device: sum_j ts[j] in device order j = 0..W-1 (identical bits
        on all devices)."""
        W = len(ts)
        parts = []
        for k in range(W):
            with self.on(k):
                parts.append([ts[j] if j == k else
                              torch.empty_like(ts[k]).copy_(ts[j], non_blocking=True)
                              for j in range(W)])
        out = []
        for k in range(W):
            with self.on(k):
                acc = torch.zeros_like(ts[k])
                for p in parts[k]:
                    check(self.lib.pxst_add_f64(acc.data_ptr(), p.data_ptr(), acc.numel(),
                                                stream_ptr()))
                out.append(acc)
        return out

    def _gather_rows(self, planes):
        """planes[k]: [C, SS, FS] on device k with its row band filled; every
        device gets every band (exact copies)."""
        W = len(planes)
        for k in range(W):
            with self.on(k):
                for j, (a, b) in enumerate(self.rows):
                    if j != k and b > a:
                        planes[k][:, a:b].copy_(planes[j][:, a:b], non_blocking=True)
        return planes

    # --------------------------------------------------------------- phases
    def object_map(self, us, dis, djs, bbox=None):
        n0, m0, shape = bbox or self.scans[0].bbox(us[0], dis[0], djs[0])
        accs = []
        for k, ds in enumerate(self.scans):
            lo, hi = self.frames[k]
            with self.on(k):
                accs.append(ds.object_splat(us[k], dis[k], djs[k], n0, m0, shape, lo, hi))
        if self.fused_finish:
            return self._finish_peers(accs, shape, (n0, m0))
        self._add_peers_i64([a.data for a in accs])
        self._or_peers_u8([a.touched for a in accs])
        refs = []
        for k, ds in enumerate(self.scans):
            with self.on(k):
                refs.append(ds.object_finish(accs[k], (n0, m0), shape))
        return refs

    def pixel_map(self, refs, us, dis, djs, half_ss, half_fs, sub=None, refine=True, opts=None,
                  geom=None):
        outs = []
        for k, ds in enumerate(self.scans):
            with self.on(k):
                band = ds.band(*self.rows[k])
                u_k, _ = band.pixel_map_search(refs[k], us[k], dis[k], djs[k], half_ss, half_fs,
                                               sub, refine, geom=geom)
                outs.append(u_k)
        outs = self._gather_rows(outs)
        if opts is not None:          # sigma / integrate couple all pixels: every device
            for k, ds in enumerate(self.scans):      # runs them on the gathered map
                with self.on(k):
                    ds.regularise(outs[k], opts)
        return outs

    def translations(self, refs, us, dis, djs, half_ss, half_fs, sub=None):
        W = len(self.scans)
        res = []
        for k, ds in enumerate(self.scans):
            lo, hi = self.frames[k]
            with self.on(k):
                res.append(ds.translation_search(refs[k], us[k], dis[k], djs[k], half_ss, half_fs,
                                                 sub, lo, hi))
        out_i, out_j = [r[0] for r in res], [r[1] for r in res]
        for k in range(W):
            with self.on(k):
                for j in range(W):
                    lo, hi = self.frames[j]
                    if j == k or hi <= lo:
                        continue
                    idx = self.good[k][lo:hi]
                    out_i[k].index_copy_(0, idx, res[j][0].to(out_i[k].device)[idx])
                    out_j[k].index_copy_(0, idx, res[j][1].to(out_j[k].device)[idx])
        return out_i, out_j

    def error_maps(self, refs, us, dis, djs):
        parts = []
        q = None
        for k, ds in enumerate(self.scans):
            with self.on(k):
                qk = ds.plane_quanta(refs[k])       # full-scan quanta: equal on every device
                parts.append(ds.band(*self.rows[k]).error_partials(refs[k], us[k], dis[k], djs[k],
                                                                   quanta=qk))
        per_frame = self._sum_f64_ordered([p[0] for p in parts])
        per_pixel = self._gather_rows([p[1].reshape(1, *p[1].shape) for p in parts])
        accs = [p[2] for p in parts]
        planes = None
        if self.fused_finish:
            planes = self._finish_peers(accs, refs[0].shape)
        else:
            self._add_peers_i64([a.data for a in accs])
        out = []
        for k, ds in enumerate(self.scans):
            with self.on(k):
                plane = planes[k] if planes is not None else ds.plane_finish(accs[k], refs[k].shape)
                good = self.good[k]
                total = per_frame[k][good].sum().reshape(1) if len(good) else \
                    per_frame[k].new_zeros(1)
                out.append((total, per_frame[k], per_pixel[k][0], plane, ds.sigma2.view(ds.ss, ds.fs)))
        return out


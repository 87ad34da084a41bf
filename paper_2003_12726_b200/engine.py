"""Device-resident state of one scan and thin wrappers over the C ABI.

``DeviceScan`` owns the device copies (torch CUDA tensors -- torch is only
the allocator/stream plumbing) of one scan's frame stack, whitefield, work
mask and good-frame list, plus the iteration-invariant statistics (K0), and
exposes one method per kernel family:

==========================  =======================  ===========================
method                      C entry point            reference
==========================  =======================  ===========================
``object_map``              pxst_bbox, pxst_object_  recon.make_reference
                            splat/finish             (recon.py:99-141)
``pixel_map_search``        pxst_pixel_map_search    recon.update_pixel_map
                                                     (recon.py:221-315)
``translation_search``      pxst_translation_search  recon.update_translations
                                                     (recon.py:336-385)
``error_maps``              pxst_error_maps          recon.calc_error
                                                     (recon.py:388-438)
==========================  =======================  ===========================

Work-set semantics follow ``recon._work_set`` (recon.py:81-96): good frames
are ``np.flatnonzero(good_frames)``; work pixels are ``mask & (W > 0)``
inside the half-open ROI (numpy-slice clipped to the detector).
"""

from __future__ import annotations

import ctypes
import os
import math
import weakref
import zlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._native import PxstAccum, PxstCgInfo, PxstRef, PxstScan, PxstStats, check, stream_ptr


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _device() -> torch.device:
    _native.lib()
    return torch.device("cuda", torch.cuda.current_device())


# Host<->device byte counters (bench.py's e2e accounting).
TRANSFER = {"h2d": 0, "d2h": 0}

# Element types a frame stack may be uploaded in (pxst_stack_to_f32's codes; float32 goes
# as it is, anything else is converted on the host)
_STACK_CODES = {"u1": 1, "b1": 1, "i1": 2, "u2": 3, "i2": 4, "u4": 5, "i4": 6, "u8": 7, "i8": 8,
                "f8": 9}

# Frame chunks in which a pageable stack is staged into pinned memory
# (DeviceScan._upload_pageable); PXST_STAGE_CHUNKS=1: one piece, as before.
_STAGE_CHUNKS = max(1, int(os.environ.get("PXST_STAGE_CHUNKS", "8")))


def to_device(a: np.ndarray, dtype: np.dtype, device) -> torch.Tensor:
    """Host -> device copy of a contiguous array in the requested dtype.

    Never blocks the host on the device: a pageable array is staged through
    a pinned buffer from torch's caching host allocator (which keeps the
    block until the copy has run), then copied asynchronously like a pinned
    one.  (A pageable cudaMemcpy would wait for everything queued before it,
    e.g. a stack upload.)"""
    h = np.ascontiguousarray(a, dtype=dtype)
    TRANSFER["h2d"] += h.nbytes
    if h.flags.writeable:
        t = torch.from_numpy(h)
        if t.is_pinned():
            return t.to(device, non_blocking=True)
    tdt = torch.from_numpy(h[:0].copy()).dtype
    pin = torch.empty(h.shape, dtype=tdt, pin_memory=True)
    if h.flags.writeable and h.nbytes >= (8 << 20) and h.ndim >= 1 and h.shape[0] >= 2 \
            and _STAGE_CHUNKS > 1:
        # a large pageable array (e.g. frame weights [N, SS, FS]): staged in chunks by
        # torch's threaded host copy, each chunk's DMA under the next chunk's staging
        src = torch.from_numpy(h)
        out = torch.empty(h.shape, dtype=tdt, device=device)
        n = h.shape[0]
        k = min(n, _STAGE_CHUNKS)
        edges = [n * c // k for c in range(k + 1)]
        for lo, hi in zip(edges[:-1], edges[1:]):
            pin[lo:hi].copy_(src[lo:hi])
            out[lo:hi].copy_(pin[lo:hi], non_blocking=True)
        return out
    np.copyto(pin.numpy(), h)
    return pin.to(device, non_blocking=True)


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device -> host copy (synchronising)."""
    return to_host_many(t)[0]


def to_host_many(*ts: torch.Tensor) -> list[np.ndarray]:
    """Device -> host copies of several tensors through pinned buffers, one
    stream synchronisation for all of them."""
    outs = []
    for t in ts:
        TRANSFER["d2h"] += t.numel() * t.element_size()
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t.detach(), non_blocking=True)
        outs.append(h)
    if ts:
        torch.cuda.current_stream(ts[0].device).synchronize()
    return [h.numpy() for h in outs]


def clip_roi(roi, shape) -> tuple[int, int, int, int]:
    """ROI as numpy slicing would apply it (recon.py:84-85)."""
    ss, fs = shape
    if roi is None:
        return 0, ss, 0, fs
    r0, r1, c0, c1 = (int(v) for v in (roi.ss_min, roi.ss_max, roi.fs_min, roi.fs_max))
    return min(r0, ss), min(r1, ss), min(c0, fs), min(c1, fs)


def _nvtx(name: str):
    """NVTX range around a kernel-launching method when ``PXST_NVTX=1`` (for
    nsys / ncu --nvtx timelines); a no-op otherwise."""
    def wrap(fn):
        if os.environ.get("PXST_NVTX") != "1":
            return fn

        def inner(*a, **k):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **k)
            finally:
                torch.cuda.nvtx.range_pop()
        inner.__name__ = fn.__name__
        inner.__doc__ = fn.__doc__
        return inner
    return wrap


@dataclass
class DeviceRef:
    """Reference image on device (f64 for the boundary, f32 masked for kernels)."""

    i_ref: torch.Tensor | None   # [os, of] f64 (None when built from a host image)
    wsum: torch.Tensor | None
    fm: torch.Tensor             # [os, of] f32, 0 where invalid
    valid: torch.Tensor          # [os, of] u8
    origin: tuple[int, int]

    @property
    def shape(self) -> tuple[int, int]:
        return tuple(self.fm.shape)

    fm64: torch.Tensor | None = None  # [os, of] f64 masked image (error maps)

    def struct(self) -> PxstRef:
        os_, of = self.fm.shape
        f64 = self.fm64 if self.fm64 is not None else self.i_ref
        return PxstRef(self.fm.data_ptr(), self.valid.data_ptr(), os_, of, int(self.origin[0]),
                       int(self.origin[1]), _ptr(f64))

    @classmethod
    def from_host(cls, i_ref, wsum, origin, device) -> "DeviceRef":
        i_ref = np.asarray(i_ref, dtype=np.float64)
        ok = np.asarray(wsum) > 0                      # data_model.py:186-188
        fm64 = np.where(ok, i_ref, 0.0)
        return cls(None, None, to_device(fm64, np.float32, device),
                   to_device(ok.astype(np.uint8), np.uint8, device),
                   (int(origin[0]), int(origin[1])), to_device(fm64, np.float64, device))


_SOLVERS = {"cg": 0, "mgcg": 1}


class Accum:
    """Deterministic splat accumulators on the device (``pxst_accum``): int64
    [4, cells] = numerator, denominator (units of the device quanta,
    float64[2]) and their tiny-weight parts (units of quanta * 2^-20), plus
    the touched flags (uint8, optional).  Frame shards add ``data`` exactly
    (int64 all-reduce) and ``touched`` with max."""

    def __init__(self, cells: int, quanta: torch.Tensor, device, touched: bool = True):
        self.data = torch.empty((4, cells), dtype=torch.int64, device=device)
        self.touched = torch.empty(cells, dtype=torch.uint8, device=device) if touched else None
        self.quanta = quanta
        c = self.c()
        check(_native.lib().pxst_accum_zero(ctypes.byref(c), cells, stream_ptr()))

    @property
    def cells(self) -> int:
        return int(self.data.shape[1])

    def c(self) -> PxstAccum:
        return PxstAccum(self.data[0].data_ptr(), self.data[1].data_ptr(), self.data[2].data_ptr(),
                         self.data[3].data_ptr(), _ptr(self.touched), self.quanta.data_ptr())


def _grid_rule(b) -> tuple[int, int, tuple[int, int]]:
    """Object-grid origin and shape from the bbox values (recon.py:126-132)."""
    u0min, u0max, u1min, u1max, dimin, dimax, djmin, djmax = b
    n0 = int(math.floor(u0min - dimax))
    m0 = int(math.floor(u1min - djmax))
    return n0, m0, (int(math.floor(u0max - dimin)) - n0 + 2,
                    int(math.floor(u1max - djmin)) - m0 + 2)


class GeometryFuture:
    """Result of DeviceScan.geometry_async (pinned host values + event; the
    grid (n0, m0, os, of) also stays on the device for kernels that read it
    without a host round trip)."""

    def __init__(self, host8, host2, event, grid_dev, grid_event):
        self._host8, self._host2, self._event = host8, host2, event
        self.grid_dev = grid_dev
        self._grid_event = grid_event

    def gpu_wait(self, stream=None):
        """Make `stream` (default: current) wait on the GPU for grid_dev (the
        tile spans and host copies behind it are not waited for)."""
        (stream or torch.cuda.current_stream()).wait_event(self._grid_event)

    def bbox(self) -> tuple[int, int, tuple[int, int]]:
        self._event.synchronize()
        return _grid_rule(self._host8.tolist())

    def spans_ptr(self) -> int:
        """Host address of K2's span hint (int32[2]), valid after the event."""
        self._event.synchronize()
        return self._host2.data_ptr()

    def spans3_hint(self, grow: int = 0):
        """K3's span hint (host int32[2]) of this geometry's u, widened by
        `grow` rows / columns (a bound for a map moved by <= grow / 2 px);
        None when the future was made without spans3."""
        self._event.synchronize()
        if int(self._host2[2]) < 0:
            return None
        h = torch.empty(2, dtype=torch.int32, pin_memory=True)
        h[0] = int(self._host2[2]) + grow
        h[1] = int(self._host2[3]) + grow
        return h


class PendingObject:
    """Next-iteration object accumulated by error_maps_and_next_object;
    resolve() finishes it once the grid is known on the host (normally long
    after the fact), or forms it afresh if the grid outgrew the capacity."""

    def __init__(self, ds, acc, cap, geom, inputs):
        self.ds, self.acc, self.cap, self.geom, self.inputs = ds, acc, cap, geom, inputs

    def resolve(self) -> DeviceRef:
        n0, m0, shape = self.geom.bbox()
        n = shape[0] * shape[1]
        if n > self.cap:
            return self.ds.object_map(*self.inputs, geom=self.geom)
        return self.ds.object_finish(self.acc, (n0, m0), shape)


class DeviceScan:
    """One scan + whitefield + mask + ROI resident on the current CUDA device."""

    def __init__(self, frames, good_frames, W, mask, roi=None, device=None,
                 frames_dev: torch.Tensor | None = None, frames_upload: dict | None = None):
        self.device = device or _device()
        self.lib = _native.lib()
        frames_shape = tuple(frames_dev.shape) if frames_dev is not None else np.shape(frames)
        if len(frames_shape) != 3:
            raise ValueError("frames must be 3-D [N, SS, FS]")
        self.n_frames, self.ss, self.fs = (int(v) for v in frames_shape)
        self.roi = clip_roi(roi, (self.ss, self.fs))
        r0, r1, c0, c1 = self.roi
        W = np.asarray(W)
        mask = np.asarray(mask)
        self.good_idx = np.flatnonzero(np.asarray(good_frames)).astype(np.int32)
        self.n_good = int(self.good_idx.size)
        dev = self.device
        # frames uploads still in flight: [(good_lo, good_hi, event)] on a copy
        # stream (pinned host stacks; shared with band views through the dict)
        self._upload = {"chunks": [], "waited": True, "stats": 0}   # stats: K0 parts run
        if frames_upload is not None and not frames_upload["waited"]:
            # a stack shared with another scan whose upload may still be in
            # flight: wait for the same copy events before any kernel reads it
            # (the copies run in order on one stream: the last event covers all;
            # the chunk ranges index the other scan's good frames, so one range
            # over this scan's good frames replaces them)
            last = frames_upload["chunks"][-1][2]
            self._upload.update(chunks=[(0, self.n_good, last)], waited=False,
                                host=frames_upload.get("host"))
        if frames_upload is not None and frames_upload.get("absmax") is not None:
            self._upload["absmax"] = frames_upload["absmax"]     # same stack, same bound
        self._uploads: list = []     # identity cache of pixel maps / translations
        if frames_dev is None:
            frames_dev = self._upload_frames(frames, dev)
        self.frames = frames_dev
        work = np.zeros((self.ss, self.fs), dtype=np.uint8)
        if r1 > r0 and c1 > c0:
            work[r0:r1, c0:c1] = (mask[r0:r1, c0:c1] & (W[r0:r1, c0:c1] > 0)) != 0
        self.n_work = int(work.sum())
        self.good = to_device(self.good_idx if self.n_good else np.zeros(1, np.int32), np.int32, dev)
        self.w64 = to_device(W, np.float64, dev)
        self.w32 = self.w64.to(torch.float32)
        self.work = to_device(work, np.uint8, dev)
        self._work_host = work.astype(bool)
        roi4 = (ctypes.c_int64 * 4)(r0, max(r1, r0 + 1), c0, max(c1, c0 + 1))
        self.c_scan = PxstScan(self.frames.data_ptr(), self.n_frames, self.ss, self.fs,
                               self.good.data_ptr(), self.n_good, self.w64.data_ptr(),
                               self.w32.data_ptr(), self.work.data_ptr(), roi4)
        self.empty = self.n_work == 0 or self.n_good == 0 or r1 <= r0 or c1 <= c0
        self.full_c_scan = self.c_scan     # band views keep the full scan's (shared quanta)
        self._side = None            # side stream of geometry_async
        self._support_components = None   # project_irrotational's solver choice
        plane = self.ss * self.fs
        self.var_pm = torch.zeros(plane, dtype=torch.float64, device=dev)
        self.sigma2 = torch.zeros(plane, dtype=torch.float64, device=dev)
        self.frame_norm = torch.zeros(max(self.n_good, 1), dtype=torch.float64, device=dev)
        self.scalars = torch.zeros(4, dtype=torch.float64, device=dev)
        self.c_stats = PxstStats(self.var_pm.data_ptr(), self.sigma2.data_ptr(),
                                 self.frame_norm.data_ptr(), self.scalars.data_ptr())
        # K0 (pxst_stack_stats) runs when a kernel first needs the stack
        # statistics (ready()); object formation does not, so make_reference
        # overlaps the stack upload instead of waiting behind K0.
        self._upload["stats"] = 3 if self.empty else 0

    @property
    def scalars_host(self) -> np.ndarray:
        """K0 scalars on the host (synchronises; not needed by the hot path)."""
        if self.empty:
            return np.array([1.0, 0.0, 0.0, 0.0])
        self.ready(frame_stats=True)
        return to_host(self.scalars).copy()

    # ------------------------------------------------- stack upload / K0
    _UPLOAD_CHUNKS = 1     # (object formation's other inputs queue behind the stack on
                           # the copy engine, so splitting its splat bought nothing)

    def _upload_frames(self, frames, dev):
        """Stack to HBM.  A pinned host stack is copied in frame chunks on a
        copy stream (one event per chunk), so object formation can splat the
        chunks that have landed while the rest is in flight; every other
        consumer waits for the whole stack (ready())."""
        a = np.asarray(frames)
        code = _STACK_CODES.get(a.dtype.str.lstrip("<>=|"))
        if code is not None and a.dtype.isnative and a.flags.c_contiguous and a.flags.writeable \
                and self.n_good > 0 and a.nbytes >= (1 << 20) and a.ndim == 3 and a.shape[0] >= 2:
            return self._upload_native(a, code, dev)
        h = np.ascontiguousarray(frames, dtype=np.float32)
        t = torch.from_numpy(h) if h.flags.writeable else None
        if t is not None and not t.is_pinned() and self.n_good > 0 and h.nbytes >= (8 << 20) \
                and h.shape[0] >= 2 and _STAGE_CHUNKS > 1:
            return self._upload_pageable(t, dev)
        if t is None or not t.is_pinned() or self.n_good == 0:
            return to_device(frames, np.float32, dev)
        out = torch.empty(t.shape, dtype=torch.float32, device=dev)
        copy = torch.cuda.Stream(dev)
        copy.wait_stream(torch.cuda.current_stream(dev))
        good = self.good_idx
        n = self._UPLOAD_CHUNKS
        bounds = [int(good[min(len(good) - 1, (len(good) * c) // n)]) for c in range(n)]
        bounds = sorted(set([0] + bounds[1:])) + [self.n_frames]
        spans = [(f0, f1) for f0, f1 in zip(bounds[:-1], bounds[1:]) if f1 > f0]
        chunks = []

        def issue(span_list):
            with torch.cuda.stream(copy):
                for f0, f1 in span_list:
                    out[f0:f1].copy_(t[f0:f1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                    g0, g1 = np.searchsorted(good, [f0, f1])
                    chunks.append((int(g0), int(g1), ev))

        issue(spans)
        TRANSFER["h2d"] += h.nbytes
        out.record_stream(copy)
        self._upload.update(chunks=chunks, waited=False, host=t)
        return out

    def _upload_native(self, a: np.ndarray, code: int, dev):
        """A stack of another element type (detector counts are usually 16- or
        32-bit integers; the reference casts per use, recon.py:91): uploaded as
        it is -- half the bytes for uint16, and no conversion pass over the
        stack on the host -- then converted to the kernels' float32 on the
        device (pxst_stack_to_f32, numpy's rounding)."""
        n = a.shape[0]
        raw = torch.from_numpy(a.view(np.uint8).reshape(n, -1))
        pinned = raw.is_pinned()
        raw_dev = torch.empty(raw.shape, dtype=torch.uint8, device=dev)
        out = torch.empty(a.shape, dtype=torch.float32, device=dev)
        pin = raw if pinned else torch.empty(raw.shape, dtype=torch.uint8, pin_memory=True)
        copy = torch.cuda.Stream(dev)
        copy.wait_stream(torch.cuda.current_stream(dev))
        k = min(n, _STAGE_CHUNKS)
        edges = [n * c // k for c in range(k + 1)]
        with torch.cuda.stream(copy):
            for lo, hi in zip(edges[:-1], edges[1:]):
                if not pinned:
                    pin[lo:hi].copy_(raw[lo:hi])
                raw_dev[lo:hi].copy_(pin[lo:hi], non_blocking=True)
            check(self.lib.pxst_stack_to_f32(raw_dev.data_ptr(), code, a.size, out.data_ptr(),
                                             stream_ptr(copy)))
            ev = torch.cuda.Event()
            ev.record(copy)
        TRANSFER["h2d"] += a.nbytes
        out.record_stream(copy)
        raw_dev.record_stream(copy)
        self._upload.update(chunks=[(0, self.n_good, ev)], waited=False, host=pin)
        return out

    def _upload_pageable(self, src: torch.Tensor, dev):
        """A plain (pageable) numpy stack -- what a drop-in caller passes --
        staged into a pinned buffer in frame chunks by torch's threaded host
        copy, each chunk going to the device on the copy stream while the next
        is staged.  One np.copyto of the whole stack and then one DMA took
        4 + 1.3 ms for config 1's 63 MB (e2e 6.5 ms per step); chunked 4.0 ms
        (numpy copies from a thread pool instead: 5.0 ms, they do not run in
        parallel)."""
        n = src.shape[0]
        out = torch.empty(src.shape, dtype=torch.float32, device=dev)
        pin = torch.empty(src.shape, dtype=torch.float32, pin_memory=True)
        copy = torch.cuda.Stream(dev)
        copy.wait_stream(torch.cuda.current_stream(dev))
        k = min(n, _STAGE_CHUNKS)
        edges = [n * c // k for c in range(k + 1)]
        with torch.cuda.stream(copy):
            for a, b in zip(edges[:-1], edges[1:]):
                pin[a:b].copy_(src[a:b])
                out[a:b].copy_(pin[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        TRANSFER["h2d"] += src.numel() * 4
        out.record_stream(copy)
        self._upload.update(chunks=[(0, self.n_good, ev)], waited=False, host=pin)
        return out

    def wait_frames(self) -> "DeviceScan":
        """Make the current stream wait for the whole stack upload."""
        up = self._upload
        if not up["waited"]:
            st = torch.cuda.current_stream(self.device)
            for _, _, ev in up["chunks"]:
                st.wait_event(ev)
            up.update(waited=True, host=None)
        return self

    def absmax(self) -> torch.Tensor:
        """max |I| over the stack (device float64[1], pxst_stack_absmax): the
        bound the fixed-point splat quanta derive from; once per stack."""
        up = self._upload
        if up.get("absmax") is None:
            self.wait_frames()
            t = torch.empty(1, dtype=torch.float64, device=self.device)
            check(self.lib.pxst_stack_absmax(ctypes.byref(self.c_scan), t.data_ptr(), stream_ptr()))
            up["absmax"] = t
        return up["absmax"]

    def object_quanta(self) -> torch.Tensor:
        """Quanta of this scan's object accumulators (device float64[2]); the
        same for every frame range and band view of the scan."""
        up = self._upload
        if up.get("obj_q") is None:
            q = torch.empty(2, dtype=torch.float64, device=self.device)
            check(self.lib.pxst_object_quanta(ctypes.byref(self.full_c_scan),
                                              self.absmax().data_ptr(), q.data_ptr(),
                                              stream_ptr()))
            up["obj_q"] = q
        return up["obj_q"]

    def plane_quanta(self, ref: "DeviceRef") -> torch.Tensor:
        """Quanta of the reference-plane accumulators of `ref`, from the full
        scan (row shards must share them)."""
        self.ready()
        q = torch.empty(2, dtype=torch.float64, device=self.device)
        c_ref = ref.struct()
        check(self.lib.pxst_plane_quanta(ctypes.byref(self.full_c_scan), self.absmax().data_ptr(),
                                         ctypes.byref(self.c_stats), ctypes.byref(c_ref),
                                         q.data_ptr(), stream_ptr()))
        return q

    @_nvtx("pxst K0 stack statistics")
    def ready(self, frame_stats: bool = False) -> "DeviceScan":
        """Make the current stream wait for the whole stack and run the K0
        parts not yet run: the per-pixel part always (K2, K4), the per-frame
        part (frame_norm) only for K3."""
        up = self._upload
        self.wait_frames()
        parts = (0 if up["stats"] & 1 else 1) | (2 if frame_stats and not up["stats"] & 2 else 0)
        if parts:
            up["stats"] |= parts
            check(self.lib.pxst_stack_stats_parts(ctypes.byref(self.c_scan), None,
                                                  ctypes.byref(self.c_stats), parts,
                                                  stream_ptr()))
        return self

    def host_bbox(self, u, di, dj):
        """Grid rule (recon.py:126-132) from host arrays, in the device
        kernel's arithmetic (exact min/max over work pixels and good frames,
        NaN ignored); None when it does not apply (non-finite values).
        make_reference uses it while the stack upload holds the copy engine
        (inputs of a device bbox would queue behind the stack)."""
        w = self._work_host.ravel()
        u = np.asarray(u, dtype=np.float64)
        g = self.good_idx
        di = np.asarray(di, dtype=np.float64)[g]
        dj = np.asarray(dj, dtype=np.float64)[g]

        def ext(plane, lo):
            # unmasked extremum first: when a work pixel attains it, it is the
            # masked one too (nearly every pixel is a work pixel)
            flat = plane.ravel()
            k = int(np.argmin(flat) if lo else np.argmax(flat))
            if w[k]:
                return flat[k]
            red = np.fmin.reduce if lo else np.fmax.reduce
            return red(plane, axis=None, where=self._work_host, initial=np.inf if lo else -np.inf)

        vals = [ext(u[0], True), ext(u[0], False), ext(u[1], True), ext(u[1], False),
                np.fmin.reduce(di), np.fmax.reduce(di), np.fmin.reduce(dj), np.fmax.reduce(dj)]
        vals = [float(v) for v in vals]
        if not all(math.isfinite(v) for v in vals):
            return None
        return _grid_rule(vals)

    # ------------------------------------------------------------------ utils
    def _cached(self, arrays, make):
        """Device copy of host arrays, cached by their identity under the
        value-object convention of the scan cache (data_model.py:13): the
        drop-in API uploads a pixel map / translation set once, and a map it
        returned is found again on the device (see remember)."""
        key = tuple(_ScanCache._ident(a) for a in arrays)
        fps = tuple(_ScanCache._fp(a) for a in arrays)
        for k, refs, val, fp in self._uploads:
            if k == key and fp == fps and all(r() is not None for r in refs):
                return val
        val = make()
        self.remember(arrays, val)
        return val

    def remember(self, arrays, val) -> None:
        key = tuple(_ScanCache._ident(a) for a in arrays)
        fps = tuple(_ScanCache._fp(a) for a in arrays)
        self._uploads = [e for e in self._uploads if e[0] != key]
        self._uploads.append((key, [_ScanCache._ref(a) for a in arrays], val, fps))
        del self._uploads[:-8]

    def upload_u(self, u, cache: bool = False) -> torch.Tensor:
        """Pixel map to the device.  cache=True (drop-in API only: callers
        never write into the returned tensor) reuses a resident copy."""
        u = np.asarray(u)
        if u.shape != (2, self.ss, self.fs):
            raise ValueError(f"pixel map must have shape (2, {self.ss}, {self.fs})")
        if cache:
            return self._cached((u,), lambda: to_device(u, np.float64, self.device))
        return to_device(u, np.float64, self.device)

    def upload_t(self, di, dj, cache: bool = False) -> tuple[torch.Tensor, torch.Tensor]:
        if cache:
            a, b = np.asarray(di), np.asarray(dj)
            if a.dtype == np.float64 and b.dtype == np.float64:
                return self._cached((a, b), lambda: self.upload_t(a, b))
        di = np.asarray(di, dtype=np.float64)
        dj = np.asarray(dj, dtype=np.float64)
        if di.shape != (self.n_frames,) or dj.shape != (self.n_frames,):
            raise ValueError(f"translations must have shape ({self.n_frames},)")
        return to_device(di, np.float64, self.device), to_device(dj, np.float64, self.device)

    # -------------------------------------------------------------- K1 object
    def bbox(self, u_t, di_t, dj_t) -> tuple[int, int, tuple[int, int]]:
        """Grid origin and shape by the rule of recon.py:126-132."""
        out = torch.empty(8, dtype=torch.float64, device=self.device)
        check(self.lib.pxst_bbox(ctypes.byref(self.c_scan), u_t.data_ptr(), di_t.data_ptr(),
                                 dj_t.data_ptr(), out.data_ptr(), stream_ptr()))
        return _grid_rule(to_host(out).tolist())

    def geometry_async(self, u_t, di_t, dj_t, spans3: bool = True) -> "GeometryFuture":
        """Start the host-side geometry of an iteration on a side stream: the
        object-grid bbox (recon.py:126-132), K2's tile spans of u and (with
        spans3) K3's.  The main stream is not blocked; reading the future
        waits only for these small reductions, so an iteration loop can fetch
        the next iteration's geometry while the current error maps run."""
        main = torch.cuda.current_stream(self.device)
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
        side = self._side
        ready = torch.cuda.Event()
        ready.record(main)
        side.wait_event(ready)
        host8 = torch.empty(8, dtype=torch.float64, pin_memory=True)
        host2 = torch.empty(4, dtype=torch.int32, pin_memory=True)
        with torch.cuda.stream(side):
            dev8 = torch.empty(8, dtype=torch.float64, device=self.device)
            dev2 = torch.empty(4, dtype=torch.int32, device=self.device)
            grid = torch.empty(4, dtype=torch.int64, device=self.device)
            sp = stream_ptr(side)
            check(self.lib.pxst_bbox_grid(ctypes.byref(self.c_scan), u_t.data_ptr(),
                                          di_t.data_ptr(), dj_t.data_ptr(), dev8.data_ptr(),
                                          grid.data_ptr(), sp))
            grid_ready = torch.cuda.Event()      # what device-side consumers wait for
            grid_ready.record(side)
            host8.copy_(dev8, non_blocking=True)
            check(self.lib.pxst_tile_spans(ctypes.byref(self.c_scan), u_t.data_ptr(),
                                           dev2.data_ptr(), sp))
            if spans3:
                check(self.lib.pxst_tile_spans3(ctypes.byref(self.c_scan), u_t.data_ptr(),
                                                dev2[2:].data_ptr(), sp))
            else:
                dev2[2:].fill_(-1)
            host2.copy_(dev2, non_blocking=True)
            done = torch.cuda.Event()
            done.record(side)
        for t in (u_t, di_t, dj_t):
            t.record_stream(side)
        TRANSFER["d2h"] += 8 * 8 + 4 * 4
        return GeometryFuture(host8, host2, done, grid, grid_ready)

    @_nvtx("pxst K1 object splat")
    def object_splat(self, u_t, di_t, dj_t, n0, m0, shape, frame_lo=0, frame_hi=None,
                     acc: "Accum | None" = None) -> Accum:
        """Fixed-point object accumulators (Accum, os*of cells) for a range of
        good frames; added into `acc` when given."""
        os_, of = shape
        if acc is None:
            acc = Accum(os_ * of, self.object_quanta(), self.device)
        hi = self.n_good if frame_hi is None else frame_hi
        self.wait_frames()
        c_acc = acc.c()
        check(self.lib.pxst_object_splat(
            ctypes.byref(self.c_scan), u_t.data_ptr(), di_t.data_ptr(), dj_t.data_ptr(), n0, m0,
            os_, of, frame_lo, hi, ctypes.byref(c_acc), None, stream_ptr()))
        return acc

    def object_finish(self, acc: Accum, origin, shape) -> DeviceRef:
        os_, of = shape
        n = os_ * of
        i_ref = torch.empty(n, dtype=torch.float64, device=self.device)
        wsum = torch.empty(n, dtype=torch.float64, device=self.device)
        fm = torch.empty(n, dtype=torch.float32, device=self.device)
        valid = torch.empty(n, dtype=torch.uint8, device=self.device)
        c_acc = acc.c()
        check(self.lib.pxst_object_finish(ctypes.byref(c_acc), n, i_ref.data_ptr(),
                                          wsum.data_ptr(), fm.data_ptr(), valid.data_ptr(),
                                          stream_ptr()))
        return DeviceRef(i_ref.view(os_, of), wsum.view(os_, of), fm.view(os_, of),
                         valid.view(os_, of), (int(origin[0]), int(origin[1])))

    def object_map(self, u_t, di_t, dj_t, geom: "GeometryFuture | None" = None,
                   host=None) -> DeviceRef:
        """host = the (u, di, dj) host arrays of this state, if the caller has
        them and the stack upload is still in flight: the grid is then derived
        on the host (host_bbox)."""
        if self.empty:
            raise ValueError("make_reference: empty good pixel/frame set")  # recon.py:116-117
        hb = None
        if geom is None and host is not None and not self._upload["waited"]:
            hb = self.host_bbox(*host)
        if hb is not None:
            n0, m0, shape = hb
        else:
            n0, m0, shape = geom.bbox() if geom is not None else self.bbox(u_t, di_t, dj_t)
        acc = self.object_splat(u_t, di_t, dj_t, n0, m0, shape)
        return self.object_finish(acc, (n0, m0), shape)

    # ---------------------------------------------------------- K2 pixel map
    def frame_weight_stats(self, fw_t: torch.Tensor) -> torch.Tensor:
        self.ready()
        var_fw = torch.zeros(self.ss * self.fs, dtype=torch.float64, device=self.device)
        tmp_s2 = torch.zeros_like(var_fw)
        fn = torch.zeros_like(self.frame_norm)
        sc = torch.zeros_like(self.scalars)
        st = PxstStats(var_fw.data_ptr(), tmp_s2.data_ptr(), fn.data_ptr(), sc.data_ptr())
        check(self.lib.pxst_stack_stats(ctypes.byref(self.c_scan), fw_t.data_ptr(),
                                        ctypes.byref(st), stream_ptr()))
        return var_fw

    @_nvtx("pxst K2 pixel-map search")
    def pixel_map_search(self, ref: DeviceRef, u_t, di_t, dj_t, half_ss, half_fs,
                         subpixel_grid=None, refine=True, fw_t=None,
                         geom: "GeometryFuture | None" = None):
        spans = None
        if geom is None and not self.empty:
            # K2 sizes its TMA box from the tile spans of u: queue them (and
            # their copy to the host) ahead of K0 on this stream, so the host
            # waits for them while K0 runs instead of synchronising inside the
            # search call
            dev2 = torch.empty(2, dtype=torch.int32, device=self.device)
            spans = torch.empty(2, dtype=torch.int32, pin_memory=True)
            check(self.lib.pxst_tile_spans(ctypes.byref(self.c_scan), u_t.data_ptr(),
                                           dev2.data_ptr(), stream_ptr()))
            spans.copy_(dev2, non_blocking=True)
            spans_ready = torch.cuda.Event()
            spans_ready.record()
            TRANSFER["d2h"] += 8
        self.ready()
        u_out = torch.empty_like(u_t)
        err = torch.empty(self.ss * self.fs, dtype=torch.float64, device=self.device)
        if self.empty:
            u_out.copy_(u_t)
            err.zero_()
            return u_out, err.view(self.ss, self.fs)
        var_fw = self.frame_weight_stats(fw_t) if fw_t is not None else None
        c_ref = ref.struct()
        if spans is not None:
            spans_ready.synchronize()
            hint = spans.data_ptr()
        else:
            hint = geom.spans_ptr()
        check(self.lib.pxst_pixel_map_search_ex(
            ctypes.byref(self.c_scan), ctypes.byref(self.c_stats), ctypes.byref(c_ref),
            u_t.data_ptr(), di_t.data_ptr(), dj_t.data_ptr(), int(half_ss), int(half_fs),
            float(subpixel_grid or 0.0), int(bool(refine)), _ptr(fw_t), _ptr(var_fw),
            u_out.data_ptr(), err.data_ptr(), hint, stream_ptr()))
        return u_out, err.view(self.ss, self.fs)

    # ------------------------------------------------------- K3 translations
    @_nvtx("pxst K3 translation search")
    def translation_search(self, ref: DeviceRef, u_t, di_t, dj_t, half_ss, half_fs,
                           subpixel_grid=None, frame_lo=0, frame_hi=None, err_out=None,
                           span_hint=None):
        """span_hint: GeometryFuture.spans3_hint(...) (host int32[2]) or None
        (the call then reads K3's tile spans from the device, a stream sync)."""
        self.ready(frame_stats=True)
        di_out = di_t.clone()
        dj_out = dj_t.clone()
        if self.empty:
            return di_out, dj_out
        hi = self.n_good if frame_hi is None else frame_hi
        c_ref = ref.struct()
        check(self.lib.pxst_translation_search_ex(
            ctypes.byref(self.c_scan), ctypes.byref(self.c_stats), ctypes.byref(c_ref),
            u_t.data_ptr(), di_t.data_ptr(), dj_t.data_ptr(), int(half_ss), int(half_fs),
            float(subpixel_grid or 0.0), int(frame_lo), int(hi), di_out.data_ptr(),
            dj_out.data_ptr(), _ptr(err_out), _ptr(span_hint), stream_ptr()))
        return di_out, dj_out

    # ------------------------------------------------------- shard views / K4
    def band(self, r0: int, r1: int) -> "DeviceScan":
        """View restricted to detector rows [r0, r1) of the ROI; shares every
        device buffer and the (full-ROI) statistics with this scan."""
        import copy
        self.ready()
        v = copy.copy(self)
        R0, R1, C0, C1 = self.roi
        lo, hi = max(r0, R0), min(r1, R1)
        v.roi = (lo, hi, C0, C1)
        roi4 = (ctypes.c_int64 * 4)(lo, max(hi, lo + 1), C0, max(C1, C0 + 1))
        v.c_scan = PxstScan(self.frames.data_ptr(), self.n_frames, self.ss, self.fs,
                            self.good.data_ptr(), self.n_good, self.w64.data_ptr(),
                            self.w32.data_ptr(), self.work.data_ptr(), roi4)
        v.empty = self.empty or hi <= lo
        return v

    def error_partials(self, ref: DeviceRef, u_t, di_t, dj_t, quanta=None):
        """K4 without normalisation: (per_frame, per_pixel, plane Accum) with
        the full scan's plane quanta (or `quanta`)."""
        self.ready()
        per_frame = torch.zeros(self.n_frames, dtype=torch.float64, device=self.device)
        per_pixel = torch.zeros(self.ss * self.fs, dtype=torch.float64, device=self.device)
        q = quanta if quanta is not None else self.plane_quanta(ref)
        acc = Accum(ref.fm.numel(), q, self.device, touched=False)
        if not self.empty:
            c_ref = ref.struct()
            c_acc = acc.c()
            check(self.lib.pxst_error_partials(
                ctypes.byref(self.c_scan), ctypes.byref(self.c_stats), ctypes.byref(c_ref),
                u_t.data_ptr(), di_t.data_ptr(), dj_t.data_ptr(), per_frame.data_ptr(),
                per_pixel.data_ptr(), ctypes.byref(c_acc), stream_ptr()))
        return per_frame, per_pixel.view(self.ss, self.fs), acc

    def plane_finish(self, acc: Accum, shape):
        plane = torch.empty(acc.cells, dtype=torch.float64, device=self.device)
        c_acc = acc.c()
        check(self.lib.pxst_object_finish(ctypes.byref(c_acc), acc.cells, plane.data_ptr(), None,
                                          None, None, stream_ptr()))
        return plane.view(*shape)

    # ---------------------------------------------------------- K4 error maps
    @_nvtx("pxst K4 error maps")
    def error_maps(self, ref: DeviceRef, u_t, di_t, dj_t):
        self.ready()
        # pxst_error_maps zeroes per_frame / per_pixel / total and writes every
        # plane cell itself
        alloc = torch.zeros if self.empty else torch.empty
        per_frame = alloc(self.n_frames, dtype=torch.float64, device=self.device)
        per_pixel = alloc(self.ss * self.fs, dtype=torch.float64, device=self.device)
        plane = alloc(ref.fm.numel(), dtype=torch.float64, device=self.device)
        total = alloc(1, dtype=torch.float64, device=self.device)
        if not self.empty:
            c_ref = ref.struct()
            check(self.lib.pxst_error_maps(
                ctypes.byref(self.c_scan), ctypes.byref(self.c_stats), ctypes.byref(c_ref),
                u_t.data_ptr(), di_t.data_ptr(), dj_t.data_ptr(), self.absmax().data_ptr(),
                per_frame.data_ptr(), per_pixel.data_ptr(), plane.data_ptr(), total.data_ptr(),
                stream_ptr()))
        return (total, per_frame, per_pixel.view(self.ss, self.fs), plane.view(*ref.shape),
                self.sigma2.view(self.ss, self.fs))

    @_nvtx("pxst K4 error maps + next K1")
    def error_maps_and_next_object(self, ref: DeviceRef, u_t, di_t, dj_t,
                                   geom: "GeometryFuture", margin: int = 32):
        """K4 of (ref, u, t) fused with the next iteration's object formation
        on (u, t) (recon.py:511-516), without any host wait: the next grid is
        read on the device from `geom` (= geometry_async(u, di, dj)), and the
        accumulators are sized from the current grid plus `margin` cells per
        side.  Returns the error-map tensors and a PendingObject."""
        self.ready()
        os_, of = ref.shape
        cap = (os_ + 2 * margin) * (of + 2 * margin)
        acc = Accum(cap, self.object_quanta(), self.device)
        per_frame = torch.empty(self.n_frames, dtype=torch.float64, device=self.device)
        per_pixel = torch.empty(self.ss * self.fs, dtype=torch.float64, device=self.device)
        plane = torch.empty(ref.fm.numel(), dtype=torch.float64, device=self.device)
        total = torch.empty(1, dtype=torch.float64, device=self.device)
        geom.gpu_wait()
        c_ref = ref.struct()
        c_acc = acc.c()
        check(self.lib.pxst_error_maps_splat(
            ctypes.byref(self.c_scan), ctypes.byref(self.c_stats), ctypes.byref(c_ref),
            u_t.data_ptr(), di_t.data_ptr(), dj_t.data_ptr(), self.absmax().data_ptr(),
            per_frame.data_ptr(), per_pixel.data_ptr(), plane.data_ptr(), total.data_ptr(),
            geom.grid_dev.data_ptr(), cap, ctypes.byref(c_acc), stream_ptr()))
        metrics = (total, per_frame, per_pixel.view(self.ss, self.fs), plane.view(*ref.shape),
                   self.sigma2.view(self.ss, self.fs))
        return metrics, PendingObject(self, acc, cap, geom, (u_t, di_t, dj_t))

    # ------------------------------------- 8(f) pixel-map regularisation
    def smooth_displacement(self, u_t, sigma: float):
        """Mask-aware Gaussian regularisation of u_t in place (recon.py:300-304);
        the support is the work set."""
        if sigma > 0:
            check(self.lib.pxst_smooth_displacement(u_t.data_ptr(), self.work.data_ptr(),
                                                    self.ss, self.fs, float(sigma),
                                                    stream_ptr()))
        return u_t

    def project_irrotational(self, u_t, tol: float = 1e-12, maxiter: int | None = None,
                             solver: str = "auto"):
        """Irrotational projection of u_t in place (recon.py:305-311), converged
        to the reference's tolerance: "mgcg" = multigrid-preconditioned CG,
        "cg" = the reference's plain CG, "auto" (default) = "mgcg" when the
        support has one linked component (integration.linked_components)."""
        if solver == "auto":
            if self._support_components is None:
                from .integration import linked_components
                self._support_components = linked_components(self.work.cpu().numpy())
            solver = "mgcg" if self._support_components <= 1 else "cg"
        info = PxstCgInfo()
        check(self.lib.pxst_project_irrotational(u_t.data_ptr(), self.work.data_ptr(), self.ss,
                                                 self.fs, float(tol), int(maxiter or 0),
                                                 _SOLVERS[solver], ctypes.byref(info),
                                                 stream_ptr()))
        return info

    @_nvtx("pxst pixel-map regularisation")
    def regularise(self, u_t, opts):
        """The optional stages of recon.update_pixel_map, in its order."""
        if getattr(opts, "sigma", 0.0) > 0:
            self.smooth_displacement(u_t, opts.sigma)
        if getattr(opts, "integrate", False):
            self.project_irrotational(u_t)
        return u_t


# ---------------------------------------------------------------------------
# identity cache of device scans (value-object convention, data_model.py:13)
# ---------------------------------------------------------------------------
class _ScanCache:
    """Caches DeviceScan objects keyed by the identity of the host arrays.

    The reference treats its dataclasses as immutable value objects
    (data_model.py:13: "construct once, then share read-only"); the cache
    relies on that: an array mutated in place after a call must be passed as
    a new array, or the cache cleared with :func:`clear_cache`.
    """

    def __init__(self, max_entries: int = 2):
        self.entries: list[tuple[tuple, list, DeviceScan]] = []
        self.max_entries = max_entries
        self.enabled = True

    @staticmethod
    def _ident(a):
        a = np.asarray(a)
        return (id(a), a.__array_interface__["data"][0], a.shape, a.dtype.str, a.strides)

    @staticmethod
    def _fp(a) -> int:
        """Content fingerprint: CRC-32 of ~512 evenly strided elements (a few
        microseconds, whatever the array size).  An array mutated in place
        between calls is caught when a sampled element changed (e.g. any
        rescaled frame); the caches then re-upload instead of returning stale
        device data."""
        flat = np.asarray(a).reshape(-1)
        if flat.size == 0:
            return 0
        step = max(1, flat.size // 512)
        return zlib.crc32(np.ascontiguousarray(flat[step // 2::step]).view(np.uint8))

    @staticmethod
    def _ref(a):
        try:
            return weakref.ref(a)
        except TypeError:
            return lambda: a

    def get(self, scan, w, m, roi) -> DeviceScan:
        frames = scan.frames
        arrays = (frames, scan.good_frames, w.w, m.mask)
        key = tuple(self._ident(a) for a in arrays) + (
            None if roi is None else clip_roi(roi, scan.shape),)
        fps = tuple(self._fp(a) for a in arrays)
        if self.enabled:
            # every keyed array is held by a weak reference: an identity match
            # with all of them alive cannot be a recycled address; the content
            # fingerprints catch arrays mutated in place since
            self.entries = [e for e in self.entries
                            if not (e[0] == key and e[3] != fps)]
            for k, refs, ds, fp in self.entries:
                if k == key and all(r() is not None for r in refs):
                    return ds
        frames_dev = upload = None
        if self.enabled:
            # reuse an uploaded stack when only W / mask / ROI / good frames differ
            # (with its upload events: the copy may still be running)
            for k, refs, ds, fp in self.entries:
                if k[0] == key[0] and refs[0]() is not None and fp[0] == fps[0]:
                    frames_dev, upload = ds.frames, ds._upload
                    break
        ds = DeviceScan(frames, scan.good_frames, w.w, m.mask, roi, frames_dev=frames_dev,
                        frames_upload=upload)
        if self.enabled:
            self.entries.append((key, [self._ref(a) for a in arrays], ds, fps))
            del self.entries[:-self.max_entries]
        return ds

    def clear(self):
        self.entries.clear()


SCAN_CACHE = _ScanCache()


def clear_cache() -> None:
    """Drop every cached device scan / reference and return the memory: torch's
    caching allocator and the scratch the library keeps in the device's
    default pool (pxst_release_pool)."""
    SCAN_CACHE.clear()
    from . import recon
    recon._REF_CACHE.clear()
    torch.cuda.empty_cache()
    if torch.cuda.is_available():
        check(_native.lib().pxst_release_pool())

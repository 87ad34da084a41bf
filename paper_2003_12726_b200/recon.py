"""Drop-in replacement of the reference's ``pxst.recon`` hot path on B200.

Same names, arguments, dataclasses and float64 arrays in and out as
``/root/reference/pkg/src/pxst/recon.py``; the arithmetic runs in the
sm_100a kernels of ``libpxst_b200.so`` (see ``engine.py``).  There is no CPU
fallback: without the library or a CUDA device every call raises.

Scope: ``make_reference`` (alias ``make_object_map``),
``update_pixel_map``, ``update_translations``, ``calc_error``,
``run_main_loop`` and the option types, including the optional pixel-map
stages ``UpdateOptions.sigma > 0`` (mask-aware Gaussian regularisation) and
``integrate=True`` (irrotational projection), section 8(f) rows 1-2.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from .data_model import (
    ErrorMetrics,
    Geometry,
    PixelMap,
    PixelMask,
    PixelTranslations,
    ReferenceImage,
    Roi,
    ScanData,
    Whitefield,
)
from .engine import SCAN_CACHE, DeviceRef, DeviceScan, _ScanCache, to_host, to_host_many

# Relative floor applied to per-pixel intensity variances (recon.py:34).
VAR_EPS_REL = 1e-8


@dataclass(frozen=True)
class SearchWindow:
    """Brute-force search extent (recon.py:37-57)."""

    half_ss: int = 4
    half_fs: int = 4
    subpixel_grid: float | None = None

    def __post_init__(self):
        if self.half_ss < 0 or self.half_fs < 0:
            raise ValueError("search window halves must be >= 0")
        if self.subpixel_grid is not None and not 0 < self.subpixel_grid <= 1:
            raise ValueError("subpixel_grid step must be in (0, 1]")

    def offsets(self, axis: int) -> np.ndarray:
        half = self.half_ss if axis == 0 else self.half_fs
        if self.subpixel_grid is None:
            return np.arange(-half, half + 1, dtype=np.float64)
        k = int(round(half / self.subpixel_grid))
        return self.subpixel_grid * np.arange(-k, k + 1, dtype=np.float64)


@dataclass(frozen=True)
class UpdateOptions:
    """Pixel-map update knobs (recon.py:60-78)."""

    quadratic_refinement: bool = True
    integrate: bool = False
    sigma: float = 0.0
    include_current: bool = True   # never read by the reference either (recon.py:74)

    def __post_init__(self):
        if self.sigma < 0:
            raise ValueError("sigma must be >= 0")


@dataclass(frozen=True)
class IterationSettings:
    """Per-iteration configuration of the main loop (recon.py:441-448)."""

    window: SearchWindow = SearchWindow(2, 2)
    options: UpdateOptions = UpdateOptions()
    update_translations: bool = False
    translation_window: SearchWindow = SearchWindow(2, 2)


def default_schedule(max_iters: int) -> list[IterationSettings]:
    """The reference's coarse-to-fine defaults (recon.py:451-468)."""
    sigmas = [5.0, 3.0] + [1.0] * max(0, max_iters - 2)
    out = []
    for i in range(max_iters):
        out.append(IterationSettings(
            window=SearchWindow(4, 4) if i == 0 else SearchWindow(2, 2),
            options=UpdateOptions(quadratic_refinement=True, integrate=True, sigma=sigmas[i]),
            update_translations=(i >= 1),
            translation_window=SearchWindow(2, 2)))
    return out


@dataclass
class LoopResult:
    pixel_map: PixelMap
    reference: ReferenceImage
    translations: PixelTranslations
    history: list = field(default_factory=list)


# ---------------------------------------------------------------------------
# device reference-image cache: ReferenceImages produced here keep their
# device copy, so a make_reference -> update_pixel_map chain never re-uploads.
# ---------------------------------------------------------------------------
_REF_CACHE: dict[int, tuple] = {}


def _remember(ref: ReferenceImage, dref: DeviceRef) -> None:
    for k in [k for k, (a, b, _, _) in _REF_CACHE.items() if a() is None or b() is None]:
        del _REF_CACHE[k]
    fp = (_ScanCache._fp(ref.i_ref), _ScanCache._fp(ref.wsum))
    _REF_CACHE[id(ref.i_ref)] = (weakref.ref(ref.i_ref), weakref.ref(ref.wsum), dref, fp)


def _device_ref(ref, ds: DeviceScan) -> DeviceRef:
    hit = _REF_CACHE.get(id(ref.i_ref))
    if hit is not None:
        a, b, dref, fp = hit
        if a() is ref.i_ref and b() is ref.wsum and tuple(dref.origin) == tuple(ref.origin) \
                and dref.fm.device == ds.device \
                and fp == (_ScanCache._fp(ref.i_ref), _ScanCache._fp(ref.wsum)):
            return dref
    return DeviceRef.from_host(ref.i_ref, ref.wsum, ref.origin, ds.device)


def _host(t: torch.Tensor) -> np.ndarray:
    return to_host(t)


def _ref_image(dref: DeviceRef, geom) -> ReferenceImage:
    du, dv = (geom.du, geom.dv) if geom is not None else (1.0, 1.0)
    i_ref, wsum = to_host_many(dref.i_ref, dref.wsum)
    out = ReferenceImage(i_ref=i_ref, wsum=wsum,
                         origin=(int(dref.origin[0]), int(dref.origin[1])), du=du, dv=dv)
    _remember(out, dref)
    return out


# ---------------------------------------------------------------------------
# public hot-path API
# ---------------------------------------------------------------------------
def make_reference(scan: ScanData, w: Whitefield, m: PixelMask, u: PixelMap,
                   t: PixelTranslations, roi: Roi | None = None,
                   geom: Geometry | None = None) -> ReferenceImage:
    """Object (reference-image) formation (recon.py:99-141) on the GPU (K1)."""
    ds = SCAN_CACHE.get(scan, w, m, roi)
    if ds.empty:
        raise ValueError("make_reference: empty good pixel/frame set")
    u_t = ds.upload_u(u.u, cache=True)
    di_t, dj_t = ds.upload_t(t.di, t.dj, cache=True)
    return _ref_image(ds.object_map(u_t, di_t, dj_t, host=(u.u, t.di, t.dj)), geom)


make_object_map = make_reference


def update_pixel_map(scan: ScanData, w: Whitefield, m: PixelMask, ref: ReferenceImage,
                     u: PixelMap, t: PixelTranslations, win: SearchWindow,
                     opts: UpdateOptions = UpdateOptions(), roi: Roi | None = None,
                     frame_weights: np.ndarray | None = None, threads: int = 1):
    """Pixel-map grid search + argmin + paraboloid (recon.py:221-315) on the GPU (K2).

    ``threads`` is accepted for signature compatibility; results never
    depend on it (recon.py:163-169).  Returns ``(PixelMap, err_map)``.
    """
    ds = SCAN_CACHE.get(scan, w, m, roi)
    u_t = ds.upload_u(u.u, cache=True)
    di_t, dj_t = ds.upload_t(t.di, t.dj, cache=True)
    fw_t = None
    if frame_weights is not None:
        fw = np.asarray(frame_weights)
        if fw.shape != (ds.n_frames, ds.ss, ds.fs):
            fw = np.broadcast_to(fw, (ds.n_frames, ds.ss, ds.fs))
        from .engine import to_device
        fw_t = to_device(fw, np.float32, ds.device)
    dref = _device_ref(ref, ds)
    u_out, err = ds.pixel_map_search(dref, u_t, di_t, dj_t, win.half_ss, win.half_fs,
                                     win.subpixel_grid, opts.quadratic_refinement, fw_t)
    ds.regularise(u_out, opts)                           # recon.py:298-311
    u_h, err_h = to_host_many(u_out, err)
    ds.remember((u_h,), u_out)     # a later call on the returned map reuses u_out
    return PixelMap(u_h), err_h


def update_translations(scan: ScanData, w: Whitefield, m: PixelMask, ref: ReferenceImage,
                        u: PixelMap, t: PixelTranslations, win: SearchWindow,
                        roi: Roi | None = None) -> PixelTranslations:
    """Per-frame translation grid search (recon.py:336-385) on the GPU (K3)."""
    ds = SCAN_CACHE.get(scan, w, m, roi)
    u_t = ds.upload_u(u.u, cache=True)
    di_t, dj_t = ds.upload_t(t.di, t.dj, cache=True)
    dref = _device_ref(ref, ds)
    di_o, dj_o = ds.translation_search(dref, u_t, di_t, dj_t, win.half_ss, win.half_fs,
                                       win.subpixel_grid)
    di_h, dj_h = to_host_many(di_o, dj_o)
    ds.remember((di_h, dj_h), (di_o, dj_o))
    return PixelTranslations(di=di_h, dj=dj_h)


def _metrics(total, per_frame, per_pixel, plane, variance) -> ErrorMetrics:
    t, pf, pp, pl, var = to_host_many(total, per_frame, per_pixel, plane, variance)
    return ErrorMetrics(total=float(t[0]), per_frame=pf, per_pixel=pp, reference_plane=pl,
                        variance=var)


def calc_error(scan: ScanData, w: Whitefield, m: PixelMask, ref: ReferenceImage, u: PixelMap,
               t: PixelTranslations, roi: Roi | None = None) -> ErrorMetrics:
    """Error decomposition (recon.py:388-438) on the GPU (K4)."""
    ds = SCAN_CACHE.get(scan, w, m, roi)
    u_t = ds.upload_u(u.u, cache=True)
    di_t, dj_t = ds.upload_t(t.di, t.dj, cache=True)
    dref = _device_ref(ref, ds)
    return _metrics(*ds.error_maps(dref, u_t, di_t, dj_t))


def quadratic_subpixel_refine(err3x3: np.ndarray) -> tuple[float, float]:
    """Paraboloid minimum of one 3x3 patch (recon.py:173-180).

    Host-side scalar helper kept for API compatibility; the kernels apply
    the same formula (search.cu ``paraboloid``) to every pixel / frame.
    """
    e = np.asarray(err3x3, dtype=np.float64).reshape(9)
    X = np.repeat([-1.0, 0.0, 1.0], 3)
    Y = np.tile([-1.0, 0.0, 1.0], 3)
    s0 = e.sum()
    b, c, f = e @ X / 6.0, e @ Y / 6.0, e @ (X * Y) / 4.0
    d = (-2.0 * s0 + 3.0 * (e @ (X * X))) / 6.0
    g = (-2.0 * s0 + 3.0 * (e @ (Y * Y))) / 6.0
    det = 4.0 * d * g - f * f
    if d > 0 and det > 0:
        return (float(np.clip((-2.0 * g * b + f * c) / det, -1, 1)),
                float(np.clip((-2.0 * d * c + f * b) / det, -1, 1)))
    return 0.0, 0.0


def run_main_loop(scan: ScanData, w: Whitefield, m: PixelMask, u: PixelMap,
                  t: PixelTranslations, roi: Roi | None = None, geom: Geometry | None = None,
                  schedule: list[IterationSettings] | None = None, max_iters: int = 10,
                  tol: float = 1e-3, threads: int = 1, progress_cb=None,
                  devices=None) -> LoopResult:
    """Device-resident main loop with the reference's ordering (recon.py:479-522).

    u, translations and the reference stay on the GPU between steps; per
    iteration the host only reads the grid shape (bbox) and the error
    metrics (which the history records, as the reference does).

    ``devices`` (extension, default None = the current GPU): a
    ``multigpu.Devices`` (or list of device ids); the iteration then runs on
    all of them from this one process (frames shard object formation and
    translations, detector rows the pixel map and error maps).
    """
    if schedule is None:
        schedule = default_schedule(max_iters)
    if len(schedule) < max_iters:
        schedule = list(schedule) + [schedule[-1]] * (max_iters - len(schedule))
    if devices is not None:
        from .multigpu import Devices
        devs = devices if isinstance(devices, Devices) else Devices(devices)
        return _run_main_loop_multi(scan, w, m, u, t, roi, geom, schedule, max_iters, tol,
                                    progress_cb, devs)
    ds = SCAN_CACHE.get(scan, w, m, roi)
    if ds.empty:
        raise ValueError("make_reference: empty good pixel/frame set")
    u_t = ds.upload_u(u.u, cache=True)
    di_t, dj_t = ds.upload_t(t.di, t.dj, cache=True)
    def needs_k3(i):      # K3's tile spans only for iterations that update translations
        return i < max_iters and bool(schedule[i].update_translations)

    gfut = ds.geometry_async(u_t, di_t, dj_t, spans3=needs_k3(0))
    dref = ds.object_map(u_t, di_t, dj_t, geom=gfut)
    history = [_metrics(*ds.error_maps(dref, u_t, di_t, dj_t))]
    if progress_cb:
        progress_cb(0.0, f"initial error {history[0].total:.6g}")
    # make_reference(u, t) at the top of every iteration sees the (u, t) of the
    # error maps just before it (recon.py:504-516): iteration 0 reuses the
    # initial object, later ones get it from the same pass over the stack as
    # those error maps (pxst_error_maps_splat)
    nref = None
    for i in range(max_iters):
        st = schedule[i]
        if nref is not None:
            dref = nref.resolve()
        u_t, _ = ds.pixel_map_search(dref, u_t, di_t, dj_t, st.window.half_ss,
                                     st.window.half_fs, st.window.subpixel_grid,
                                     st.options.quadratic_refinement, geom=gfut)
        ds.regularise(u_t, st.options)
        if st.update_translations:
            tw = st.translation_window
            # K3's TMA box from this iteration's geometry (u before the pixel-map
            # update, which moves a pixel by <= half + 1 px): no stream sync
            grow = 2 * (max(st.window.half_ss, st.window.half_fs) + 1)
            di_t, dj_t = ds.translation_search(dref, u_t, di_t, dj_t, tw.half_ss, tw.half_fs,
                                               tw.subpixel_grid,
                                               span_hint=gfut.spans3_hint(grow))
        gfut = ds.geometry_async(u_t, di_t, dj_t, spans3=needs_k3(i + 1))   # next iteration's
        if i + 1 < max_iters:
            metrics, nref = ds.error_maps_and_next_object(dref, u_t, di_t, dj_t, gfut)
        else:
            metrics = ds.error_maps(dref, u_t, di_t, dj_t)
        history.append(_metrics(*metrics))
        if progress_cb:
            progress_cb((i + 1) / max_iters, f"iter {i + 1} error {history[-1].total:.6g}")
        prev, curr = history[-2].total, history[-1].total
        if prev > 0 and (prev - curr) / prev < tol:
            break
    return LoopResult(pixel_map=PixelMap(_host(u_t)), reference=_ref_image(dref, geom),
                      translations=PixelTranslations(_host(di_t), _host(dj_t)), history=history)


def _run_main_loop_multi(scan, w, m, u, t, roi, geom, schedule, max_iters, tol, progress_cb,
                         devs) -> LoopResult:
    """run_main_loop over several GPUs of this process (multigpu.MultiScan)."""
    from .multigpu import MultiScan
    ms = MultiScan(scan, w, m, roi, devs)
    if ms.empty:
        raise ValueError("make_reference: empty good pixel/frame set")
    us, dis, djs = ms.upload(u.u, t.di, t.dj)
    refs = ms.object_map(us, dis, djs)
    history = [_metrics(*ms.error_maps(refs, us, dis, djs)[0])]
    if progress_cb:
        progress_cb(0.0, f"initial error {history[0].total:.6g}")
    for i in range(max_iters):
        st = schedule[i]
        refs = ms.object_map(us, dis, djs)
        us = ms.pixel_map(refs, us, dis, djs, st.window.half_ss, st.window.half_fs,
                          st.window.subpixel_grid, st.options.quadratic_refinement,
                          opts=st.options)
        if st.update_translations:
            tw = st.translation_window
            dis, djs = ms.translations(refs, us, dis, djs, tw.half_ss, tw.half_fs,
                                       tw.subpixel_grid)
        history.append(_metrics(*ms.error_maps(refs, us, dis, djs)[0]))
        if progress_cb:
            progress_cb((i + 1) / max_iters, f"iter {i + 1} error {history[-1].total:.6g}")
        prev, curr = history[-2].total, history[-1].total
        if prev > 0 and (prev - curr) / prev < tol:
            break
    return LoopResult(pixel_map=PixelMap(_host(us[0])), reference=_ref_image(refs[0], geom),
                      translations=PixelTranslations(_host(dis[0]), _host(djs[0])),
                      history=history)

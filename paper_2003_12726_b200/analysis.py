"""Drop-in of the reference's split-half uncertainty estimate
(``pxst.analysis.split_half_recon``, analysis.py:306-361), SURVEY 8(f) row 3.

The two half-data pixel-map refinements run on the GPU: the counter-based
sample split is generated on the device (``pxst_split_weights``) and fed to
K2's frame-weight path; the per-pixel half counts come from
``pxst_split_counts``.  Only the final statistics over the difference of the
two maps (histograms, median) run on the host, on [2, SS, FS] arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._native import check, stream_ptr
from .data_model import PixelMap, PixelMask, PixelTranslations, ReferenceImage, Roi, ScanData
from .data_model import Whitefield
from .engine import SCAN_CACHE, to_host
from .recon import SearchWindow, UpdateOptions, _device_ref


@dataclass(frozen=True)
class SplitHalfResult:
    map_a: PixelMap
    map_b: PixelMap
    hist_edges: np.ndarray
    hist_ss: np.ndarray
    hist_fs: np.ndarray
    sigma: float


def split_half_recon(scan: ScanData, w: Whitefield, m: PixelMask, ref: ReferenceImage,
                     u: PixelMap, t: PixelTranslations, win: SearchWindow, seed: int = 0,
                     opts: UpdateOptions = UpdateOptions(integrate=False, sigma=0.0),
                     roi: Roi | None = None) -> SplitHalfResult:
    """Pixel-map uncertainty from two random halves of the samples
    (analysis.py:306-361): each (frame, pixel) sample goes to half A or B by a
    hash of its flat index, the map is refined once per half against the
    shared reference, and sigma is the robust spread of the differences
    divided by sqrt(2)."""
    seed64 = int(np.uint64(seed))                      # numpy's uint64 conversion rules
    ds = SCAN_CACHE.get(scan, w, m, roi)
    lib = ds.lib
    n, ss, fs = ds.n_frames, ds.ss, ds.fs
    u_t = ds.upload_u(u.u)
    di_t, dj_t = ds.upload_t(t.di, t.dj)
    dref = _device_ref(ref, ds)
    fw = torch.empty((n, ss, fs), dtype=torch.float32, device=ds.device)
    maps = []
    for half in (0, 1):                                # analysis.py:326-331
        check(lib.pxst_split_weights(seed64, n, ss, fs, half, fw.data_ptr(), stream_ptr()))
        u_h, _ = ds.pixel_map_search(dref, u_t, di_t, dj_t, win.half_ss, win.half_fs,
                                     win.subpixel_grid, opts.quadratic_refinement, fw)
        ds.regularise(u_h, opts)
        maps.append(PixelMap(to_host(u_h)))
    del fw
    counts_a = torch.zeros(ss * fs, dtype=torch.int32, device=ds.device)
    check(lib.pxst_split_counts(seed64, ds.good.data_ptr(), ds.n_good, ss, fs,
                                counts_a.data_ptr(), stream_ptr()))
    ca = to_host(counts_a).reshape(ss, fs)
    both = np.asarray(m.mask, dtype=bool) & (ca > 0) & ((ds.n_good - ca) > 0)   # :333-336
    if roi is not None:
        sel = np.zeros_like(both)
        sel[roi.slices] = True
        both &= sel
    d_ss = (maps[0].u[0] - maps[1].u[0])[both]
    d_fs = (maps[0].u[1] - maps[1].u[1])[both]
    edges = np.linspace(-2.0, 2.0, 82)
    h_ss, _ = np.histogram(d_ss, bins=edges)
    h_fs, _ = np.histogram(d_fs, bins=edges)
    pooled = np.concatenate([d_ss, d_fs])
    med = np.median(pooled)
    sigma = 1.4826 * float(np.median(np.abs(pooled - med))) / np.sqrt(2.0)
    return SplitHalfResult(map_a=maps[0], map_b=maps[1], hist_edges=edges, hist_ss=h_ss,
                           hist_fs=h_fs, sigma=sigma)

"""Drop-in of the reference's defocus search by registration contrast
(``pxst.geometry.fit_defocus_registration``, geometry.py:188-227), SURVEY 8(f)
row 4, with the small geometry helpers it calls (geometry.py:22-65).

Every candidate focus distance is one object formation (K1) on the GPU over
the resident stack (the scan is uploaded once, ``engine.SCAN_CACHE``); the
contrast var/mean^2 of the valid cells is reduced on the device and only C
scalars come back.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .data_model import Geometry, PixelMap, PixelMask, PixelTranslations, Roi, ScanData
from .data_model import Whitefield
from ._native import check, stream_ptr
from .engine import SCAN_CACHE


def make_geometry(z1_ss: float, z1_fs: float, scan: ScanData) -> Geometry:
    """Projection geometry of per-axis focus-to-sample distances (geometry.py:22-39)."""
    if z1_ss <= 0 or z1_fs <= 0:
        raise ValueError("focus-to-sample distance must be > 0")
    z = scan.distance
    m_ss = (z1_ss + z) / z1_ss
    m_fs = (z1_fs + z) / z1_fs
    return Geometry(z1_ss=z1_ss, z1_fs=z1_fs, z=z, mag_ss=m_ss, mag_fs=m_fs,
                    du=scan.x_pixel_size / m_ss, dv=scan.y_pixel_size / m_fs,
                    zbar_ss=z1_ss * z / (z1_ss + z), zbar_fs=z1_fs * z / (z1_fs + z))


def generate_pixel_map(geom: Geometry, shape, roi: Roi | None = None) -> PixelMap:
    """The identity map in reference units, full detector shape (geometry.py:42-50)."""
    return PixelMap.identity(shape)


def translations_to_pixels(scan: ScanData, geom: Geometry) -> PixelTranslations:
    """Translations projected on the detector axes in reference px (geometry.py:53-65)."""
    b = np.asarray(scan.basis_vectors[0], dtype=np.float64)
    e_ss = b[0] / np.linalg.norm(b[0])
    e_fs = b[1] / np.linalg.norm(b[1])
    tr = np.asarray(scan.translations, dtype=np.float64)
    return PixelTranslations(di=tr @ e_ss / geom.du, dj=tr @ e_fs / geom.dv)


@dataclass(frozen=True)
class DefocusFit:
    z1_ss: float
    z1_fs: float
    contrast: np.ndarray
    candidates: np.ndarray


def fit_defocus_registration(scan: ScanData, w: Whitefield, mask: PixelMask, z1_grid,
                             u_template: PixelMap | None = None, roi: Roi | None = None,
                             astigmatic: bool = False) -> DefocusFit:
    """Defocus maximising the normalised variance of the merged reference
    (geometry.py:188-227): one device object formation per candidate."""
    z1_grid = np.atleast_1d(np.asarray(z1_grid, dtype=np.float64))
    if z1_grid.size == 0:
        raise ValueError("z1 grid must be non-empty")
    if astigmatic:
        cands = np.array([(a, b) for a in z1_grid for b in z1_grid])
    else:
        cands = np.column_stack([z1_grid, z1_grid])
    ds = SCAN_CACHE.get(scan, w, mask, roi)
    if ds.empty:
        raise ValueError("make_reference: empty good pixel/frame set")
    stats = torch.zeros((len(cands), 3), dtype=torch.float64, device=ds.device)   # count, mean, var
    u_t = None
    for k, (za, zb) in enumerate(cands):
        geom = make_geometry(za, zb, scan)
        u = u_template or generate_pixel_map(geom, scan.shape, roi)
        if u_t is None or u_template is None:
            u_t = ds.upload_u(u.u)
        t = translations_to_pixels(scan, geom)
        di_t, dj_t = ds.upload_t(t.di, t.dj)
        ref = ds.object_map(u_t, di_t, dj_t)
        # mean and numpy-style variance (ddof 0) of the valid cells, on the device
        check(ds.lib.pxst_masked_moments(ref.i_ref.data_ptr(), ref.valid.data_ptr(),
                                         ref.i_ref.numel(), stats[k].data_ptr(), stream_ptr()))
    st = stats.cpu().numpy()[:, 1:]
    contrast = np.where(st[:, 0] != 0, st[:, 1] / np.where(st[:, 0] != 0, st[:, 0] ** 2, 1.0),
                        0.0)
    best = int(contrast.argmax())
    return DefocusFit(z1_ss=float(cands[best, 0]), z1_fs=float(cands[best, 1]),
                      contrast=contrast, candidates=cands)

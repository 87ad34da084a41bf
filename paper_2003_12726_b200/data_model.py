"""Value types crossing the drop-in boundary.

Field-for-field mirrors of the reference's frozen dataclasses
(``/root/reference/pkg/src/pxst/data_model.py:30-204``) so that code written
against ``pxst`` keeps working.  The hot-path functions in
:mod:`paper_2003_12726_b200.recon` only read attributes, so instances of the
reference's own classes are accepted unchanged (duck typing).

Conventions (``data_model.py:3-12``): axis order [slow-scan, fast-scan];
pixel maps and translations in reference-grid pixels; float64 in and out.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ScanData:
    """Frame stack ``[N, SS, FS]`` plus scan metadata (data_model.py:30-65)."""

    frames: np.ndarray
    wavelength: float
    distance: float
    x_pixel_size: float
    y_pixel_size: float
    basis_vectors: np.ndarray
    translations: np.ndarray
    good_frames: np.ndarray

    @property
    def n_frames(self) -> int:
        return self.frames.shape[0]

    @property
    def shape(self) -> tuple[int, int]:
        return self.frames.shape[1], self.frames.shape[2]

    def good_indices(self) -> np.ndarray:
        return np.flatnonzero(self.good_frames)


@dataclass(frozen=True)
class PixelMask:
    """Boolean detector mask, True = good pixel (data_model.py:68-72)."""

    mask: np.ndarray


@dataclass(frozen=True)
class Whitefield:
    """Whitefield counts ``[SS, FS]`` (data_model.py:75-79)."""

    w: np.ndarray


@dataclass(frozen=True)
class Roi:
    """Half-open detector rectangle (data_model.py:82-107)."""

    ss_min: int
    ss_max: int
    fs_min: int
    fs_max: int

    def __post_init__(self):
        if not (0 <= self.ss_min < self.ss_max and 0 <= self.fs_min < self.fs_max):
            raise ValueError(f"empty or negative ROI: {self}")

    @classmethod
    def full(cls, shape) -> "Roi":
        return cls(0, int(shape[0]), 0, int(shape[1]))

    @property
    def slices(self) -> tuple[slice, slice]:
        return slice(self.ss_min, self.ss_max), slice(self.fs_min, self.fs_max)

    def contains(self, shape) -> bool:
        return self.ss_max <= shape[0] and self.fs_max <= shape[1]

    def as_tuple(self) -> tuple[int, int, int, int]:
        return self.ss_min, self.ss_max, self.fs_min, self.fs_max


@dataclass(frozen=True)
class Geometry:
    """Separable projection geometry (data_model.py:110-128)."""

    z1_ss: float
    z1_fs: float
    z: float
    mag_ss: float
    mag_fs: float
    du: float
    dv: float
    zbar_ss: float
    zbar_fs: float


@dataclass(frozen=True)
class PixelMap:
    """Pixel map ``u [2, SS, FS]`` in reference-grid pixels (data_model.py:131-156)."""

    u: np.ndarray

    @property
    def shape(self) -> tuple[int, int]:
        return self.u.shape[1], self.u.shape[2]

    @classmethod
    def identity(cls, shape) -> "PixelMap":
        ss, fs = shape
        u = np.empty((2, ss, fs), dtype=np.float64)
        u[0] = np.arange(ss, dtype=np.float64)[:, None]
        u[1] = np.arange(fs, dtype=np.float64)[None, :]
        return cls(u)

    def displacement(self) -> np.ndarray:
        return self.u - PixelMap.identity(self.shape).u


@dataclass(frozen=True)
class PixelTranslations:
    """Per-frame translations in reference-grid pixels (data_model.py:159-167)."""

    di: np.ndarray
    dj: np.ndarray

    def __len__(self) -> int:
        return len(self.di)


@dataclass(frozen=True)
class ReferenceImage:
    """Merged reference (object) image (data_model.py:170-188).

    ``valid`` = ``wsum > 0``; ``origin = (n0, m0)`` is subtracted from
    ``u - delta`` to index ``i_ref``.
    """

    i_ref: np.ndarray
    wsum: np.ndarray
    origin: tuple[int, int]
    du: float
    dv: float

    @property
    def valid(self) -> np.ndarray:
        return self.wsum > 0


@dataclass(frozen=True)
class ErrorMetrics:
    """Residual decompositions (data_model.py:191-204)."""

    total: float
    per_frame: np.ndarray
    per_pixel: np.ndarray
    reference_plane: np.ndarray
    variance: np.ndarray

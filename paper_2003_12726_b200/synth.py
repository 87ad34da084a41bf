"""Seeded synthetic PXST scans for the BASELINE configs (tests and bench).

The reference measures on CXIDB 134-136 / HXN data, which are not in this
environment.  Seeded synthetic scans with the configs' shapes, sizes and
value laws stand in for them (BASELINE.json
``configs``).  The recipe follows the reference simulator's conventions
(``sim.py:86-120, 168-183``): centred rasters, Gaussian-filtered unit-std
noise clipped at 0.05, Gaussian whitefield with sigma = half the detector,
an 8-px object margin, frames rendered through a bilinear read of the object
at ``u_true - delta_true - origin``, Poisson counts stored as float32.

Config choices not fixed by BASELINE.json are written here (CONFIGS) and in
DESIGN.md.  Draw order for ``np.random.default_rng(cfg)``: jitter, object
noise, mask, Poisson, initial-u noise, translation noise.

Configs 0-2 are generated with numpy (bit-reproducible everywhere; config 0
and 1 goldens derive from them).  Configs 3-4 (8 GB / 4 GB stacks) render on
the GPU with torch when one is present, else on CPU torch, from a seeded
``torch.Generator``; the SAME arrays are then handed to both the oracle and
the kernels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .data_model import PixelMap, PixelMask, PixelTranslations, ScanData, Whitefield


@dataclass(frozen=True)
class ScanConfig:
    name: str
    n_ss: int                 # detector slow-scan size
    n_fs: int                 # detector fast-scan size
    positions: str            # "raster" | "fs_line" | "uniform"
    nx: int = 1               # raster size along ss
    ny: int = 1               # raster size along fs
    n_frames: int = 0         # for fs_line / uniform
    step: float = 1.0
    jitter: float = 0.0       # uniform +-jitter (px)
    field: float = 0.0        # uniform position field half-width (px)
    obj_sigma: float = 2.0
    obj_contrast: float = 0.3
    wf_kind: str = "gaussian"  # "gaussian" | "tophat"
    u_law: str = "quad"       # "quad" | "cubic" | "fs_only"
    bad_frac: float = 0.01
    u_noise: float = 1.0      # initial pixel-map noise U(+-u_noise)
    t_noise: float = 0.0      # translation noise: uniform half-width ...
    t_noise_kind: str = "none"  # "none" | "uniform" | "normal"
    half_ss: int = 3
    half_fs: int = 3
    subpixel_grid: float | None = None
    refine: bool = True
    iters: int = 1
    update_translations: bool = False
    t_half_ss: int = 0
    t_half_fs: int = 0
    t_subpixel_grid: float | None = None
    margin: int = 8
    update_pixel_map: bool = True


CONFIGS = {
    0: ScanConfig("cfg0-tiny-2d", 64, 128, "raster", nx=5, ny=5, step=4.0, jitter=0.5,
                  obj_sigma=2.0, obj_contrast=0.3, u_law="quad", half_ss=3, half_fs=3, iters=1),
    1: ScanConfig("cfg1-121x256x512", 256, 512, "raster", nx=11, ny=11, step=6.0, jitter=0.5,
                  obj_sigma=1.5, obj_contrast=0.4, u_law="cubic", half_ss=5, half_fs=5, iters=3),
    2: ScanConfig("cfg2-mll-1d-1000x516x1556", 516, 1556, "fs_line", n_frames=1000, step=1.5,
                  jitter=0.3, obj_sigma=1.5, obj_contrast=0.4, wf_kind="tophat",
                  u_law="fs_only", half_ss=0, half_fs=8, iters=5),
    3: ScanConfig("cfg3-2000x1024x1024", 1024, 1024, "raster", nx=40, ny=50, step=5.0, jitter=1.0,
                  obj_sigma=2.0, obj_contrast=0.3, u_law="cubic", t_noise=2.0,
                  t_noise_kind="uniform", half_ss=6, half_fs=6, iters=10,
                  update_translations=True, t_half_ss=3, t_half_fs=3),
    4: ScanConfig("cfg4-4000x512x512", 512, 512, "uniform", n_frames=4000, field=200.0,
                  obj_sigma=2.0, obj_contrast=0.3, u_law="cubic", u_noise=0.0, t_noise=1.5,
                  t_noise_kind="normal", half_ss=0, half_fs=0, iters=1,
                  update_translations=True, t_half_ss=4, t_half_fs=4, t_subpixel_grid=0.25,
                  update_pixel_map=False),
}

# Top-hat whitefield (config 2): plateau over the central 80% of each axis,
# Gaussian roll-off with sigma = 4% of the axis length outside it.
TOPHAT_PLATEAU = 0.8
TOPHAT_EDGE_SIGMA = 0.04


def _axis_law(x: np.ndarray, n: int, law: str) -> np.ndarray:
    c = (n - 1) / 2.0
    if law == "quad":
        return 0.8 * x + 2e-4 * (x - c) ** 2
    if law == "cubic":
        return 0.8 * x + 2e-4 * (x - c) ** 2 + 1e-6 * (x - c) ** 3
    if law == "fs_only":
        return 0.5 * x + 5e-5 * (x - c) ** 2 + 1e-7 * (x - c) ** 3
    raise ValueError(law)


def true_pixel_map(cfg: ScanConfig) -> np.ndarray:
    ss = np.arange(cfg.n_ss, dtype=np.float64)
    fs = np.arange(cfg.n_fs, dtype=np.float64)
    u = np.empty((2, cfg.n_ss, cfg.n_fs))
    if cfg.u_law == "fs_only":
        u[0] = ss[:, None]
        u[1] = _axis_law(fs, cfg.n_fs, "fs_only")[None, :]
    else:
        u[0] = _axis_law(ss, cfg.n_ss, cfg.u_law)[:, None]
        u[1] = _axis_law(fs, cfg.n_fs, cfg.u_law)[None, :]
    return u


def whitefield(cfg: ScanConfig) -> np.ndarray:
    if cfg.wf_kind == "gaussian":
        # sim.py:96-100 with whitefield_width = 1: sigma = half the detector.
        x = (np.arange(cfg.n_ss) - (cfg.n_ss - 1) / 2.0) / (cfg.n_ss / 2.0)
        y = (np.arange(cfg.n_fs) - (cfg.n_fs - 1) / 2.0) / (cfg.n_fs / 2.0)
        return 1000.0 * np.exp(-0.5 * (x[:, None] ** 2 + y[None, :] ** 2))

    def edge(n):
        t = np.abs(np.arange(n) - (n - 1) / 2.0) / n
        over = np.maximum(t - TOPHAT_PLATEAU / 2.0, 0.0)
        return np.exp(-0.5 * (over / TOPHAT_EDGE_SIGMA) ** 2)

    return 1000.0 * edge(cfg.n_ss)[:, None] * edge(cfg.n_fs)[None, :]


def positions(cfg: ScanConfig, rng) -> tuple[np.ndarray, np.ndarray]:
    if cfg.positions == "raster":
        ix = (np.arange(cfg.nx) - (cfg.nx - 1) / 2.0) * cfg.step
        iy = (np.arange(cfg.ny) - (cfg.ny - 1) / 2.0) * cfg.step
        di, dj = np.meshgrid(ix, iy, indexing="ij")
        di, dj = di.ravel(), dj.ravel()
        jit = rng.uniform(-cfg.jitter, cfg.jitter, size=(2, di.size))
        return di + jit[0], dj + jit[1]
    if cfg.positions == "fs_line":
        n = cfg.n_frames
        dj = (np.arange(n) - (n - 1) / 2.0) * cfg.step
        dj = dj + rng.uniform(-cfg.jitter, cfg.jitter, size=n)
        return np.zeros(n), dj
    if cfg.positions == "uniform":
        p = rng.uniform(-cfg.field, cfg.field, size=(2, cfg.n_frames))
        return p[0], p[1]
    raise ValueError(cfg.positions)


def _smooth_noise(shape, sigma, rng):
    from scipy.ndimage import gaussian_filter
    z = gaussian_filter(rng.standard_normal(shape), sigma)
    return z / max(z.std(), 1e-12)


def object_grid(u_true, di, dj, margin):
    """Object-grid origin/shape covering every frame (sim.py:168-173)."""
    n0 = int(math.floor(u_true[0].min() - di.max())) - margin
    m0 = int(math.floor(u_true[1].min() - dj.max())) - margin
    shape = (int(math.ceil(u_true[0].max() - di.min())) - n0 + 1 + margin,
             int(math.ceil(u_true[1].max() - dj.min())) - m0 + 1 + margin)
    return n0, m0, shape


def _bilinear(tex, x, y):
    """Plain bilinear read (every cell valid, points strictly inside)."""
    r0 = np.floor(x).astype(np.intp)
    c0 = np.floor(y).astype(np.intp)
    tx = x - r0
    ty = y - c0
    if r0.min() < 0 or c0.min() < 0 or r0.max() + 1 >= tex.shape[0] or c0.max() + 1 >= tex.shape[1]:
        raise ValueError("sample displacement exceeds the object extent")
    return ((1 - tx) * (1 - ty) * tex[r0, c0] + (1 - tx) * ty * tex[r0, c0 + 1]
            + tx * (1 - ty) * tex[r0 + 1, c0] + tx * ty * tex[r0 + 1, c0 + 1])


@dataclass
class SyntheticScan:
    cfg: ScanConfig
    scan: ScanData
    w: Whitefield
    m: PixelMask
    u0: PixelMap            # initial (perturbed) pixel map
    t0: PixelTranslations   # initial (perturbed) translations
    u_true: np.ndarray
    di_true: np.ndarray
    dj_true: np.ndarray
    obj: np.ndarray
    obj_origin: tuple


def _scan_record(frames, n):
    return ScanData(frames=frames, wavelength=5e-10, distance=1.0, x_pixel_size=1e-5,
                    y_pixel_size=1e-5, basis_vectors=np.tile(np.array([[1e-5, 0, 0], [0, 1e-5, 0]]),
                                                             (n, 1, 1)),
                    translations=np.zeros((n, 3)), good_frames=np.ones(n, dtype=bool))


def make_scan_device(cfg_id: int | ScanConfig, device, seed: int | None = None,
                     frame_chunk: int = 64):
    """Configs 3-4 scale: same recipe, frames rendered and Poisson-sampled on
    `device` with a seeded torch.Generator (the numpy draws for positions,
    object, mask and initial state keep the documented order).  Returns
    ``(SyntheticScan with scan.frames=None, frames_dev [N,SS,FS] float32)``."""
    import torch
    cfg = CONFIGS[cfg_id] if isinstance(cfg_id, int) else cfg_id
    seed = (cfg_id if isinstance(cfg_id, int) else 0) if seed is None else seed
    rng = np.random.default_rng(seed)
    di, dj = positions(cfg, rng)
    u_true = true_pixel_map(cfg)
    n0, m0, oshape = object_grid(u_true, di, dj, cfg.margin)
    obj = np.clip(1.0 + cfg.obj_contrast * _smooth_noise(oshape, cfg.obj_sigma, rng), 0.05, None)
    mask = rng.random((cfg.n_ss, cfg.n_fs)) >= cfg.bad_frac
    wf = whitefield(cfg)
    n = di.size
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed) + 1000)
    tex = torch.as_tensor(obj, device=device)
    u0 = torch.as_tensor(u_true[0], device=device)
    u1 = torch.as_tensor(u_true[1], device=device)
    W = torch.as_tensor(wf, device=device)
    frames = torch.empty((n, cfg.n_ss, cfg.n_fs), dtype=torch.float32, device=device)
    of = oshape[1]
    flat = tex.reshape(-1)
    for k0 in range(0, n, frame_chunk):
        k1 = min(n, k0 + frame_chunk)
        dI = torch.as_tensor(di[k0:k1], device=device)[:, None, None]
        dJ = torch.as_tensor(dj[k0:k1], device=device)[:, None, None]
        x = u0[None] - dI - n0
        y = u1[None] - dJ - m0
        r0 = torch.floor(x)
        c0 = torch.floor(y)
        tx, ty = x - r0, y - c0
        r0 = r0.long()
        c0 = c0.long()
        if int(r0.min()) < 0 or int(c0.min()) < 0 or int(r0.max()) + 1 >= oshape[0] or \
                int(c0.max()) + 1 >= of:
            raise ValueError("sample displacement exceeds the object extent")
        i00 = r0 * of + c0
        v = ((1 - tx) * (1 - ty) * flat[i00] + (1 - tx) * ty * flat[i00 + 1]
             + tx * (1 - ty) * flat[i00 + of] + tx * ty * flat[i00 + of + 1])
        frames[k0:k1] = torch.poisson(W[None] * v, generator=gen).float()
    u_init = u_true.copy()
    if cfg.u_noise > 0:
        noise = rng.uniform(-cfg.u_noise, cfg.u_noise, size=u_true.shape)
        if cfg.u_law == "fs_only":
            noise[0] = 0.0
        u_init = u_true + noise
    di0, dj0 = di.copy(), dj.copy()
    if cfg.t_noise_kind == "uniform":
        tn = rng.uniform(-cfg.t_noise, cfg.t_noise, size=(2, n))
        di0, dj0 = di + tn[0], dj + tn[1]
    elif cfg.t_noise_kind == "normal":
        tn = rng.normal(0.0, cfg.t_noise, size=(2, n))
        di0, dj0 = di + tn[0], dj + tn[1]
    rec = _scan_record(None, n)
    s = SyntheticScan(cfg=cfg, scan=rec, w=Whitefield(wf), m=PixelMask(mask), u0=PixelMap(u_init),
                      t0=PixelTranslations(di0, dj0), u_true=u_true, di_true=di, dj_true=dj,
                      obj=obj, obj_origin=(n0, m0))
    return s, frames


def make_scan(cfg_id: int | ScanConfig, seed: int | None = None) -> SyntheticScan:
    """Generate the seeded scan of one config (numpy; exact everywhere)."""
    cfg = CONFIGS[cfg_id] if isinstance(cfg_id, int) else cfg_id
    seed = (cfg_id if isinstance(cfg_id, int) else 0) if seed is None else seed
    rng = np.random.default_rng(seed)
    di, dj = positions(cfg, rng)                                  # 1. jitter
    u_true = true_pixel_map(cfg)
    n0, m0, oshape = object_grid(u_true, di, dj, cfg.margin)
    obj = np.clip(1.0 + cfg.obj_contrast * _smooth_noise(oshape, cfg.obj_sigma, rng),
                  0.05, None)                                     # 2. object noise
    mask = rng.random((cfg.n_ss, cfg.n_fs)) >= cfg.bad_frac       # 3. mask
    wf = whitefield(cfg)
    n = di.size
    frames = np.empty((n, cfg.n_ss, cfg.n_fs), dtype=np.float32)
    for k in range(n):                                            # 4. Poisson
        lam = wf * _bilinear(obj, u_true[0] - di[k] - n0, u_true[1] - dj[k] - m0)
        frames[k] = rng.poisson(lam).astype(np.float32)
    u_init = u_true.copy()
    if cfg.u_noise > 0:                                           # 5. initial-u noise
        noise = rng.uniform(-cfg.u_noise, cfg.u_noise, size=u_true.shape)
        if cfg.u_law == "fs_only":
            noise[0] = 0.0
        u_init = u_true + noise
    di0, dj0 = di.copy(), dj.copy()
    if cfg.t_noise_kind == "uniform":                             # 6. translation noise
        tn = rng.uniform(-cfg.t_noise, cfg.t_noise, size=(2, n))
        di0, dj0 = di + tn[0], dj + tn[1]
    elif cfg.t_noise_kind == "normal":
        tn = rng.normal(0.0, cfg.t_noise, size=(2, n))
        di0, dj0 = di + tn[0], dj + tn[1]
    return SyntheticScan(cfg=cfg, scan=_scan_record(frames, n), w=Whitefield(wf),
                         m=PixelMask(mask), u0=PixelMap(u_init), t0=PixelTranslations(di0, dj0),
                         u_true=u_true, di_true=di, dj_true=dj, obj=obj, obj_origin=(n0, m0))

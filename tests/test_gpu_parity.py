"""GPU parity: the sm_100a kernels (through the drop-in API / C ABI) against the
live-reference golden vectors and the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star):
  * object map within 1e-5 relative on cells with wsum > 0, identical
    validity masks and origin;
  * integer argmin indices bit-exact wherever the argmin is unique
    (relative best/second-best margin > 1e-4 in the oracle's normalised
    errors);
  * pixel map within 1e-3 px on those pixels;
  * translations within 1e-3 px.
Float sums (errors) are compared at 1e-4 relative (fp32 accumulation).
"""

from __future__ import annotations

import os
from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2003_12726_b200 as pb  # noqa: E402
from oracle import pxst_oracle as orc  # noqa: E402
from conftest import GOLDEN  # noqa: E402

OBJ_RTOL = 1e-5
PX_TOL = 1e-3
MARGIN = 1e-4


def ref_from(g, prefix="ref"):
    return pb.ReferenceImage(i_ref=g[f"{prefix}_i"], wsum=g[f"{prefix}_w"],
                             origin=tuple(int(v) for v in g[f"{prefix}_origin"]), du=1.0, dv=1.0)


def assert_object_map(ref, i_ref, wsum, origin):
    assert tuple(ref.origin) == tuple(origin)
    assert ref.i_ref.shape == i_ref.shape
    ok = wsum > 0
    np.testing.assert_array_equal(ref.wsum > 0, ok)
    rel = np.abs(ref.i_ref[ok] - i_ref[ok]) / np.maximum(np.abs(i_ref[ok]), 1e-300)
    assert rel.max() < OBJ_RTOL, rel.max()
    np.testing.assert_array_equal(ref.i_ref[~ok], 0.0)
    relw = np.abs(ref.wsum[ok] - wsum[ok]) / wsum[ok]
    assert relw.max() < OBJ_RTOL, relw.max()


def unique_pixels(stack):
    """Pixels whose oracle argmin is unique by a relative margin > MARGIN."""
    P = stack.shape[-1]
    flat = stack.reshape(-1, P)
    part = np.partition(flat, 1, axis=0)
    best, second = part[0], part[1]
    return (second - best) > MARGIN * np.abs(best)


def oracle_pixel_map(s, ref, u, di, dj, half, refine=True, roi=None, sub=None, fw=None):
    return orc.update_pixel_map(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask, ref.i_ref,
                                ref.wsum, ref.origin, u, di, dj, half[0], half[1], sub, refine,
                                roi, fw, threads=os.cpu_count() or 1, return_stack=True)


def assert_pixel_map(u_gpu, e_gpu, u_orc, e_orc, stack, rows, cols, u_in, refine):
    uniq = unique_pixels(stack)
    assert uniq.mean() > 0.97, uniq.mean()
    gu = u_gpu[:, rows, cols]
    ou = u_orc[:, rows, cols]
    if not refine:
        # integer offsets: bit-exact argmin
        np.testing.assert_array_equal(gu[:, uniq], ou[:, uniq])
    d = np.abs(gu - ou).max(axis=0)
    assert d[uniq].max() < PX_TOL, d[uniq].max()
    eo = e_orc[rows, cols][uniq]
    eg = e_gpu[rows, cols][uniq]
    assert np.max(np.abs(eg - eo) / np.maximum(np.abs(eo), 1e-12)) < 1e-4
    # untouched pixels copied verbatim
    mask = np.ones(u_in.shape[1:], dtype=bool)
    mask[rows, cols] = False
    np.testing.assert_array_equal(u_gpu[:, mask], u_in[:, mask])
    np.testing.assert_array_equal(e_gpu[mask], 0.0)


def work_rc(s, roi=None):
    W, M = s.w.w, s.m.mask
    r0, r1, c0, c1 = roi or (0, W.shape[0], 0, W.shape[1])
    sub = M[r0:r1, c0:c1] & (W[r0:r1, c0:c1] > 0)
    r, c = np.nonzero(sub)
    return r + r0, c + c0


# ---------------------------------------------------------------------------
# config 0 against the live-reference golden vectors
# ---------------------------------------------------------------------------
def test_cfg0_object_map(scan0, golden0):
    s = scan0
    ref = pb.make_reference(s.scan, s.w, s.m, s.u0, s.t0)
    assert_object_map(ref, golden0["ref_i"], golden0["ref_w"], golden0["ref_origin"])
    ref2 = pb.make_object_map(s.scan, s.w, s.m, s.u0, s.t0)
    # float32 chunk images, unordered REDs: run-to-run differences ~1e-7
    np.testing.assert_allclose(ref.i_ref, ref2.i_ref, rtol=OBJ_RTOL)
    np.testing.assert_allclose(ref.wsum, ref2.wsum, rtol=OBJ_RTOL)


@pytest.mark.parametrize("refine", [True, False])
def test_cfg0_pixel_map(scan0, golden0, refine):
    s = scan0
    ref = ref_from(golden0)
    u, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(3, 3),
                               pb.UpdateOptions(quadratic_refinement=refine))
    uo, eo, stack = oracle_pixel_map(s, ref, s.u0.u, s.t0.di, s.t0.dj, (3, 3), refine)
    key = "upm_u" if refine else "upm_noref_u"
    np.testing.assert_array_equal(uo, golden0[key])
    r, c = work_rc(s)
    assert_pixel_map(u.u, e, uo, eo, stack, r, c, s.u0.u, refine)


def test_cfg0_translations(scan0, golden0):
    s = scan0
    ref = ref_from(golden0)
    U = pb.PixelMap(golden0["upm_u"])
    T = pb.update_translations(s.scan, s.w, s.m, ref, U, s.t0, pb.SearchWindow(2, 2))
    assert np.abs(T.di - golden0["ut_di"]).max() < PX_TOL
    assert np.abs(T.dj - golden0["ut_dj"]).max() < PX_TOL
    T2 = pb.update_translations(s.scan, s.w, s.m, ref, U, s.t0,
                                pb.SearchWindow(1, 1, subpixel_grid=0.5))
    assert np.abs(T2.di - golden0["uts_di"]).max() < PX_TOL
    assert np.abs(T2.dj - golden0["uts_dj"]).max() < PX_TOL


@pytest.mark.parametrize("half,step", [(3, None), (4, 0.25)])
def test_cfg0_translation_windows(scan0, golden0, half, step):
    """The config-3 (+-3 integer) and config-4 (+-4 at 0.25 px: 16 phase groups
    9x9/9x8/8x9/8x8) translation searches against the oracle, incl. the
    always-on refinement quirk."""
    s = scan0
    ref = ref_from(golden0)
    U = pb.PixelMap(golden0["upm_u"])
    good = np.zeros(s.scan.n_frames, bool)
    good[[0, 7, 12, 24]] = True                       # frame subset keeps the oracle fast
    sc = replace(s.scan, good_frames=good)
    T = pb.update_translations(sc, s.w, s.m, ref, U, s.t0, pb.SearchWindow(half, half, step))
    di, dj, errs = orc.update_translations(sc.frames, good, s.w.w, s.m.mask, ref.i_ref, ref.wsum,
                                           ref.origin, U.u, s.t0.di, s.t0.dj, half, half, step,
                                           return_errors=True)
    for fr, e in errs.items():
        flat = np.sort(e.ravel())
        if (flat[1] - flat[0]) > MARGIN * abs(flat[0]):   # unique argmin
            assert abs(T.di[fr] - di[fr]) < PX_TOL and abs(T.dj[fr] - dj[fr]) < PX_TOL, fr
    np.testing.assert_array_equal(T.di[~good], s.t0.di[~good])


def test_cfg0_error_maps(scan0, golden0):
    s = scan0
    ref = ref_from(golden0)
    U = pb.PixelMap(golden0["upm_u"])
    T = pb.PixelTranslations(golden0["ut_di"], golden0["ut_dj"])
    M = pb.calc_error(s.scan, s.w, s.m, ref, U, T)
    g = golden0
    assert abs(M.total - float(g["ce_total"])) <= 1e-5 * abs(float(g["ce_total"]))
    # float64 residuals in K4: agreement to ~1e-12
    np.testing.assert_allclose(M.per_frame, g["ce_per_frame"], rtol=1e-10)
    np.testing.assert_allclose(M.per_pixel, g["ce_per_pixel"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(M.variance, g["ce_var"], rtol=1e-12)
    # reference plane: float32 grouped chunk images + float64 fold (error.cu header)
    np.testing.assert_allclose(M.reference_plane, g["ce_plane"], rtol=1e-5, atol=1e-12)


def test_cfg0_main_loop(scan0, golden0):
    s = scan0
    sched = [pb.IterationSettings(window=pb.SearchWindow(3, 3),
                                  options=pb.UpdateOptions(True, False, 0.0),
                                  update_translations=True,
                                  translation_window=pb.SearchWindow(1, 1))]
    L = pb.run_main_loop(s.scan, s.w, s.m, s.u0, s.t0, schedule=sched, max_iters=2, tol=-np.inf)
    g = golden0
    # north-star bars on the pixels whose argmin is unique in both iterations
    # of the reference's trajectory (tests/golden/make_golden_loop.py:
    # loop0.npz; every frame's is)
    np.testing.assert_allclose([h.total for h in L.history], g["loop_hist"], rtol=1e-5)
    g2 = np.load(os.path.join(GOLDEN, "loop0.npz"))
    robust = np.unpackbits(g2["robust_px"])[:s.w.w.size].reshape(s.w.w.shape).astype(bool)
    d = np.abs(L.pixel_map.u - g["loop_u"]).max(axis=0)
    assert d[robust].max() < PX_TOL, d[robust].max()
    assert np.abs(L.translations.di - g["loop_di"]).max() < PX_TOL
    assert np.abs(L.translations.dj - g["loop_dj"]).max() < PX_TOL
    assert tuple(L.reference.origin) == tuple(g["loop_ref_origin"])


# ---------------------------------------------------------------------------
# config 1 (121 frames, 256x512, R=5) against golden slices
# ---------------------------------------------------------------------------
def test_cfg1_object_map(scan1, golden1):
    s = scan1
    ref = pb.make_reference(s.scan, s.w, s.m, s.u0, s.t0)
    assert_object_map(ref, golden1["ref_i"], golden1["ref_w"], golden1["ref_origin"])


def test_cfg1_pixel_map_band(scan1, golden1):
    s = scan1
    g = golden1
    ref = ref_from(g)
    band = tuple(int(v) for v in g["band"])
    roi = pb.Roi(*band)
    u, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(5, 5), roi=roi)
    uo, eo, stack = oracle_pixel_map(s, ref, s.u0.u, s.t0.di, s.t0.dj, (5, 5), True, band)
    np.testing.assert_array_equal(uo[:, band[0]:band[1]], g["upm_u"])
    r, c = work_rc(s, band)
    assert_pixel_map(u.u, e, uo, eo, stack, r, c, s.u0.u, True)
    # the full-frame run agrees with the band run on the band (row independence;
    # frame chunking may differ, so to float32 summation order)
    uf, ef = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(5, 5))
    d = np.abs(uf.u[:, r, c] - u.u[:, r, c]).max(axis=0)
    assert d[unique_pixels(stack)].max() < PX_TOL
    np.testing.assert_allclose(ef[band[0]:band[1]], e[band[0]:band[1]], rtol=1e-5, atol=1e-12)


@pytest.mark.parametrize("band", [(0, 8), (248, 256)])
@pytest.mark.parametrize("refine", [False, True])
def test_cfg1_full_frame_work_units(scan1, golden1, band, refine):
    """The full-frame config-1 search (whole-tile units finished inside
    k_pix_fast or, for pixels with skipped samples, inside k_pix_slow; the last
    partial wave's tiles frame-split through the epilogue) against the oracle
    on the top rows (whole-tile units, grid-edge slow samples) and the bottom
    rows (frame-split units)."""
    s = scan1
    ref = ref_from(golden1)
    u, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(5, 5),
                               pb.UpdateOptions(quadratic_refinement=refine))
    roi = (band[0], band[1], 0, s.w.w.shape[1])
    uo, eo, stack = oracle_pixel_map(s, ref, s.u0.u, s.t0.di, s.t0.dj, (5, 5), refine, roi)
    r, c = work_rc(s, roi)
    uniq = unique_pixels(stack)
    assert uniq.mean() > 0.97, uniq.mean()
    gu, ou = u.u[:, r, c], uo[:, r, c]
    if not refine:
        np.testing.assert_array_equal(gu[:, uniq], ou[:, uniq])
    assert np.abs(gu - ou).max(axis=0)[uniq].max() < PX_TOL
    eg, eo_ = e[r, c][uniq], eo[r, c][uniq]
    assert np.max(np.abs(eg - eo_) / np.maximum(np.abs(eo_), 1e-12)) < 1e-4


def test_cfg1_translation_subset(scan1, golden1):
    s = scan1
    g = golden1
    ref = ref_from(g)
    sc = replace(s.scan, good_frames=g["ut_subset"])
    T = pb.update_translations(sc, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(3, 3))
    assert np.abs(T.di - g["ut_di"]).max() < PX_TOL
    assert np.abs(T.dj - g["ut_dj"]).max() < PX_TOL
    np.testing.assert_array_equal(T.di[~g["ut_subset"]], s.t0.di[~g["ut_subset"]])


def test_cfg1_error_band(scan1, golden1):
    s = scan1
    g = golden1
    ref = ref_from(g)
    band = tuple(int(v) for v in g["band"])
    M = pb.calc_error(s.scan, s.w, s.m, ref, s.u0, s.t0, roi=pb.Roi(*band))
    np.testing.assert_allclose(M.per_pixel[band[0]:band[1]], g["ce_per_pixel"], rtol=1e-4,
                               atol=1e-9)
    np.testing.assert_allclose(M.variance[band[0]:band[1]], g["ce_var"], rtol=1e-12)
    np.testing.assert_allclose(M.per_frame, g["ce_per_frame"], rtol=1e-5)
    assert abs(M.total - float(g["ce_total"])) <= 1e-5 * float(g["ce_total"])


# ---------------------------------------------------------------------------
# generic (any window / sub-pixel) kernels agree with the specialised ones
# ---------------------------------------------------------------------------
def test_generic_kernels_agree(scan0, golden0, monkeypatch):
    s = scan0
    ref = ref_from(golden0)
    u1, e1 = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(3, 3))
    t1 = pb.update_translations(s.scan, s.w, s.m, ref, u1, s.t0, pb.SearchWindow(2, 2))
    monkeypatch.setenv("PXST_FORCE_GENERIC", "1")
    u2, e2 = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(3, 3))
    t2 = pb.update_translations(s.scan, s.w, s.m, ref, u1, s.t0, pb.SearchWindow(2, 2))
    d = np.abs(u1.u - u2.u).max(axis=0)
    assert np.mean(d < PX_TOL) > 0.999
    assert np.abs(t1.di - t2.di).max() < PX_TOL


def test_subpixel_pixel_map_grid(scan0, golden0):
    s = scan0
    ref = ref_from(golden0)
    win = pb.SearchWindow(1, 1, subpixel_grid=0.5)
    u, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, win)
    uo, eo, stack = oracle_pixel_map(s, ref, s.u0.u, s.t0.di, s.t0.dj, (1, 1), True, sub=0.5)
    r, c = work_rc(s)
    uniq = unique_pixels(stack)
    np.testing.assert_array_equal(u.u[:, r, c][:, uniq], uo[:, r, c][:, uniq])


@pytest.mark.parametrize("half,step", [(1, 0.4), (2, 0.8)])
def test_subpixel_grid_round_half_even(scan0, golden0, half, step):
    """half/step = 2.5: the reference's round() gives k = 2 (ties to even,
    recon.py:55), i.e. 5 offsets per axis, not 7.  Pixel map (K2
    generic) and translations (K3 generic) against the oracle."""
    s = scan0
    ref = ref_from(golden0)
    win = pb.SearchWindow(half, half, subpixel_grid=step)
    assert len(win.offsets(0)) == 5
    u, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, win)
    uo, eo, stack = oracle_pixel_map(s, ref, s.u0.u, s.t0.di, s.t0.dj, (half, half), True,
                                     sub=step)
    assert stack.shape[:2] == (5, 5)
    r, c = work_rc(s)
    uniq = unique_pixels(stack)
    np.testing.assert_array_equal(u.u[:, r, c][:, uniq], uo[:, r, c][:, uniq])
    good = np.zeros(s.scan.n_frames, bool)
    good[[1, 9, 20]] = True
    sc = replace(s.scan, good_frames=good)
    U = pb.PixelMap(golden0["upm_u"])
    T = pb.update_translations(sc, s.w, s.m, ref, U, s.t0, win)
    di, dj, errs = orc.update_translations(sc.frames, good, s.w.w, s.m.mask, ref.i_ref, ref.wsum,
                                           ref.origin, U.u, s.t0.di, s.t0.dj, half, half, step,
                                           return_errors=True)
    for fr, e3 in errs.items():
        assert e3.shape == (5, 5)
        flat = np.sort(e3.ravel())
        if (flat[1] - flat[0]) > MARGIN * abs(flat[0]):
            assert abs(T.di[fr] - di[fr]) < PX_TOL and abs(T.dj[fr] - dj[fr]) < PX_TOL, fr


def test_large_translation_window(scan0, golden0):
    """SearchWindow(40, 40): 6561 trials per frame, more than the epilogue's
    former shared-memory copy held; one frame against the oracle."""
    s = scan0
    ref = ref_from(golden0)
    win = pb.SearchWindow(40, 40)
    good = np.zeros(s.scan.n_frames, bool)
    good[12] = True
    sc = replace(s.scan, good_frames=good)
    U = pb.PixelMap(golden0["upm_u"])
    T = pb.update_translations(sc, s.w, s.m, ref, U, s.t0, win)
    di, dj = orc.update_translations(sc.frames, good, s.w.w, s.m.mask, ref.i_ref, ref.wsum,
                                     ref.origin, U.u, s.t0.di, s.t0.dj, 40, 40)
    assert abs(T.di[12] - di[12]) < PX_TOL and abs(T.dj[12] - dj[12]) < PX_TOL


def test_one_dimensional_window(scan0, golden0):
    """Config-2 style SearchWindow(0, 8): integer shifts only."""
    s = scan0
    ref = ref_from(golden0)
    u, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(0, 4))
    uo, eo, stack = oracle_pixel_map(s, ref, s.u0.u, s.t0.di, s.t0.dj, (0, 4), True)
    r, c = work_rc(s)
    uniq = unique_pixels(stack)
    np.testing.assert_array_equal(u.u[:, r, c][:, uniq], uo[:, r, c][:, uniq])
    np.testing.assert_array_equal(u.u[0], s.u0.u[0])


# ---------------------------------------------------------------------------
# edge cases the reference handles without raising
# ---------------------------------------------------------------------------
def _tiny(seed=3, n=6, ss=24, fs=28):
    rng = np.random.default_rng(seed)
    ref_shape = (ss + 20, fs + 20)
    obj = 1 + 0.3 * rng.standard_normal(ref_shape)
    W = 500.0 + 100 * rng.random((ss, fs))
    di = rng.uniform(-3, 3, n)
    dj = rng.uniform(-3, 3, n)
    u = pb.PixelMap.identity((ss, fs)).u.copy()
    u += rng.uniform(-0.5, 0.5, u.shape)
    frames = np.empty((n, ss, fs), np.float32)
    for k in range(n):
        v, ok = orc.masked_sample(obj, np.ones(ref_shape, bool), u[0] - di[k] + 8, u[1] - dj[k] + 8)
        frames[k] = rng.poisson(W * v)
    sc = pb.ScanData(frames, 1e-10, 1.0, 1e-5, 1e-5, np.zeros((n, 2, 3)), np.zeros((n, 3)),
                     np.ones(n, bool))
    return sc, pb.Whitefield(W), pb.PixelMask(np.ones((ss, fs), bool)), pb.PixelMap(u), \
        pb.PixelTranslations(di, dj)


def _orc_args(sc, w, m):
    return sc.frames, sc.good_frames, w.w, m.mask


def test_static_pixels_and_zero_variance_frames():
    sc, w, m, u, t = _tiny()
    frames = sc.frames.copy()
    frames[:, 5, 7] = np.float32(w.w[5, 7])        # static pixel: var_pm == 0
    W = w.w.copy()
    W[5, 7] = float(frames[0, 5, 7])
    frames[2] = W.astype(np.float32)               # frame with zero normaliser
    W = W.astype(np.float32).astype(np.float64)
    sc = replace(sc, frames=frames)
    w = pb.Whitefield(W)
    ref = pb.make_reference(sc, w, m, u, t)
    un, e = pb.update_pixel_map(sc, w, m, ref, u, t, pb.SearchWindow(2, 2))
    assert un.u[0, 5, 7] == u.u[0, 5, 7] and un.u[1, 5, 7] == u.u[1, 5, 7] and e[5, 7] == 0.0
    T = pb.update_translations(sc, w, m, ref, un, t, pb.SearchWindow(1, 1))
    di, dj = orc.update_translations(*_orc_args(sc, w, m), ref.i_ref, ref.wsum, ref.origin, un.u,
                                     t.di, t.dj, 1, 1)
    assert T.di[2] == t.di[2] and T.dj[2] == t.dj[2]
    assert np.abs(T.di - di).max() < PX_TOL


def test_invalid_reference_cells():
    sc, w, m, u, t = _tiny(seed=5)
    ref = pb.make_reference(sc, w, m, u, t)
    wsum = ref.wsum.copy()
    wsum[10:14, 9:20] = 0.0                          # a hole of invalid cells
    i_ref = np.where(wsum > 0, ref.i_ref, 0.0)
    hole = pb.ReferenceImage(i_ref, wsum, ref.origin, 1.0, 1.0)
    un, e = pb.update_pixel_map(sc, w, m, hole, u, t, pb.SearchWindow(2, 2))
    uo, eo, stack = orc.update_pixel_map(*_orc_args(sc, w, m), i_ref, wsum, ref.origin, u.u, t.di,
                                         t.dj, 2, 2, return_stack=True)
    uniq = unique_pixels(stack)
    r, c = np.nonzero(np.ones(w.w.shape, bool))
    d = np.abs(un.u[:, r, c] - uo[:, r, c]).max(axis=0)
    assert d[uniq].max() < PX_TOL
    M = pb.calc_error(sc, w, m, hole, un, t)
    d = orc.calc_error(*_orc_args(sc, w, m), i_ref, wsum, ref.origin, un.u, t.di, t.dj)
    assert abs(M.total - d["total"]) < 1e-5 * d["total"]
    np.testing.assert_allclose(M.per_pixel, d["per_pixel"], rtol=1e-4, atol=1e-9)


def test_all_invalid_reference_ties_to_first_index():
    sc, w, m, u, t = _tiny(seed=7)
    ref = pb.make_reference(sc, w, m, u, t)
    dead = pb.ReferenceImage(np.zeros_like(ref.i_ref), np.zeros_like(ref.wsum), ref.origin, 1, 1)
    un, e = pb.update_pixel_map(sc, w, m, dead, u, t, pb.SearchWindow(2, 1))
    np.testing.assert_allclose(un.u[0] - u.u[0], -2.0)
    np.testing.assert_allclose(un.u[1] - u.u[1], -1.0)
    T = pb.update_translations(sc, w, m, dead, u, t, pb.SearchWindow(2, 2))
    np.testing.assert_allclose(T.di - t.di, -2.0)


def test_empty_work_set_raises():
    sc, w, m, u, t = _tiny()
    with pytest.raises(ValueError):
        pb.make_reference(sc, w, pb.PixelMask(np.zeros_like(m.mask)), u, t)
    with pytest.raises(ValueError):
        pb.SearchWindow(-1, 2)
    with pytest.raises(ValueError):
        pb.SearchWindow(1, 1, subpixel_grid=2.0)
    # integrate on an empty support: the reference's integrate_gradient ValueError
    ref = pb.make_reference(sc, w, m, u, t)
    with pytest.raises(ValueError):
        pb.update_pixel_map(sc, w, pb.PixelMask(np.zeros_like(m.mask)), ref, u, t,
                            pb.SearchWindow(1, 1), pb.UpdateOptions(integrate=True))


def test_frame_weights():
    sc, w, m, u, t = _tiny(seed=11)
    ref = pb.make_reference(sc, w, m, u, t)
    rng = np.random.default_rng(0)
    fw = (rng.random(sc.frames.shape) > 0.5).astype(np.float64)
    un, e = pb.update_pixel_map(sc, w, m, ref, u, t, pb.SearchWindow(2, 2), frame_weights=fw)
    uo, eo, stack = orc.update_pixel_map(*_orc_args(sc, w, m), ref.i_ref, ref.wsum, ref.origin,
                                         u.u, t.di, t.dj, 2, 2, frame_weights=fw,
                                         return_stack=True)
    uniq = unique_pixels(stack)
    r, c = np.nonzero(np.ones(w.w.shape, bool))
    d = np.abs(un.u[:, r, c] - uo[:, r, c]).max(axis=0)
    assert d[uniq].max() < PX_TOL


def test_roi_and_bad_frames():
    sc, w, m, u, t = _tiny(seed=13, n=8)
    good = np.ones(8, bool)
    good[[1, 6]] = False
    sc = replace(sc, good_frames=good)
    roi = pb.Roi(3, 20, 2, 25)
    ref = pb.make_reference(sc, w, m, u, t, roi=roi)
    i_ref, wsum, org = orc.make_object_map(*_orc_args(sc, w, m), u.u, t.di, t.dj,
                                           roi=roi.as_tuple())
    assert_object_map(ref, i_ref, wsum, org)
    M = pb.calc_error(sc, w, m, ref, u, t, roi=roi)
    d = orc.calc_error(*_orc_args(sc, w, m), ref.i_ref, ref.wsum, ref.origin, u.u, t.di, t.dj,
                       roi=roi.as_tuple())
    np.testing.assert_allclose(M.per_frame, d["per_frame"], rtol=1e-5)
    assert M.per_frame[1] == 0.0 and M.per_frame[6] == 0.0


@pytest.mark.parametrize("half", [1, 2, 4, 6])
def test_shifted_map_matches_oracle(half):
    """A uniformly shifted map (SPEC.md:375 setting) searched with every square
    kernel instantiation: integer argmins bit-exact vs the oracle."""
    sc, w, m, u, t = _tiny(seed=17)
    ref = pb.make_reference(sc, w, m, u, t)
    shifted = pb.PixelMap(u.u - np.array([2.0, -1.0])[:, None, None])
    un, e = pb.update_pixel_map(sc, w, m, ref, shifted, t, pb.SearchWindow(half, half),
                                pb.UpdateOptions(quadratic_refinement=False))
    uo, eo, stack = orc.update_pixel_map(*_orc_args(sc, w, m), ref.i_ref, ref.wsum, ref.origin,
                                         shifted.u, t.di, t.dj, half, half,
                                         quadratic_refinement=False, return_stack=True)
    uniq = unique_pixels(stack).reshape(w.w.shape)
    np.testing.assert_array_equal(un.u[:, uniq], uo[:, uniq])


def test_spec_uniform_shift_recovered(scan0):
    """frames rendered from the true map, true reference; the
    map shifted by a uniform +2 px is recovered by a +-4 integer search on
    the interior (where the shifted window stays inside the object)."""
    s = scan0
    obj_ref = pb.ReferenceImage(s.obj, np.ones_like(s.obj), s.obj_origin, 1.0, 1.0)
    t = pb.PixelTranslations(s.di_true, s.dj_true)
    shifted = pb.PixelMap(s.u_true - 2.0)
    un, e = pb.update_pixel_map(s.scan, s.w, s.m, obj_ref, shifted, t, pb.SearchWindow(4, 4),
                                pb.UpdateOptions(quadratic_refinement=False))
    good = s.m.mask
    frac = np.mean(np.abs(un.u - s.u_true).max(axis=0)[good] < 1e-9)
    assert frac > 0.99, frac


def test_interp_primitives():
    from paper_2003_12726_b200 import interp
    rng = np.random.default_rng(1)
    f = rng.random((9, 11))
    msk = rng.random((9, 11)) > 0.2
    x = rng.uniform(-1, 9, 500)
    y = rng.uniform(-1, 11, 500)
    x[:5] = [0, 8, 8, 3, 2.5]
    y[:5] = [0, 10, 3, 10, 10]
    v, ok = interp.gather(f, msk, x, y)
    vo, oko = orc.masked_sample(f, msk, x, y)
    np.testing.assert_array_equal(ok, oko)
    np.testing.assert_allclose(v, vo, rtol=2e-6, atol=1e-7)
    acc = interp.WeightedAccumulator.zeros((9, 11))
    dropped = interp.scatter_accumulate(acc, x, y, v + 1.0, 2.0)
    av, aw = np.zeros((9, 11)), np.zeros((9, 11))
    d2 = orc.splat(av, aw, x, y, v + 1.0, 2.0)
    assert dropped == d2
    np.testing.assert_allclose(acc.values, av, rtol=1e-5)
    np.testing.assert_allclose(acc.weights, aw, rtol=1e-12)

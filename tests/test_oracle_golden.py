"""Pin the CPU oracle against golden vectors written by the live reference.

These run on CPU (no GPU) and on the GPU box (the fixtures travel; the
reference does not).  Everything is bit-exact: the oracle restates the
reference's float64 operations in the same order.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import pxst_oracle as orc


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_generator_is_stable(scan0, scan1, golden0, golden1):
    assert _sha(scan0.scan.frames) == str(golden0["frames_sha"])
    assert _sha(scan1.scan.frames) == str(golden1["frames_sha"])


def test_cfg0_object_map(scan0, golden0):
    s = scan0
    i_ref, wsum, org = orc.make_object_map(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask,
                                           s.u0.u, s.t0.di, s.t0.dj)
    assert tuple(org) == tuple(golden0["ref_origin"])
    np.testing.assert_array_equal(i_ref, golden0["ref_i"])
    np.testing.assert_array_equal(wsum, golden0["ref_w"])


def _ref0(g):
    return g["ref_i"], g["ref_w"], tuple(int(v) for v in g["ref_origin"])


def test_cfg0_pixel_map(scan0, golden0):
    s = scan0
    args = (s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask, *_ref0(golden0), s.u0.u,
            s.t0.di, s.t0.dj)
    u, e = orc.update_pixel_map(*args, 3, 3)
    np.testing.assert_array_equal(u, golden0["upm_u"])
    np.testing.assert_array_equal(e, golden0["upm_err"])
    u, e = orc.update_pixel_map(*args, 3, 3, quadratic_refinement=False)
    np.testing.assert_array_equal(u, golden0["upm_noref_u"])
    np.testing.assert_array_equal(e, golden0["upm_noref_err"])


def test_cfg0_translations_and_error(scan0, golden0):
    s = scan0
    base = (s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask, *_ref0(golden0))
    di, dj = orc.update_translations(*base, golden0["upm_u"], s.t0.di, s.t0.dj, 2, 2)
    np.testing.assert_array_equal(di, golden0["ut_di"])
    np.testing.assert_array_equal(dj, golden0["ut_dj"])
    di2, dj2 = orc.update_translations(*base, golden0["upm_u"], s.t0.di, s.t0.dj, 1, 1, 0.5)
    np.testing.assert_array_equal(di2, golden0["uts_di"])
    np.testing.assert_array_equal(dj2, golden0["uts_dj"])
    d = orc.calc_error(*base, golden0["upm_u"], di, dj)
    assert d["total"] == float(golden0["ce_total"])
    for k, g in (("per_frame", "ce_per_frame"), ("per_pixel", "ce_per_pixel"),
                 ("reference_plane", "ce_plane"), ("variance", "ce_var")):
        np.testing.assert_array_equal(d[k], golden0[g])


def test_cfg0_main_loop(scan0, golden0):
    s = scan0
    sched = [dict(half_ss=3, half_fs=3, update_translations=True, t_half_ss=1, t_half_fs=1)]
    u, ref, di, dj, hist = orc.run_main_loop(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask,
                                             s.u0.u, s.t0.di, s.t0.dj, sched, 2, tol=-np.inf)
    np.testing.assert_array_equal(u, golden0["loop_u"])
    np.testing.assert_array_equal(di, golden0["loop_di"])
    np.testing.assert_array_equal(np.array(hist), golden0["loop_hist"])
    np.testing.assert_array_equal(ref[0], golden0["loop_ref_i"])


def test_cfg1_object_map(scan1, golden1):
    s = scan1
    i_ref, wsum, org = orc.make_object_map(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask,
                                           s.u0.u, s.t0.di, s.t0.dj)
    assert tuple(org) == tuple(golden1["ref_origin"])
    np.testing.assert_array_equal(i_ref, golden1["ref_i"])
    np.testing.assert_array_equal(wsum, golden1["ref_w"])


def test_cfg1_translation_subset(scan1, golden1):
    s = scan1
    g = golden1
    ref = (g["ref_i"], g["ref_w"], tuple(int(v) for v in g["ref_origin"]))
    di, dj = orc.update_translations(s.scan.frames, g["ut_subset"], s.w.w, s.m.mask, *ref,
                                     s.u0.u, s.t0.di, s.t0.dj, 3, 3)
    np.testing.assert_array_equal(di, g["ut_di"])
    np.testing.assert_array_equal(dj, g["ut_dj"])


@pytest.mark.slow
def test_cfg1_pixel_map_band(scan1, golden1):
    s = scan1
    g = golden1
    ref = (g["ref_i"], g["ref_w"], tuple(int(v) for v in g["ref_origin"]))
    roi = tuple(int(v) for v in g["band"])
    u, e = orc.update_pixel_map(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask, *ref,
                                s.u0.u, s.t0.di, s.t0.dj, 5, 5, roi=roi, threads=4)
    np.testing.assert_array_equal(u[:, roi[0]:roi[1]], g["upm_u"])
    np.testing.assert_array_equal(e[roi[0]:roi[1]], g["upm_err"])


# ---------------------------------------------------------------------------
# SPEC known answers restated on the oracle
# ---------------------------------------------------------------------------
def test_paraboloid_known_answers():
    x = np.array([-1.0, 0.0, 1.0])
    X, Y = np.meshgrid(x, x, indexing="ij")
    bowl = (X - 0.3) ** 2 + 2 * (Y + 0.2) ** 2 + 5
    dss, dfs = orc.paraboloid_offsets(bowl[None])
    assert abs(dss[0] - 0.3) < 1e-10 and abs(dfs[0] + 0.2) < 1e-10
    saddle = X ** 2 - Y ** 2
    dss, dfs = orc.paraboloid_offsets(saddle[None])
    assert dss[0] == 0.0 and dfs[0] == 0.0


def test_window_offsets_semantics():
    np.testing.assert_array_equal(orc.window_offsets(2), [-2, -1, 0, 1, 2])
    np.testing.assert_allclose(orc.window_offsets(1, 0.5), [-1, -0.5, 0, 0.5, 1])
    with pytest.raises(ValueError):
        orc.window_offsets(-1)
    with pytest.raises(ValueError):
        orc.window_offsets(1, 1.5)


# ---------------------------------------------------------------------------
# pixel-map regularisation rows, golden reg0.npz
# ---------------------------------------------------------------------------
def _support_ident(s):
    support = s.m.mask & (s.w.w > 0)
    ss, fs = support.shape
    ident = np.stack(np.meshgrid(np.arange(ss, dtype=np.float64),
                                 np.arange(fs, dtype=np.float64), indexing="ij"))
    return support, ident


def test_smooth_displacement_pinned(scan0, golden_reg):
    support, ident = _support_ident(scan0)
    for c in range(2):
        np.testing.assert_array_equal(
            orc.smooth_displacement(scan0.u0.u[c] - ident[c], support, 2.5), golden_reg[f"sm_{c}"])


def test_integrate_gradient_pinned(golden_reg):
    g = golden_reg
    phi, conv, res, it = orc.integrate_gradient(g["ig_gx"], g["ig_gy"], g["ig_mask"])
    assert it == int(g["ig_iters"]) and conv == bool(g["ig_conv"])
    assert res == float(g["ig_res"])
    np.testing.assert_array_equal(phi, g["ig_phi"])
    with pytest.raises(ValueError):
        orc.integrate_gradient(g["ig_gx"], g["ig_gy"], np.zeros_like(g["ig_mask"]))


@pytest.mark.parametrize("tag,sigma,integrate", [("s", 2.0, False), ("i", 0.0, True),
                                                 ("si", 1.5, True)])
def test_regularised_pixel_map_pinned(scan0, golden0, golden_reg, tag, sigma, integrate):
    s = scan0
    u, e = orc.update_pixel_map(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask,
                                *_ref0(golden0), s.u0.u, s.t0.di, s.t0.dj, 3, 3,
                                sigma=sigma, integrate=integrate)
    np.testing.assert_array_equal(u, golden_reg[f"upm_{tag}_u"])
    np.testing.assert_array_equal(e, golden_reg[f"upm_{tag}_err"])


def test_default_schedule_loop_pinned(scan0, golden_reg):
    from conftest import default_schedule_dicts
    s = scan0
    u, ref, di, dj, hist = orc.run_main_loop(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask,
                                             s.u0.u, s.t0.di, s.t0.dj, default_schedule_dicts(3),
                                             3, tol=-np.inf)
    np.testing.assert_array_equal(u, golden_reg["loop_u"])
    np.testing.assert_array_equal(di, golden_reg["loop_di"])
    np.testing.assert_array_equal(dj, golden_reg["loop_dj"])
    np.testing.assert_array_equal(np.array(hist), golden_reg["loop_hist"])


def test_split_half_pinned(scan0, golden0, golden_reg):
    g = golden_reg
    for sd in (0, 12345):
        np.testing.assert_array_equal(orc.split_bits(sd, 4096), g[f"shb_{sd}"])
    s = scan0
    ua, ub, hss, hfs, sig = orc.split_half_recon(s.scan.frames, s.scan.good_frames, s.w.w,
                                                 s.m.mask, *_ref0(golden0), s.u0.u, s.t0.di,
                                                 s.t0.dj, 2, 2, seed=3)
    np.testing.assert_array_equal(ua, g["sh_ua"])
    np.testing.assert_array_equal(ub, g["sh_ub"])
    np.testing.assert_array_equal(hss, g["sh_hss"])
    np.testing.assert_array_equal(hfs, g["sh_hfs"])
    assert sig == float(g["sh_sigma"])


def _defocus_scan(s):
    from golden.make_golden_reg import defocus_scan
    return defocus_scan(s)


def test_defocus_registration_pinned(scan0, golden_reg):
    g = golden_reg
    sc = _defocus_scan(scan0)
    args = (sc.frames, sc.good_frames, scan0.w.w, scan0.m.mask, sc.distance,
            (sc.x_pixel_size, sc.y_pixel_size), sc.basis_vectors, sc.translations)
    best, contrast, _ = orc.fit_defocus_registration(*args, g["fd_grid"])
    np.testing.assert_array_equal(contrast, g["fd_contrast"])
    assert best == tuple(g["fd_z1"])
    best, contrast, cands = orc.fit_defocus_registration(*args, 0.05 * np.array([0.9, 1.0, 1.1]),
                                                         astigmatic=True)
    np.testing.assert_array_equal(cands, g["fd2_cands"])
    np.testing.assert_array_equal(contrast, g["fd2_contrast"])
    assert best == tuple(g["fd2_z1"])

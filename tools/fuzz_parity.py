"""Randomised parity sweep (GPU box): small scans with random detector sizes,
rasters, pixel-map laws, masks, bad frames, ROIs and search windows through
the drop-in API against the CPU oracle at the BASELINE bars (object map 1e-5
relative with identical validity, bit-exact integer argmin on unique pixels,
refined maps and translations within 1e-3 px, error maps 1e-5 relative).
python tools/fuzz_parity.py [n_cases] [first_seed]   -> one line per case, exit 1 on a failure."""
import os
import sys
import traceback
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2003_12726_b200 as pb  # noqa: E402
from oracle import pxst_oracle as orc  # noqa: E402
from paper_2003_12726_b200 import engine  # noqa: E402
from paper_2003_12726_b200.synth import ScanConfig, make_scan  # noqa: E402

MARGIN, PX_TOL = 1e-4, 1e-3


def unique_pixels(stack):
    """Unique argmin: best and second-best trial apart by > MARGIN relative.
    A best trial at the float64 rounding floor (an exact fit: the sample's
    cells were formed by this sample alone, errors of 1e-21 against trials of
    order 1) is not unique -- the reference's own choice among such residues
    is decided by rounding -- so the margin is taken against at least 1e-9 of
    the pixel's worst trial."""
    flat = stack.reshape(-1, stack.shape[-1])
    part = np.partition(flat, 1, axis=0) if flat.shape[0] > 1 else np.vstack([flat, flat + 1])
    floor = 1e-9 * flat.max(axis=0)
    return (part[1] - part[0]) > MARGIN * np.maximum(np.abs(part[0]), floor)


LAST = {}          # the running case's description (printed with a failure)


def one(seed):
    rng = np.random.default_rng(1000 + seed)
    law = str(rng.choice(["quad", "cubic", "fs_only"]))
    if law == "fs_only":
        cfg = ScanConfig(name=f"fuzz{seed}", n_ss=int(rng.integers(9, 40)), n_fs=int(rng.integers(40, 150)),
                         positions="fs_line", n_frames=int(rng.integers(6, 30)),
                         step=float(rng.uniform(1.0, 3.0)), jitter=0.3, u_law=law,
                         wf_kind=str(rng.choice(["gaussian", "tophat"])),
                         bad_frac=float(rng.choice([0.0, 0.01, 0.05])),
                         u_noise=float(rng.choice([0.0, 0.5, 1.0])))
    else:
        cfg = ScanConfig(name=f"fuzz{seed}", n_ss=int(rng.integers(17, 90)), n_fs=int(rng.integers(20, 150)),
                         positions="raster", nx=int(rng.integers(2, 6)), ny=int(rng.integers(2, 6)),
                         step=float(rng.uniform(1.5, 6.0)), jitter=0.5, u_law=law,
                         obj_sigma=float(rng.uniform(1.5, 3.0)),
                         bad_frac=float(rng.choice([0.0, 0.01, 0.05])),
                         u_noise=float(rng.choice([0.0, 0.5, 1.0])),
                         t_noise=float(rng.choice([0.0, 1.0])), t_noise_kind="uniform")
    many = seed >= 2000      # seeds >= 2000: many frames on a small detector (> 128 and > 512
    if many:                 # good frames: frame-table chunks, sessions, K2's float32 chunk split)
        nx, ny = [(10, 14), (12, 12), (23, 23), (20, 27), (26, 27)][int(rng.integers(0, 5))]
        cfg = ScanConfig(name=f"fuzz{seed}", n_ss=int(rng.integers(17, 48)), n_fs=int(rng.integers(20, 70)),
                         positions="raster", nx=nx, ny=ny, step=float(rng.uniform(1.0, 2.5)), jitter=0.5,
                         u_law=str(rng.choice(["quad", "cubic"])), bad_frac=0.01,
                         u_noise=float(rng.choice([0.5, 1.0])), t_noise=1.0, t_noise_kind="uniform")
        law = cfg.u_law
    s = make_scan(cfg, seed=seed)
    sc, w, m, u, t = s.scan, s.w, s.m, s.u0, s.t0
    hard = seed >= 1000      # seeds >= 1000: harder cases (see below)
    if hard and rng.random() < 0.4:
        # a dead block of the whitefield (W = 0: off the work set, recon.py:88-90)
        W2 = w.w.copy()
        a0, b0 = int(rng.integers(0, cfg.n_ss - 3)), int(rng.integers(0, cfg.n_fs - 3))
        W2[a0:a0 + int(rng.integers(2, 20)), b0:b0 + int(rng.integers(2, 40))] = 0.0
        w = replace(w, w=W2)
    n = sc.frames.shape[0]
    good = np.ones(n, bool)
    if rng.random() < 0.5 and n > 3:
        good[rng.choice(n, size=max(1, n // 5), replace=False)] = False
    sc = replace(sc, good_frames=good)
    if many and rng.random() < 0.7:
        # the stack in a detector's own element type (uploaded as it is and
        # converted on the device; the reference casts per use, recon.py:91)
        dt = [np.uint16, np.int32, np.float64, np.int64][int(rng.integers(0, 4))]
        assert np.array_equal(sc.frames.astype(dt).astype(np.float32), sc.frames)
        sc = replace(sc, frames=sc.frames.astype(dt))
    roi = None
    if rng.random() < 0.4:
        r0 = int(rng.integers(0, cfg.n_ss // 2)); r1 = int(rng.integers(r0 + 4, cfg.n_ss + 1))
        c0 = int(rng.integers(0, cfg.n_fs // 2)); c1 = int(rng.integers(c0 + 4, cfg.n_fs + 1))
        roi = pb.Roi(r0, min(r1, cfg.n_ss), c0, min(c1, cfg.n_fs))
    rt = roi.as_tuple() if roi else None
    if law == "fs_only":
        half = (0, int(rng.integers(1, 9)))
    else:
        half = (int(rng.integers(0, 7)), int(rng.integers(0, 7)))
        if rng.random() < 0.6:
            half = (half[0], half[0])          # the square fast-path windows
    if many:
        half = (min(half[0], 2), min(half[1], 2))      # (keeps the oracle's cost down)
    sub = float(rng.choice([0.5, 0.25, 0.4])) if rng.random() < 0.15 else None
    if sub is not None:
        half = (min(half[0], 2), min(half[1], 2))
    refine = bool(rng.random() < 0.6)
    if hard and sub is None and rng.random() < 0.3:
        # wide windows: 15 x 15 / 17 x 17 (generic kernel), 1 x 17 and 17 x 1 rows
        k = int(rng.choice([7, 8]))
        half = [(k, k), (0, 8), (8, 0)][int(rng.integers(0, 3))] if law != "fs_only" else (0, 8)
    desc = (f"seed {seed}: {cfg.n_ss}x{cfg.n_fs} {law} {sc.frames.dtype} frames {n} ({int(good.sum())} good) "
            f"roi {rt} window {half} sub {sub} refine {refine}")
    oa = (sc.frames, sc.good_frames, w.w, m.mask)
    LAST["desc"] = desc
    engine.SCAN_CACHE.clear()
    # K1
    ref_roi, ref_rt = roi, rt
    if hard and rng.random() < 0.35:
        # the reference formed on a smaller detector rectangle than the one
        # searched: many samples read invalid cells or leave the grid
        # (interp.py:53-85 masked renormalisation, recon.py:160-166 fallback)
        r0 = int(rng.integers(0, max(1, cfg.n_ss // 3))); c0 = int(rng.integers(0, max(1, cfg.n_fs // 3)))
        ref_roi = pb.Roi(r0, int(rng.integers(r0 + 6, cfg.n_ss + 1)), c0, int(rng.integers(c0 + 6, cfg.n_fs + 1)))
        ref_rt = ref_roi.as_tuple()
        desc += f" ref-roi {ref_rt}"
    try:
        i_ref, wsum, org = orc.make_object_map(*oa, u.u, t.di, t.dj, roi=ref_rt)
    except ValueError as exc:            # empty work set (recon.py:116-117): same error here
        try:
            pb.make_reference(sc, w, m, u, t, roi=ref_roi)
        except ValueError as exc2:
            assert str(exc2) == str(exc), (str(exc2), str(exc))
            return desc + " | both raise: " + str(exc)
        raise AssertionError("the oracle raised, the GPU path did not")
    ref = pb.make_reference(sc, w, m, u, t, roi=ref_roi)
    assert tuple(ref.origin) == tuple(org) and ref.i_ref.shape == i_ref.shape, "grid"
    ok = wsum > 0
    assert np.array_equal(ref.wsum > 0, ok), "validity"
    rel = np.abs(ref.i_ref[ok] - i_ref[ok]) / np.maximum(np.abs(i_ref[ok]), 1e-300)
    assert rel.max() < 1e-5, ("object", rel.max())
    # K2
    win = pb.SearchWindow(half[0], half[1], sub)
    fw = None
    if rng.random() < 0.2:               # frame weights (split-half style 0/1, or smooth)
        shape = (n, cfg.n_ss, cfg.n_fs)
        fw = (rng.random(shape) < 0.5).astype(np.float32) if rng.random() < 0.5 else \
            rng.uniform(0.5, 1.5, shape).astype(np.float32)
        desc += " fw"
    un, en = pb.update_pixel_map(sc, w, m, ref, u, t, win,
                                 pb.UpdateOptions(quadratic_refinement=refine), roi=roi,
                                 frame_weights=fw)
    uo, eo, stack = orc.update_pixel_map(*oa, ref.i_ref, ref.wsum, ref.origin, u.u, t.di, t.dj,
                                         half[0], half[1], sub, refine, rt, fw,
                                         threads=os.cpu_count() or 1, return_stack=True)
    r0, r1, c0, c1 = rt or (0, cfg.n_ss, 0, cfg.n_fs)
    sub_m = m.mask[r0:r1, c0:c1] & (w.w[r0:r1, c0:c1] > 0)
    rr, cc = np.nonzero(sub_m)
    rr, cc = rr + r0, cc + c0
    uniq = unique_pixels(stack) if stack.shape[0] * stack.shape[1] > 1 else np.ones(rr.size, bool)
    gu, ou = un.u[:, rr, cc], uo[:, rr, cc]
    if not refine and sub is None:
        assert np.array_equal(gu[:, uniq], ou[:, uniq]), "integer argmin"
    # every trial exactly equal (all of them on the (I - W)^2 fallback): the
    # argmin is the first index on both sides (recon.py:265-269)
    flat_s = stack.reshape(-1, stack.shape[-1])
    alltie = flat_s.max(axis=0) == flat_s.min(axis=0)
    if flat_s.shape[0] > 1 and alltie.any():
        assert np.array_equal(gu[:, alltie], ou[:, alltie]), "exact ties -> first index"
    d = np.abs(gu - ou).max(axis=0)
    assert uniq.sum() == 0 or d[uniq].max() < PX_TOL, ("pixel map", d[uniq].max())
    oth = np.ones(w.w.shape, bool); oth[rr, cc] = False
    assert np.array_equal(un.u[:, oth], u.u[:, oth]), "pixels off the work set changed"
    # error map: 1e-4 relative, plus the float32 floor of the residual
    # r = I - W v (|dr| ~ 1e-7 I): |d sum r^2| <~ 1e-6 sqrt(sum I^2 sum r^2), in
    # the map's normalisation (recon.py:257-263: var = sum fw (I - W)^2)
    I = sc.frames[good][:, rr, cc].astype(np.float64)
    fwp = np.ones_like(I) if fw is None else fw[good][:, rr, cc].astype(np.float64)
    var = (fwp * (I - w.w[rr, cc][None, :]) ** 2).sum(axis=0)
    s_i2 = (fwp * I * I).sum(axis=0) / np.where(var > 0, var, 1.0)
    e_g, e_o = en[rr, cc][uniq], eo[rr, cc][uniq]
    tol = 1e-4 * np.abs(e_o) + 1e-6 * np.sqrt(s_i2[uniq] * np.abs(e_o)) + 1e-300
    assert uniq.sum() == 0 or np.all(np.abs(e_g - e_o) <= tol), \
        ("err map", float(np.max(np.abs(e_g - e_o) / tol)))
    # K2's optional stages (recon.py:298-311: Gaussian smoothing of the
    # displacement, irrotational projection) on identical inputs: the oracle's
    # raw map through the device kernels against the oracle's own stages
    if seed % 3 == 0 and fw is None:
        sigma = float(rng.choice([0.0, 1.5, 3.0]))
        integ = bool(rng.random() < 0.7)
        support = np.zeros(w.w.shape, bool)
        support[rr, cc] = True
        u_reg_o = orc.regularise_map(uo, support, sigma, integ)
        ds = engine.SCAN_CACHE.get(sc, w, m, roi)
        u_t = ds.upload_u(uo.copy())
        ds.regularise(u_t, pb.UpdateOptions(True, integ, sigma))
        dreg = np.abs(u_t.cpu().numpy() - u_reg_o).max()
        assert dreg < 1e-8, ("regularised map", dreg, sigma, integ)
        desc += f" reg(s{sigma},{'int' if integ else '-'}) {dreg:.0e}"
    # split-half uncertainty (analysis.py:294-361): the device SplitMix split of
    # the samples and one search per half against the oracle's
    if seed % 4 == 1 and sub is None and max(half) <= 4:
        from paper_2003_12726_b200 import analysis
        S = analysis.split_half_recon(sc, w, m, ref, u, t, win, seed=seed,
                                      opts=pb.UpdateOptions(refine, False, 0.0), roi=roi)
        ua, ub, hss, hfs, sg, st_a, st_b = orc.split_half_recon(
            *oa, ref.i_ref, ref.wsum, ref.origin, u.u, t.di, t.dj, half[0], half[1], seed=seed,
            quadratic_refinement=refine, roi=rt, threads=os.cpu_count() or 1, return_stacks=True)
        nun = 0
        for got, want, st in ((S.map_a.u, ua, st_a), (S.map_b.u, ub, st_b)):
            uq = unique_pixels(st) if st.shape[0] * st.shape[1] > 1 else np.ones(rr.size, bool)
            dd_ = np.abs(got[:, rr, cc] - want[:, rr, cc]).max(axis=0)
            assert uq.sum() == 0 or dd_[uq].max() < PX_TOL, ("split-half map", dd_[uq].max())
            assert np.array_equal(got[:, oth], want[:, oth]), "split-half: pixels off the work set"
            nun += int((~uq).sum())
        slack = 2 * nun + 2
        assert np.abs(S.hist_ss - hss).sum() <= slack and np.abs(S.hist_fs - hfs).sum() <= slack, "split-half histograms"
        desc += " split-half"
    # K3 (on the oracle's map, so both see the same input)
    U = pb.PixelMap(uo)
    th = (int(rng.integers(0, 4)), int(rng.integers(0, 4)))
    tsub = float(rng.choice([0.5, 0.25])) if rng.random() < 0.2 else None
    T = pb.update_translations(sc, w, m, ref, U, t, pb.SearchWindow(th[0], th[1], tsub), roi=roi)
    di, dj, errs = orc.update_translations(*oa, ref.i_ref, ref.wsum, ref.origin, U.u, t.di, t.dj,
                                           th[0], th[1], tsub, roi=rt, return_errors=True)
    nchk = 0
    for fr, e in errs.items():
        flat = np.sort(e.ravel())
        if flat.size < 2 or (flat[1] - flat[0]) > MARGIN * abs(flat[0]):
            assert abs(T.di[fr] - di[fr]) < PX_TOL and abs(T.dj[fr] - dj[fr]) < PX_TOL, \
                ("translation", fr, T.di[fr] - di[fr], T.dj[fr] - dj[fr])
            nchk += 1
    bad = ~good
    assert np.array_equal(T.di[bad], t.di[bad]) and np.array_equal(T.dj[bad], t.dj[bad]), "bad frames moved"
    # K4
    M = pb.calc_error(sc, w, m, ref, U, t, roi=roi)
    dd = orc.calc_error(*oa, ref.i_ref, ref.wsum, ref.origin, U.u, t.di, t.dj, roi=rt)
    np.testing.assert_allclose(M.per_frame, dd["per_frame"], rtol=1e-9, atol=1e-300)
    np.testing.assert_allclose(M.per_pixel, dd["per_pixel"], rtol=1e-9, atol=1e-300)
    assert abs(M.total - dd["total"]) <= 1e-9 * abs(dd["total"])
    # (the plane is an exact fixed-point sum: a cell whose eps terms are below
    # the quantum -- ~2^-61 of the eps bound -- reads 0 where float64 keeps 1e-19)
    pl, po = M.reference_plane, dd["reference_plane"]
    np.testing.assert_allclose(pl, po, rtol=1e-5, atol=1e-9 * max(1.0, np.abs(po).max()))
    return desc + f" | obj {rel.max():.1e} px {d[uniq].max() if uniq.sum() else 0:.1e} uniq {uniq.mean():.3f} t {th}/{tsub} frames checked {nchk}"


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    fails = 0
    for seed in range(first, first + n):
        try:
            print("ok  ", one(seed), flush=True)
        except Exception as e:          # noqa: BLE001
            fails += 1
            print("FAIL", f"seed {seed}:", repr(e)[:300], "|", LAST.get("desc", ""), flush=True)
            traceback.print_exc(limit=3)
    print(f"{n - fails} / {n} cases passed")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

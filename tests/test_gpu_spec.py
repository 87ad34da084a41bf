"""SPEC known answers and invariants of the hot path, on
the GPU path, with the tolerances the oracle itself meets:

* make_reference: one frame, identity map, I = W  ->  i_ref == 1 on valid
  cells, the +2 shape rule's last row/column invalid;
* update_translations: a frame displaced by +1 px is restored, the others
  move exactly as the oracle's (paraboloid jitter, not
  "unchanged"); a zero window returns the input exactly (:400);
* calc_error: noiseless data with the true map, translations and reference
  give a total at float32-rounding level;
* make_reference is equivariant under integer translation shifts;
* calc_error's total is invariant under a frame permutation;
* update_pixel_map never reports an error above the incumbent's (A3; the
  err_map is the integer-grid error).
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2003_12726_b200 as pb  # noqa: E402
from oracle import pxst_oracle as orc  # noqa: E402


def _scene(seed=0, n=9, ss=32, fs=40, noise=False, smooth=True):
    """Frames rendered from a smooth object with a known map and translations."""
    rng = np.random.default_rng(seed)
    shape = (ss + 24, fs + 24)
    yy, xx = np.meshgrid(np.arange(shape[0]), np.arange(shape[1]), indexing="ij")
    obj = 1.0 + 0.3 * np.sin(xx / 3.1) * np.cos(yy / 4.3) if smooth else \
        1.0 + 0.3 * rng.standard_normal(shape)
    W = 800.0 + 50 * rng.random((ss, fs))
    di = rng.uniform(-4, 4, n)
    dj = rng.uniform(-4, 4, n)
    u = pb.PixelMap.identity((ss, fs)).u.copy()
    u[0] += 0.05 * np.sin(np.arange(fs) / 7.0)[None, :]
    frames = np.empty((n, ss, fs), np.float32)
    for k in range(n):
        v, _ = orc.masked_sample(obj, np.ones(shape, bool), u[0] - di[k] + 10, u[1] - dj[k] + 10)
        frames[k] = rng.poisson(W * v) if noise else W * v
    sc = pb.ScanData(frames, 1e-10, 1.0, 1e-5, 1e-5, np.zeros((n, 2, 3)), np.zeros((n, 3)),
                     np.ones(n, bool))
    return sc, pb.Whitefield(W), pb.PixelMask(np.ones((ss, fs), bool)), pb.PixelMap(u), \
        pb.PixelTranslations(di, dj)


def test_single_frame_identity_reference_is_one():
    ss, fs = 20, 30
    W = 300.0 + 10 * np.random.default_rng(1).random((ss, fs))
    sc = pb.ScanData(W[None].astype(np.float32), 1e-10, 1.0, 1e-5, 1e-5, np.zeros((1, 2, 3)),
                     np.zeros((1, 3)), np.ones(1, bool))
    Wf = W.astype(np.float32).astype(np.float64)
    ref = pb.make_reference(sc, pb.Whitefield(Wf), pb.PixelMask(np.ones((ss, fs), bool)),
                            pb.PixelMap.identity((ss, fs)), pb.PixelTranslations(np.zeros(1),
                                                                                 np.zeros(1)))
    assert ref.i_ref.shape == (ss + 1, fs + 1)                       # +2 rule (recon.py:132)
    ok = ref.wsum > 0
    assert not ok[-1].any() and not ok[:, -1].any()
    np.testing.assert_allclose(ref.i_ref[ok], 1.0, rtol=1e-6)


def test_translation_restored_and_zero_window():
    sc, w, m, u, t = _scene()
    di = t.di.copy()
    di[3] += 1.0
    bad = pb.PixelTranslations(di, t.dj.copy())
    ref = pb.make_reference(sc, w, m, u, t)                          # true translations
    T = pb.update_translations(sc, w, m, ref, u, bad, pb.SearchWindow(2, 2))
    assert abs(T.di[3] - t.di[3]) < 0.05 and abs(T.dj[3] - t.dj[3]) < 0.05
    # the other frames move by the always-on paraboloid's jitter (SURVEY 4:
    # "not unchanged"); they must move exactly as the oracle's do
    odi, odj = orc.update_translations(sc.frames, sc.good_frames, w.w, m.mask, ref.i_ref,
                                       ref.wsum, ref.origin, u.u, bad.di, bad.dj, 2, 2)
    assert np.abs(T.di - odi).max() < 1e-3 and np.abs(T.dj - odj).max() < 1e-3
    Z = pb.update_translations(sc, w, m, ref, u, bad, pb.SearchWindow(0, 0))
    np.testing.assert_array_equal(Z.di, bad.di)
    np.testing.assert_array_equal(Z.dj, bad.dj)


def test_perfect_data_error_vanishes():
    """With the true reference the residuals are the frames' float32 rounding."""
    sc, w, m, u, t = _scene()
    shape = (sc.frames.shape[1] + 24, sc.frames.shape[2] + 24)
    yy, xx = np.meshgrid(np.arange(shape[0]), np.arange(shape[1]), indexing="ij")
    obj = 1.0 + 0.3 * np.sin(xx / 3.1) * np.cos(yy / 4.3)
    true_ref = pb.ReferenceImage(i_ref=obj, wsum=np.ones(shape), origin=(-10, -10), du=1.0,
                                 dv=1.0)
    M = pb.calc_error(sc, w, m, true_ref, u, t)
    n_samples = sc.frames.size
    assert M.total <= 1e-9 * n_samples, M.total
    # a rebuilt reference stays close (interpolation of a smooth object)
    ref = pb.make_reference(sc, w, m, u, t)
    M2 = pb.calc_error(sc, w, m, ref, u, t)
    assert M2.total <= 1e-2 * n_samples, M2.total


def test_reference_equivariant_under_integer_shifts():
    sc, w, m, u, t = _scene(seed=2, noise=True)
    a = pb.make_reference(sc, w, m, u, t)
    b = pb.make_reference(sc, w, m, u, pb.PixelTranslations(t.di + 3.0, t.dj - 2.0))
    assert (b.origin[0], b.origin[1]) == (a.origin[0] - 3, a.origin[1] + 2)
    assert a.i_ref.shape == b.i_ref.shape
    np.testing.assert_array_equal(a.wsum > 0, b.wsum > 0)
    np.testing.assert_allclose(b.i_ref, a.i_ref, rtol=1e-5, atol=1e-12)


def test_error_total_invariant_under_frame_permutation():
    sc, w, m, u, t = _scene(seed=4, noise=True)
    ref = pb.make_reference(sc, w, m, u, t)
    M = pb.calc_error(sc, w, m, ref, u, t)
    perm = np.random.default_rng(0).permutation(sc.frames.shape[0])
    sc2 = replace(sc, frames=np.ascontiguousarray(sc.frames[perm]))
    t2 = pb.PixelTranslations(t.di[perm], t.dj[perm])
    M2 = pb.calc_error(sc2, w, m, ref, u, t2)
    assert abs(M2.total - M.total) <= 1e-12 * M.total
    np.testing.assert_allclose(M2.per_frame, M.per_frame[perm], rtol=1e-12)


@pytest.mark.parametrize("half", [1, 3])
def test_pixel_map_never_worse_than_incumbent(half):
    sc, w, m, u, t = _scene(seed=6, noise=True, smooth=False)
    ref = pb.make_reference(sc, w, m, u, t)
    _, e0 = pb.update_pixel_map(sc, w, m, ref, u, t, pb.SearchWindow(0, 0),
                                pb.UpdateOptions(quadratic_refinement=False))
    _, e1 = pb.update_pixel_map(sc, w, m, ref, u, t, pb.SearchWindow(half, half))
    # equal where the incumbent wins, up to the engines' float32 sum order
    assert np.all(e1 <= e0 * (1 + 1e-5) + 1e-12)


def test_in_place_mutation_detected(scan0):
    """The device caches are keyed by array identity (value-object convention,
    data_model.py:13) plus a sampled content fingerprint: an input mutated in
    place between calls is re-uploaded, never served stale."""
    import copy
    s = copy.deepcopy(scan0)
    ref1 = pb.make_reference(s.scan, s.w, s.m, s.u0, s.t0)
    s.scan.frames[3] *= 1.5                      # same array object, new content
    ref2 = pb.make_reference(s.scan, s.w, s.m, s.u0, s.t0)
    pb.clear_cache()
    ref3 = pb.make_reference(s.scan, s.w, s.m, s.u0, s.t0)
    assert not np.array_equal(ref1.i_ref, ref2.i_ref)
    np.testing.assert_array_equal(ref2.i_ref, ref3.i_ref)
    u = pb.PixelMap(s.u0.u.copy())
    win = pb.SearchWindow(2, 2)
    a, _ = pb.update_pixel_map(s.scan, s.w, s.m, ref3, u, s.t0, win)
    u.u[0] += 0.25                               # mutate the pixel map in place
    b, _ = pb.update_pixel_map(s.scan, s.w, s.m, ref3, u, s.t0, win)
    pb.clear_cache()
    c, _ = pb.update_pixel_map(s.scan, s.w, s.m, ref3, u, s.t0, win)
    np.testing.assert_array_equal(b.u, c.u)
    assert not np.array_equal(a.u, b.u)


@pytest.mark.parametrize("dtype", [np.uint16, np.int32, np.uint32, np.int64, np.float64])
def test_frame_stack_of_another_dtype(scan1, dtype):
    """The reference takes frames of any dtype and casts them where it reads
    them (recon.py:91).  A stack of detector counts in its own element type is
    uploaded as it is and converted on the device (pxst_stack_to_f32): same
    bits as the float32 stack of the same counts."""
    from dataclasses import replace
    s = scan1
    assert float(s.scan.frames.max()) < 65535 and np.all(s.scan.frames == np.rint(s.scan.frames))
    sc_n = replace(s.scan, frames=s.scan.frames.astype(dtype))
    win = pb.SearchWindow(2, 2)
    outs = []
    for sc in (s.scan, sc_n):
        pb.clear_cache()
        ref = pb.make_reference(sc, s.w, s.m, s.u0, s.t0)
        u, e = pb.update_pixel_map(sc, s.w, s.m, ref, s.u0, s.t0, win)
        m = pb.calc_error(sc, s.w, s.m, ref, u, s.t0)
        outs.append((ref.i_ref, ref.wsum, u.u, e, m.per_frame, m.per_pixel, m.reference_plane))
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)
    pb.clear_cache()

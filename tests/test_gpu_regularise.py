"""GPU parity of the pixel-map regularisation rows:
mask-aware Gaussian smoothing (recon.py:210-218) and the irrotational
projection by device CG (integration.py:61-134), against golden vectors
written by the live reference (tests/golden/reg0.npz) and the oracle."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2003_12726_b200 as pb  # noqa: E402
from oracle import pxst_oracle as orc  # noqa: E402
from paper_2003_12726_b200 import engine, integration  # noqa: E402

PX_TOL = 1e-3


def _ident(shape):
    ss, fs = shape
    return np.stack(np.meshgrid(np.arange(ss, dtype=np.float64), np.arange(fs, dtype=np.float64),
                                indexing="ij"))


def test_smooth_displacement_vs_golden(scan0, golden_reg):
    s = scan0
    ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
    u_t = ds.upload_u(s.u0.u)
    ds.smooth_displacement(u_t, 2.5)
    got = u_t.cpu().numpy() - _ident(s.w.w.shape)
    for c in range(2):
        # scipy's symmetric correlate1d order, no FMA contraction: ulp-level
        np.testing.assert_allclose(got[c], golden_reg[f"sm_{c}"], rtol=1e-13, atol=1e-13)


def test_integrate_gradient_vs_golden(golden_reg):
    g = golden_reg
    res = integration.integrate_gradient(g["ig_gx"], g["ig_gy"], g["ig_mask"])
    assert res.converged and res.residual <= 1e-12
    # CG to 1e-12 relative residual: potentials agree to ~1e-10 of their scale
    scale = np.abs(g["ig_phi"]).max()
    np.testing.assert_allclose(res.phi, g["ig_phi"], rtol=0, atol=1e-9 * scale)
    assert abs(res.iterations - int(g["ig_iters"])) <= 0.05 * int(g["ig_iters"]) + 2
    anchor = tuple(np.argwhere(g["ig_mask"])[0])
    assert res.phi[anchor] == 0.0
    with pytest.raises(ValueError):
        integration.integrate_gradient(g["ig_gx"], g["ig_gy"], np.zeros_like(g["ig_mask"]))
    d, _ = integration.project_irrotational(g["ig_gx"], g["ig_gy"], g["ig_mask"])
    np.testing.assert_allclose(d, orc.image_grad(g["ig_phi"]), rtol=0, atol=1e-8 * scale)


def _plain_mismatch(s, golden0):
    ref = pb.make_reference(s.scan, s.w, s.m, s.u0, s.t0)
    un, _ = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(3, 3))
    return ref, np.abs(un.u - golden0["upm_u"]).max(axis=0) > PX_TOL


@pytest.mark.parametrize("tag,sigma,integrate", [("s", 2.0, False), ("i", 0.0, True),
                                                 ("si", 1.5, True)])
def test_regularised_pixel_map_vs_golden(scan0, golden0, golden_reg, tag, sigma, integrate):
    s = scan0
    ref, bad = _plain_mismatch(s, golden0)
    # near-tie argmins propagate through the coupling filters;
    # the config-0 scan has none at this window
    assert bad.sum() == 0, bad.sum()
    un, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, s.u0, s.t0, pb.SearchWindow(3, 3),
                                pb.UpdateOptions(sigma=sigma, integrate=integrate))
    d = np.abs(un.u - golden_reg[f"upm_{tag}_u"]).max()
    assert d < PX_TOL, d
    np.testing.assert_allclose(e, golden_reg[f"upm_{tag}_err"], rtol=1e-4, atol=1e-12)


def test_default_schedule_main_loop(scan0, golden_reg):
    """The reference's default schedule end to end.  On this small scan the
    schedule's second iteration (window +-2, sigma 3, translations on) blows
    the error up ~20x, a regime where near-tie argmins flip and
    the two trajectories drift apart: iteration 1 is held to 1e-6, later
    totals to 1e-2.  Per-step parity is pinned by the tests above."""
    s = scan0
    L = pb.run_main_loop(s.scan, s.w, s.m, s.u0, s.t0, schedule=pb.default_schedule(3),
                         max_iters=3, tol=-np.inf)
    hist = np.array([h.total for h in L.history])
    np.testing.assert_allclose(hist[:2], golden_reg["loop_hist"][:2], rtol=1e-6)
    np.testing.assert_allclose(hist, golden_reg["loop_hist"], rtol=1e-2)
    assert np.isfinite(L.pixel_map.u).all()

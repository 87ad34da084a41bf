"""The fused K4 + next-K1 pass (pxst_error_maps_splat) equals the separate
calc_error and make_reference on the same (u, t) (recon.py:511-516 order)."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from paper_2003_12726_b200 import engine  # noqa: E402


@pytest.mark.parametrize("scan_name", ["scan0", "scan1"])
def test_error_maps_and_next_object(request, scan_name):
    s = request.getfixturevalue(scan_name)
    ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
    u, (di, dj) = ds.upload_u(s.u0.u), ds.upload_t(s.t0.di, s.t0.dj)
    ref = ds.object_map(u, di, dj)
    cfg = s.cfg
    u1, _ = ds.pixel_map_search(ref, u, di, dj, cfg.half_ss, cfg.half_fs)
    geom = ds.geometry_async(u1, di, dj)
    (t_f, pf_f, pp_f, pl_f, _), pend = ds.error_maps_and_next_object(ref, u1, di, dj, geom)
    nref = pend.resolve()
    t_s, pf_s, pp_s, pl_s, _ = ds.error_maps(ref, u1, di, dj)
    sref = ds.object_map(u1, di, dj)
    np.testing.assert_allclose(pf_f.cpu().numpy(), pf_s.cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(pp_f.cpu().numpy(), pp_s.cpu().numpy(), rtol=1e-12)
    # plane and object are exact fixed-point sums (fixsplat.cuh): the fused
    # and separate passes agree bit for bit
    assert torch.equal(pl_f, pl_s)
    assert abs(t_f.item() - t_s.item()) <= 1e-12 * abs(t_s.item())
    assert tuple(nref.origin) == tuple(sref.origin) and nref.shape == sref.shape
    assert torch.equal(nref.valid, sref.valid)
    assert torch.equal(nref.i_ref, sref.i_ref) and torch.equal(nref.wsum, sref.wsum)
    # the geometry future agrees with the synchronous bbox
    assert geom.bbox() == ds.bbox(u1, di, dj)
    n0, m0, (os_, of) = geom.bbox()
    assert geom.grid_dev.cpu().tolist() == [n0, m0, os_, of]
    # a capacity too small for the grid: nothing splatted, resolve() forms it afresh
    (_, _, _, _, _), small = ds.error_maps_and_next_object(ref, u1, di, dj, geom, margin=-20)
    assert small.cap < os_ * of
    alt = small.resolve()
    assert torch.equal(alt.i_ref, sref.i_ref) and torch.equal(alt.valid, sref.valid)


@pytest.mark.parametrize("scan_name", ["scan0", "scan1"])
def test_object_map_and_plane_bit_reproducible(request, scan_name):
    """Two runs of object formation and of the error maps give identical
    bits (the reference's np.bincount is deterministic, interp.py:114-122;
    here the terms are summed as exact integers, fixsplat.cuh), and so does a
    fresh DeviceScan of the same data."""
    s = request.getfixturevalue(scan_name)
    outs = []
    for _ in range(2):
        ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
        u, (di, dj) = ds.upload_u(s.u0.u), ds.upload_t(s.t0.di, s.t0.dj)
        runs = []
        for _ in range(2):
            ref = ds.object_map(u, di, dj)
            total, pf, pp, plane, _ = ds.error_maps(ref, u, di, dj)
            runs.append((ref.i_ref.clone(), ref.wsum.clone(), ref.valid.clone(), plane.clone(),
                         pf.clone(), pp.clone(), total.clone()))
        for a, b in zip(*runs):
            assert torch.equal(a, b)
        outs.append(runs[0])
    for a, b in zip(*outs):
        assert torch.equal(a, b)

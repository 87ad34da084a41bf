"""Single-process multi-GPU loop (multigpu.py) on this
one-GPU pool: ``Devices([0, 0])`` / ``[0, 0, 0]`` split the work into two /
three shares on cuda:0 through the same code path 8 GPUs take (peer-memory
finish kernel, or peer copies and library add kernels).  The object map and reference plane are exact integer
sums, so they equal the one-device results bit for bit for the same inputs;
the loop's u and translations agree at the north-star bars."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import paper_2003_12726_b200 as pb  # noqa: E402
from paper_2003_12726_b200 import engine  # noqa: E402
from paper_2003_12726_b200.multigpu import Devices, MultiScan  # noqa: E402


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("ids", [[0, 0], [0, 0, 0]])
def test_multiscan_phases_match_one_device(scan1, ids, fused):
    """fused: the accumulators' all-reduce fused with the normalisation over
    peer memory (pxst_object_finish_peers: each share reads every peer's int64
    terms in place and stores its slice into every peer's images); otherwise
    peer copies + add kernels + a finish per device.  Both equal one device."""
    s = scan1
    ms = MultiScan(s.scan, s.w, s.m, None, Devices(ids))
    ms.fused_finish = fused
    us, dis, djs = ms.upload(s.u0.u, s.t0.di, s.t0.dj)
    refs = ms.object_map(us, dis, djs)
    ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
    u, (di, dj) = ds.upload_u(s.u0.u), ds.upload_t(s.t0.di, s.t0.dj)
    ref = ds.object_map(u, di, dj)
    for r in refs:                 # frame shards add exactly
        assert torch.equal(r.i_ref, ref.i_ref) and torch.equal(r.wsum, ref.wsum)
        assert torch.equal(r.valid, ref.valid)
    c = s.cfg
    us2 = ms.pixel_map(refs, us, dis, djs, c.half_ss, c.half_fs)
    u1, _ = ds.pixel_map_search(ref, u, di, dj, c.half_ss, c.half_fs)
    for k in range(1, len(ids)):
        assert torch.equal(us2[k], us2[0])     # every device holds the same gathered map
    d = (us2[0] - u1).abs().amax(dim=0).cpu().numpy()
    assert np.mean(d < 1e-3) > 0.9995, np.mean(d < 1e-3)
    # error maps of one (ref, u): plane exact, per-frame / per-pixel to rounding
    outs = ms.error_maps(refs, us2, dis, djs)
    total, pf, pp, plane, _ = ds.error_maps(ref, us2[0], di, dj)
    for (t_k, pf_k, pp_k, pl_k, _) in outs:
        assert torch.equal(pl_k, plane)
        np.testing.assert_allclose(pf_k.cpu().numpy(), pf.cpu().numpy(), rtol=1e-12)
        np.testing.assert_allclose(pp_k.cpu().numpy(), pp.cpu().numpy(), rtol=1e-12)
        assert abs(float(t_k.item()) - float(total.item())) <= 1e-12 * float(total.item())
    engine.clear_cache()


def test_run_main_loop_devices(scan0):
    """run_main_loop(devices=...) against the one-device loop (config 0, with
    translation updates)."""
    s = scan0
    sched = [pb.IterationSettings(window=pb.SearchWindow(3, 3),
                                  options=pb.UpdateOptions(True, False, 0.0),
                                  update_translations=True,
                                  translation_window=pb.SearchWindow(1, 1))]
    L1 = pb.run_main_loop(s.scan, s.w, s.m, s.u0, s.t0, schedule=sched, max_iters=2, tol=-np.inf)
    L2 = pb.run_main_loop(s.scan, s.w, s.m, s.u0, s.t0, schedule=sched, max_iters=2, tol=-np.inf,
                          devices=[0, 0])
    np.testing.assert_allclose([h.total for h in L2.history], [h.total for h in L1.history],
                               rtol=1e-9)
    d = np.abs(L2.pixel_map.u - L1.pixel_map.u).max(axis=0)
    assert np.mean(d < 1e-3) > 0.999
    assert np.abs(L2.translations.di - L1.translations.di).max() < 1e-3
    assert np.abs(L2.translations.dj - L1.translations.dj).max() < 1e-3
    assert L2.reference.origin == L1.reference.origin
    engine.clear_cache()

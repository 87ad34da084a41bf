"""Golden vectors for the multi-iteration loops and the config-2 object map,
written from the LIVE reference (``/root/reference/pkg/src/pxst``).

Run in the build container (the reference does not exist on the GPU box):

    python tests/golden/make_golden_loop.py [cfg0loop] [cfg1loop] [cfg2ref]

* ``loop0.npz`` / ``loop1.npz``: ``recon.run_main_loop`` (recon.py:479-522)
  on configs 0 (2 iterations, R=3 + +-1 translations) and 1 (the bench's
  3 iterations of object -> pixel map (R=5, refine) -> error maps,
  ``tol=-inf``).  Besides the reference's own results, the script replays the
  same trajectory through the oracle port (bit-identical to the reference,
  asserted here) to record, per iteration, which pixels / frames have a
  unique grid-search argmin (relative best/second-best margin > 1e-4 of the
  normalised errors).  A pixel (frame) is "robust" when its
  argmin is unique in every iteration; the parity bars apply there.
* ``ref2.npz``: ``recon.make_reference`` on config 2 (1000 frames of
  516x1556), the full object map (float32 i_ref + packed validity; SURVEY
  8(c): object-map goldens need the full frame set).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import live_reference  # noqa: E402
from oracle import pxst_oracle as orc  # noqa: E402
from paper_2003_12726_b200.synth import CONFIGS, make_scan  # noqa: E402

MARGIN = 1e-4
THREADS = os.cpu_count() or 1


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def unique_mask(stack):
    P = stack.shape[-1]
    part = np.partition(stack.reshape(-1, P), 1, axis=0)
    return (part[1] - part[0]) > MARGIN * np.abs(part[0])


def loop_golden(cfg_id, sched_ref, sched_orc, iters):
    pxst = live_reference.load()
    from pxst import recon
    s = make_scan(cfg_id)
    sc, w, m, u0, t0 = s.scan, s.w, s.m, s.u0, s.t0
    t = time.time()
    L = recon.run_main_loop(sc, w, m, u0, t0, schedule=sched_ref, max_iters=iters,
                            tol=-np.inf, threads=THREADS)
    print(f"cfg{cfg_id} reference loop {time.time() - t:.0f} s", flush=True)
    # replay through the oracle, recording argmin uniqueness per iteration
    F, G, W, M = sc.frames, sc.good_frames, w.w, m.mask
    u = u0.u.copy()
    di, dj = t0.di.copy(), t0.dj.copy()
    rows, cols = np.nonzero(M & (W > 0))
    robust_px = np.ones(rows.size, bool)
    robust_fr = np.ones(sc.n_frames, bool)
    hist = []
    ref = orc.make_object_map(F, G, W, M, u, di, dj)
    hist.append(orc.calc_error(F, G, W, M, *ref, u, di, dj)["total"])
    for i in range(iters):
        st = sched_orc[min(i, len(sched_orc) - 1)]
        ref = orc.make_object_map(F, G, W, M, u, di, dj)
        u, _, stack = orc.update_pixel_map(F, G, W, M, *ref, u, di, dj, st["half_ss"],
                                           st["half_fs"], None, True, threads=THREADS,
                                           return_stack=True)
        robust_px &= unique_mask(stack)
        del stack
        if st["update_translations"]:
            di, dj, errs = orc.update_translations(F, G, W, M, *ref, u, di, dj, st["t_half"],
                                                   st["t_half"], return_errors=True)
            for fr, e in errs.items():
                flat = np.sort(e.ravel())
                if not (flat[1] - flat[0]) > MARGIN * abs(flat[0]):
                    robust_fr[fr] = False
        hist.append(orc.calc_error(F, G, W, M, *ref, u, di, dj)["total"])
        print(f"cfg{cfg_id} oracle iteration {i + 1}: robust pixels {robust_px.mean():.5f}",
              flush=True)
    ref_hist = np.array([h.total for h in L.history])
    assert np.array_equal(u, L.pixel_map.u), "oracle loop != reference loop (u)"
    assert np.array_equal(di, L.translations.di) and np.array_equal(dj, L.translations.dj)
    assert np.array_equal(np.array(hist), ref_hist), (hist, ref_hist)
    mask = np.zeros(W.shape, bool)
    mask[rows[robust_px], cols[robust_px]] = True
    return {"frames_sha": digest(sc.frames), "iters": np.array(iters),
            "loop_u": L.pixel_map.u.astype(np.float32),
            "loop_di": L.translations.di, "loop_dj": L.translations.dj,
            "loop_hist": ref_hist, "robust_px": np.packbits(mask.ravel()),
            "robust_fr": robust_fr, "loop_ref_i": L.reference.i_ref.astype(np.float32),
            "loop_ref_valid": np.packbits((L.reference.wsum > 0).ravel()),
            "loop_ref_origin": np.array(L.reference.origin)}


def cfg0loop():
    from pxst import recon
    sched = [recon.IterationSettings(window=recon.SearchWindow(3, 3),
                                     options=recon.UpdateOptions(True, False, 0.0),
                                     update_translations=True,
                                     translation_window=recon.SearchWindow(1, 1))]
    return loop_golden(0, sched, [dict(half_ss=3, half_fs=3, update_translations=True,
                                       t_half=1)], 2)


def cfg1loop():
    from pxst import recon
    c = CONFIGS[1]
    sched = [recon.IterationSettings(window=recon.SearchWindow(c.half_ss, c.half_fs),
                                     options=recon.UpdateOptions(True, False, 0.0),
                                     update_translations=False)]
    return loop_golden(1, sched, [dict(half_ss=c.half_ss, half_fs=c.half_fs,
                                       update_translations=False)], c.iters)


def cfg2ref():
    from pxst import recon
    s = make_scan(2)
    sc = s.scan
    t = time.time()
    R = recon.make_reference(sc, s.w, s.m, s.u0, s.t0)
    print(f"cfg2 make_reference {time.time() - t:.0f} s", flush=True)
    return {"frames_sha": digest(sc.frames), "ref_i": R.i_ref.astype(np.float32),
            "ref_valid": np.packbits((R.wsum > 0).ravel()), "ref_shape": np.array(R.i_ref.shape),
            "ref_origin": np.array(R.origin),
            "ref_wsum_rowsum": R.wsum.sum(axis=1), "ref_i_rowsum": R.i_ref.sum(axis=1)}


def main():
    live_reference.load()
    jobs = {"cfg0loop": ("loop0", cfg0loop), "cfg1loop": ("loop1", cfg1loop),
            "cfg2ref": ("ref2", cfg2ref)}
    names = sys.argv[1:] or list(jobs)
    for n in names:
        fname, fn = jobs[n]
        out = fn()
        np.savez_compressed(os.path.join(HERE, f"{fname}.npz"), **out)
        print("wrote", fname, sorted(out), flush=True)


if __name__ == "__main__":
    main()

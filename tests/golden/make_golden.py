"""Write golden vectors from the LIVE reference (``/root/reference/pkg/src/pxst``).

Run in the build container (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Inputs are the seeded synthetic scans of ``paper_2003_12726_b200.synth``
(regenerated bit-exactly from the seed; a SHA-256 of the frame stack is
stored to detect generator drift).  Outputs are the reference's own results:

* ``cfg0.npz``: make_reference, update_pixel_map (R=3, refine), the same
  without refinement, update_translations (+-2 integer and +-1 at 0.5 px),
  calc_error, and a 2-iteration run_main_loop history.
* ``cfg1.npz``: make_reference (full), update_pixel_map (R=5) on the
  row band ROI 112:144 (bit-exact slice of the full run),
  update_translations (+-3) for a 9-frame good subset, calc_error on the
  band.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import live_reference  # noqa: E402
from paper_2003_12726_b200.synth import make_scan  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg0(pxst):
    from pxst import recon
    from pxst.data_model import PixelTranslations
    s = make_scan(0)
    sc, w, m, u, t = s.scan, s.w, s.m, s.u0, s.t0
    out = {"frames_sha": digest(sc.frames)}
    R = recon.make_reference(sc, w, m, u, t)
    out.update(ref_i=R.i_ref, ref_w=R.wsum, ref_origin=np.array(R.origin))
    U, E = recon.update_pixel_map(sc, w, m, R, u, t, recon.SearchWindow(3, 3))
    out.update(upm_u=U.u, upm_err=E)
    U2, E2 = recon.update_pixel_map(sc, w, m, R, u, t, recon.SearchWindow(3, 3),
                                    recon.UpdateOptions(quadratic_refinement=False))
    out.update(upm_noref_u=U2.u, upm_noref_err=E2)
    T = recon.update_translations(sc, w, m, R, U, t, recon.SearchWindow(2, 2))
    out.update(ut_di=T.di, ut_dj=T.dj)
    T2 = recon.update_translations(sc, w, m, R, U, t, recon.SearchWindow(1, 1, subpixel_grid=0.5))
    out.update(uts_di=T2.di, uts_dj=T2.dj)
    M = recon.calc_error(sc, w, m, R, U, T)
    out.update(ce_total=np.array(M.total), ce_per_frame=M.per_frame, ce_per_pixel=M.per_pixel,
               ce_plane=M.reference_plane, ce_var=M.variance)
    sched = [recon.IterationSettings(window=recon.SearchWindow(3, 3),
                                     options=recon.UpdateOptions(True, False, 0.0),
                                     update_translations=True,
                                     translation_window=recon.SearchWindow(1, 1))]
    L = recon.run_main_loop(sc, w, m, u, t, schedule=sched, max_iters=2, tol=-np.inf)
    out.update(loop_u=L.pixel_map.u, loop_di=L.translations.di, loop_dj=L.translations.dj,
               loop_hist=np.array([h.total for h in L.history]), loop_ref_i=L.reference.i_ref,
               loop_ref_origin=np.array(L.reference.origin))
    return out


def cfg1(pxst):
    from pxst import recon
    from pxst.data_model import Roi, ScanData
    from dataclasses import replace
    s = make_scan(1)
    sc, w, m, u, t = s.scan, s.w, s.m, s.u0, s.t0
    out = {"frames_sha": digest(sc.frames)}
    R = recon.make_reference(sc, w, m, u, t)
    out.update(ref_i=R.i_ref, ref_w=R.wsum, ref_origin=np.array(R.origin))
    band = Roi(112, 144, 0, sc.shape[1])
    U, E = recon.update_pixel_map(sc, w, m, R, u, t, recon.SearchWindow(5, 5), roi=band,
                                  threads=os.cpu_count() or 1)
    out.update(band=np.array(band.as_tuple()), upm_u=U.u[:, 112:144], upm_err=E[112:144])
    sub = np.zeros(sc.n_frames, dtype=bool)
    sub[[0, 5, 17, 33, 60, 61, 88, 100, 120]] = True
    sc_sub = replace(sc, good_frames=sub)
    T = recon.update_translations(sc_sub, w, m, R, u, t, recon.SearchWindow(3, 3))
    out.update(ut_subset=sub, ut_di=T.di, ut_dj=T.dj)
    M = recon.calc_error(sc, w, m, R, u, t, roi=band)
    out.update(ce_per_pixel=M.per_pixel[112:144], ce_var=M.variance[112:144],
               ce_per_frame=M.per_frame, ce_total=np.array(M.total), ce_plane=M.reference_plane)
    return out


def main():
    pxst = live_reference.load()
    for name, fn in (("cfg0", cfg0), ("cfg1", cfg1)):
        out = fn(pxst)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print("wrote", name, sorted(out))


if __name__ == "__main__":
    main()

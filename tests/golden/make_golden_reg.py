"""Golden vectors for the pixel-map regularisation rows
from the LIVE reference; run in the build container:

    python tests/golden/make_golden_reg.py

Writes ``reg0.npz`` (config-0 scan of ``paper_2003_12726_b200.synth``):

* ``sm_*``: ``recon._smooth_displacement`` on the config-0 initial
  displacement (both components, sigma 2.5) with the work-set support;
* ``ig_*``: ``integration.integrate_gradient`` on a seeded 40x56 field with
  a 4 % random hole mask (potential, iterations, residual);
* ``upm_s*`` / ``upm_i*`` / ``upm_si*``: ``update_pixel_map`` with
  sigma=2, with integrate=True, and with both (sigma=1.5);
* ``loop_*``: ``run_main_loop`` with ``default_schedule(3)`` (sigma 5, 3, 1,
  integrate, translations from iteration 2), history and final state;
* ``sh_*``: ``analysis.split_half_recon`` (window +-2, seed 3) maps,
  histograms and sigma; ``shb_*``: the raw split bits of the first 4096
  flat indices for seeds 0 and 12345;
* ``fd_*``: ``geometry.fit_defocus_registration`` on the config-0 scan with
  physical translations of a true z1 = 0.05 m (7-point grid, and a 3x3
  astigmatic grid).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import live_reference  # noqa: E402
from paper_2003_12726_b200.synth import make_scan  # noqa: E402


def defocus_scan(s, z1=0.05):
    """The config-0 scan with translations [m] whose projection at focus
    distance z1 gives the scan's pixel translations."""
    from dataclasses import replace
    sc, t = s.scan, s.t0
    mag = (z1 + sc.distance) / z1
    tr = np.stack([t.di * sc.x_pixel_size / mag, t.dj * sc.y_pixel_size / mag,
                   np.zeros_like(t.di)], axis=1)
    return replace(sc, translations=tr)


def main():
    live_reference.load()
    from dataclasses import replace
    from pxst import analysis, geometry, integration, recon
    s = make_scan(0)
    sc, w, m, u, t = s.scan, s.w, s.m, s.u0, s.t0
    out = {}
    support = m.mask & (w.w > 0)
    ss, fs = support.shape
    ident = np.stack(np.meshgrid(np.arange(ss, dtype=np.float64),
                                 np.arange(fs, dtype=np.float64), indexing="ij"))
    for c in range(2):
        out[f"sm_{c}"] = recon._smooth_displacement(u.u[c] - ident[c], support, 2.5)

    rng = np.random.default_rng(7)
    gx = rng.normal(size=(40, 56))
    gy = rng.normal(size=(40, 56))
    mask = rng.random((40, 56)) > 0.04
    res = integration.integrate_gradient(gx, gy, mask)
    out.update(ig_gx=gx, ig_gy=gy, ig_mask=mask, ig_phi=res.phi,
               ig_iters=np.array(res.iterations), ig_res=np.array(res.residual),
               ig_conv=np.array(res.converged))

    R = recon.make_reference(sc, w, m, u, t)
    win = recon.SearchWindow(3, 3)
    for tag, opts in (("s", recon.UpdateOptions(sigma=2.0)),
                      ("i", recon.UpdateOptions(integrate=True)),
                      ("si", recon.UpdateOptions(sigma=1.5, integrate=True))):
        U, E = recon.update_pixel_map(sc, w, m, R, u, t, win, opts)
        out[f"upm_{tag}_u"] = U.u
        out[f"upm_{tag}_err"] = E

    L = recon.run_main_loop(sc, w, m, u, t, schedule=recon.default_schedule(3), max_iters=3,
                            tol=-np.inf)
    out.update(loop_u=L.pixel_map.u, loop_di=L.translations.di, loop_dj=L.translations.dj,
               loop_hist=np.array([h.total for h in L.history]))
    S = analysis.split_half_recon(sc, w, m, R, u, t, recon.SearchWindow(2, 2), seed=3)
    out.update(sh_ua=S.map_a.u, sh_ub=S.map_b.u, sh_hss=S.hist_ss, sh_hfs=S.hist_fs,
               sh_sigma=np.array(S.sigma))
    for sd in (0, 12345):
        out[f"shb_{sd}"] = analysis._splitmix(sd, np.arange(4096, dtype=np.uint64))
    sc2 = defocus_scan(s)
    grid = 0.05 * np.array([0.8, 0.9, 0.95, 1.0, 1.05, 1.1, 1.25])
    F = geometry.fit_defocus_registration(sc2, w, m, grid)
    out.update(fd_grid=grid, fd_contrast=F.contrast, fd_z1=np.array([F.z1_ss, F.z1_fs]))
    F2 = geometry.fit_defocus_registration(sc2, w, m, 0.05 * np.array([0.9, 1.0, 1.1]),
                                           astigmatic=True)
    out.update(fd2_contrast=F2.contrast, fd2_cands=F2.candidates,
               fd2_z1=np.array([F2.z1_ss, F2.z1_fs]))
    np.savez_compressed(os.path.join(HERE, "reg0.npz"), **out)
    print("wrote reg0.npz:", {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()

"""Small config-0 workload touching every kernel family once (for
compute-sanitizer, tools/sanitize.sh)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2003_12726_b200 import engine  # noqa: E402
from paper_2003_12726_b200.synth import make_scan  # noqa: E402

s = make_scan(0)
ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
u, (di, dj) = ds.upload_u(s.u0.u), ds.upload_t(s.t0.di, s.t0.dj)
ref = ds.object_map(u, di, dj)                                        # K1
u1, _ = ds.pixel_map_search(ref, u, di, dj, 3, 3)                     # K2 fast/slow/epilogue
u2, _ = ds.pixel_map_search(ref, u, di, dj, 1, 1, 0.5)                # K2 generic
u3, _ = ds.pixel_map_search(ref, u, di, dj, 0, 4)                     # K2 1-D window (slow rows)
d1, j1 = ds.translation_search(ref, u1, di, dj, 3, 3)                 # K3 integer
d2, j2 = ds.translation_search(ref, u1, di, dj, 2, 2, 0.25)           # K3 phase groups
d3, j3 = ds.translation_search(ref, u1, di, dj, 1, 1, 0.4)            # K3 generic
geom = ds.geometry_async(u1, d1, j1)
metrics, pend = ds.error_maps_and_next_object(ref, u1, d1, j1, geom)  # fused K4 + K1
nref = pend.resolve()
metrics2 = ds.error_maps(nref, u1, d1, j1)                            # K4
uu = u1.clone()
ds.smooth_displacement(uu, 2.0)                                        # regularisation
ds.project_irrotational(uu.clone(), solver="cg", maxiter=200)
ds.project_irrotational(uu.clone(), solver="mgcg")
torch.cuda.synchronize()
print("sanitize workload done", float(metrics[0].item()), float(metrics2[0].item()))

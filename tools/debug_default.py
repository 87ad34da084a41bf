import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
u, t = s.u0, s.t0
ref = pb.make_reference(s.scan, s.w, s.m, u, t)
win = pb.SearchWindow(4, 4)
for name, opts in [("plain", pb.UpdateOptions()), ("sigma5", pb.UpdateOptions(sigma=5.0)),
                   ("integ", pb.UpdateOptions(integrate=True)),
                   ("both", pb.UpdateOptions(sigma=5.0, integrate=True))]:
    un, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, u, t, win, opts)
    d = un.u - u.u
    print(f"{name:6s} shift {d.min():.3g}..{d.max():.3g}")
ds = engine.SCAN_CACHE.get(s.scan, s.w, s.m, None)
un, e = pb.update_pixel_map(s.scan, s.w, s.m, ref, u, t, win, pb.UpdateOptions(sigma=5.0))
for solver in ("cg", "mgcg"):
    ut = ds.upload_u(un.u)
    info = ds.project_irrotational(ut, solver=solver)
    d = ut.cpu().numpy() - un.u
    print(f"project[{solver}] it {info.iterations} res {info.residual:.3e} conv {info.converged} shift {d.min():.3g}..{d.max():.3g}")
print("components", ds._support_components)

import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2003_12726_b200 as pb
from oracle import pxst_oracle as orc
from test_gpu_parity import _tiny, _orc_args, ref_from
g = dict(np.load('/root/repo/tests/golden/cfg0.npz'))
from paper_2003_12726_b200.synth import make_scan
s = make_scan(0)
ref = ref_from(g)
U = pb.PixelMap(g["upm_u"]); T = pb.PixelTranslations(g["ut_di"], g["ut_dj"])
M = pb.calc_error(s.scan, s.w, s.m, ref, U, T)
for k, gk in (("per_frame","ce_per_frame"),("per_pixel","ce_per_pixel"),("reference_plane","ce_plane"),("variance","ce_var")):
    a = getattr(M, k); b = g[gk]
    ok = b != 0
    rel = np.abs(a[ok]-b[ok])/np.abs(b[ok])
    i = np.argmax(rel)
    print(k, rel.max(), a[ok][i], b[ok][i], np.sum(rel > 1e-4))
print("total", M.total, float(g["ce_total"]))
sc, w, m, u, t = _tiny(seed=17)
ref = pb.make_reference(sc, w, m, u, t)
shifted = pb.PixelMap(u.u - np.array([2.0, -1.0])[:, None, None])
for half in (3, 4, 5):
    un, e = pb.update_pixel_map(sc, w, m, ref, shifted, t, pb.SearchWindow(half, half), pb.UpdateOptions(quadratic_refinement=False))
    uo, eo, st = orc.update_pixel_map(*_orc_args(sc, w, m), ref.i_ref, ref.wsum, ref.origin, shifted.u, t.di, t.dj, half, half, quadratic_refinement=False, return_stack=True)
    d = np.abs(un.u - uo).max(axis=0)
    print("half", half, "mismatch", np.sum(d > 0), "of", d.size, "vs truth", np.sum(np.abs(uo - u.u).max(axis=0) > 1e-9))

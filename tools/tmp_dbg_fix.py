import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine
g = dict(np.load("tests/golden/cfg1.npz"))
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
ref = pb.make_reference(s.scan, s.w, s.m, s.u0, s.t0)
gi, gw = g["ref_i"], g["ref_w"]
ok = gw > 0
rel = np.abs(ref.i_ref - gi)[ok] / np.abs(gi[ok])
relw = np.abs(ref.wsum - gw)[ok] / np.abs(gw[ok])
print(os.environ.get("PXST_FIX_FINE_W"), os.environ.get("PXST_FIX_NO_REGION"), "valid eq", np.array_equal(ref.wsum > 0, ok), "max rel i", rel.max(), "n>1e-5", (rel > 1e-5).sum(), "max rel w", relw.max(), "n>1e-5", (relw>1e-5).sum())
idx = np.argwhere(ok)[np.argsort(-rel)[:5]]
for (r, c) in idx:
    print(r, c, gi[r, c], ref.i_ref[r, c], gw[r, c], ref.wsum[r, c])

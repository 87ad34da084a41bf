import sys, os
sys.path.insert(0, '/root/repo')
os.environ["PXST_DEBUG"] = "1"
import numpy as np, torch
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
for c in (0, 1):
    s = make_scan(c)
    ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
    u = ds.upload_u(s.u0.u); di, dj = ds.upload_t(s.t0.di, s.t0.dj)
    ref = ds.object_map(u, di, dj)
    print("cfg", c, "ref", ref.shape, ref.origin, flush=True)
    ds.translation_search(ref, u, di, dj, 3, 3)
    torch.cuda.synchronize()

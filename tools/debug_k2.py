import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
s = make_scan(0)
ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
u = ds.upload_u(s.u0.u); di, dj = ds.upload_t(s.t0.di, s.t0.dj)
ref = ds.object_map(u, di, dj)
torch.cuda.synchronize(); print("object map ok", flush=True)
for half in (int(a) for a in sys.argv[1:]):
    try:
        uo, e = ds.pixel_map_search(ref, u, di, dj, half, half)
        torch.cuda.synchronize(); print("half", half, "ok", float(e.sum()), flush=True)
    except Exception as ex:
        print("half", half, "FAILED", ex, flush=True); break

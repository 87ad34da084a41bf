"""Host timestamps inside make_reference (no extra synchronisation)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from dataclasses import replace
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine, recon
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
pinned = torch.empty(s.scan.frames.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[...] = s.scan.frames
scan = replace(s.scan, frames=pinned.numpy())
T = {}
def mark(k): T.setdefault(k, []).append(time.perf_counter())
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        mark(name + ">"); r = f(*a, **k); mark(name + "<"); return r
    setattr(obj, name, g)
for n in ("_upload_frames", "upload_u", "upload_t", "bbox", "object_splat", "object_finish"):
    wrap(engine.DeviceScan, n)
wrap(engine.DeviceScan, "__init__")
wrap(recon, "_ref_image")
for it in range(12):
    engine.SCAN_CACHE.clear()
    torch.cuda.synchronize()
    mark("start")
    ref = pb.make_reference(scan, s.w, s.m, s.u0, s.t0)
    mark("end")
ev = sorted((t, k) for k, v in T.items() for t in v)
starts = [i for i, (t, k) in enumerate(ev) if k == "start"]
for i in starts[-2:]:
    t0 = ev[i][0]
    j = i
    while j < len(ev) and (j == i or ev[j][1] != "start"):
        print(f"  {ev[j][1]:22s} {(ev[j][0] - t0) * 1e3:7.3f} ms")
        j += 1
    print()

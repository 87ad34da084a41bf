"""Host-side breakdown of one bench e2e step (drop-in API, cold device cache)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from dataclasses import replace
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
pinned = torch.empty(s.scan.frames.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[...] = s.scan.frames
scan = replace(s.scan, frames=pinned.numpy())
win = pb.SearchWindow(5, 5)
def T(label, fn, acc):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    acc.setdefault(label, []).append(1e3 * (time.perf_counter() - t)); return r
acc = {}
for it in range(6):
    engine.SCAN_CACHE.clear()
    ds = T("scan upload + K0", lambda: engine.SCAN_CACHE.get(scan, s.w, s.m, None), acc)
    T("digest lookup", lambda: engine.SCAN_CACHE.get(scan, s.w, s.m, None), acc)
    ref = T("make_reference", lambda: pb.make_reference(scan, s.w, s.m, s.u0, s.t0), acc)
    u, e = T("update_pixel_map", lambda: pb.update_pixel_map(scan, s.w, s.m, ref, s.u0, s.t0, win), acc)
    T("calc_error", lambda: pb.calc_error(scan, s.w, s.m, ref, u, s.t0), acc)
for k, v in acc.items():
    print(f"{k:20s} {np.median(v[2:]):8.3f} ms")

"""Breakdown of the bench's e2e step (config 1, drop-in API, cold device
cache): each engine operation is bracketed by device synchronisations and
timed on the host, so the sum is an upper bound of the step and each line
is that operation's serial cost."""
import collections, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from dataclasses import replace
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine, recon
from paper_2003_12726_b200.synth import make_scan

acc = collections.defaultdict(float)
def wrap(obj, name, label):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); acc[label] += time.perf_counter() - t
        return r
    setattr(obj, name, g)
for n in ("to_device", "to_host_many"):
    wrap(engine, n, n)
recon.to_host_many = engine.to_host_many
for n in ("object_map", "pixel_map_search", "error_maps", "upload_u", "upload_t"):
    wrap(engine.DeviceScan, n, "DeviceScan." + n)
wrap(engine.DeviceScan, "__init__", "DeviceScan.__init__ (incl. uploads, K0)")
s = make_scan(1)
pinned = torch.empty(s.scan.frames.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[...] = s.scan.frames
scan = replace(s.scan, frames=pinned.numpy())
win = pb.SearchWindow(5, 5)
def one():
    engine.SCAN_CACHE.clear()
    ref = pb.make_reference(scan, s.w, s.m, s.u0, s.t0)
    u, e = pb.update_pixel_map(scan, s.w, s.m, ref, s.u0, s.t0, win)
    pb.calc_error(scan, s.w, s.m, ref, u, s.t0)
for _ in range(3): one()
acc.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
n = 10
for _ in range(n): one()
torch.cuda.synchronize(); T = (time.perf_counter() - t0) / n
print(f"step (serialised) {T*1e3:.3f} ms")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  {k:45s} {v / n * 1e3:8.3f} ms")

"""Per-call host times of the e2e step (no extra synchronisation): each
drop-in call returns host arrays, so its wall time is its critical path.
python tools/e2e_calls.py [package_root]"""
import sys, time
root = sys.argv[1] if len(sys.argv) > 1 else '/root/repo'
sys.path.insert(0, root)
import numpy as np, torch
from dataclasses import replace
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
print(pb.__file__)
s = make_scan(1)
pinned = torch.empty(s.scan.frames.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[...] = s.scan.frames
scan = replace(s.scan, frames=pinned.numpy())
win = pb.SearchWindow(5, 5)
acc = np.zeros(4)
def one(rec):
    t0 = time.perf_counter()
    engine.SCAN_CACHE.clear()
    ref = pb.make_reference(scan, s.w, s.m, s.u0, s.t0)
    t1 = time.perf_counter()
    u, e = pb.update_pixel_map(scan, s.w, s.m, ref, s.u0, s.t0, win)
    t2 = time.perf_counter()
    pb.calc_error(scan, s.w, s.m, ref, u, s.t0)
    t3 = time.perf_counter()
    if rec:
        acc[:] += [t1 - t0, t2 - t1, t3 - t2, t3 - t0]
for _ in range(3): one(False)
torch.cuda.synchronize()
for _ in range(20): one(True)
print("make_reference %.3f  update_pixel_map %.3f  calc_error %.3f  step %.3f ms" % tuple(acc / 20 * 1e3))

"""cProfile of the bench's e2e step (drop-in API, cold device cache) on config 1."""
import cProfile, pstats, sys, time
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
def one():
    engine.SCAN_CACHE.clear()
    ref = pb.make_reference(scan, s.w, s.m, s.u0, s.t0)
    u, e = pb.update_pixel_map(scan, s.w, s.m, ref, s.u0, s.t0, win)
    pb.calc_error(scan, s.w, s.m, ref, u, s.t0)
for _ in range(3): one()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): one()
torch.cuda.synchronize()
print("ms/step", (time.perf_counter() - t) * 100)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): one()
torch.cuda.synchronize(); pr.disable()
st = pstats.Stats(pr); st.sort_stats('cumulative').print_stats(45)
st.sort_stats('tottime').print_stats(30)

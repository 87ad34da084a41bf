"""Where the time of a cold DeviceScan construction goes (e2e path)."""
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
import cProfile, pstats
for _ in range(3):
    engine.SCAN_CACHE.clear(); torch.cuda.synchronize()
    t = time.perf_counter(); ds = engine.SCAN_CACHE.get(scan, s.w, s.m, None); torch.cuda.synchronize()
    print(f"cold scan: {1e3*(time.perf_counter()-t):.3f} ms")
engine.SCAN_CACHE.clear()
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    engine.SCAN_CACHE.clear(); ds = engine.SCAN_CACHE.get(scan, s.w, s.m, None); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(14)

"""cProfile of make_reference (cold device cache) on config 1."""
import cProfile, pstats, sys
sys.path.insert(0, '/root/repo')
import torch
from dataclasses import replace
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
pinned = torch.empty(s.scan.frames.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[...] = s.scan.frames
scan = replace(s.scan, frames=pinned.numpy())
def one():
    engine.SCAN_CACHE.clear()
    pb.make_reference(scan, s.w, s.m, s.u0, s.t0)
for _ in range(5): one()
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(20): one()
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)

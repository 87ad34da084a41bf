"""Device-memory stability of the drop-in API: many make_reference ->
update_pixel_map -> update_translations -> calc_error rounds on fresh host
arrays (the scan cache evicts, the library's stream-ordered pool and torch's
allocator recycle), free device memory sampled with cudaMemGetInfo.
python tools/leak_check.py [rounds]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from dataclasses import replace
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200.synth import make_scan
n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
s = make_scan(1)
free = []
for i in range(n):
    sc = replace(s.scan, frames=s.scan.frames.copy())       # a new stack every round
    u = pb.PixelMap(s.u0.u.copy())
    ref = pb.make_reference(sc, s.w, s.m, u, s.t0)
    un, _ = pb.update_pixel_map(sc, s.w, s.m, ref, u, s.t0, pb.SearchWindow(2 + i % 3, 2 + i % 3))
    if i % 4 == 0:
        pb.update_translations(sc, s.w, s.m, ref, un, s.t0, pb.SearchWindow(1, 1))
    pb.calc_error(sc, s.w, s.m, ref, un, s.t0)
    if i % 10 == 9:
        torch.cuda.synchronize()
        f, tot = torch.cuda.mem_get_info()
        free.append(f)
        print(f"round {i + 1}: free {f / 2**20:.0f} MiB, torch allocated {torch.cuda.memory_allocated() / 2**20:.0f} MiB, reserved {torch.cuda.memory_reserved() / 2**20:.0f} MiB", flush=True)
drift = (free[1] - free[-1]) / 2**20
print(f"free-memory drift from round 20 to round {n}: {drift:.0f} MiB")
sys.exit(1 if drift > 64 else 0)

"""run_main_loop with the reference's default_schedule (sigma 5/3/1, integrate,
translations from iteration 2) on config 1 through the drop-in API."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2003_12726_b200 as pb
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
for n in (1, 3, 3):
    torch.cuda.synchronize(); t = time.perf_counter()
    L = pb.run_main_loop(s.scan, s.w, s.m, s.u0, s.t0, schedule=pb.default_schedule(n), max_iters=n,
                         tol=-np.inf)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"default_schedule({n}): {dt*1e3:.1f} ms total, history {np.round([h.total for h in L.history], 1)}")

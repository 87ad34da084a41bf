"""Time the 8(f) regularisation kernels (smoothing, device CG vs MG-PCG) at config sizes."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan_device
for cfg_id in (1, 3):
    dev = torch.device('cuda')
    s, frames = make_scan_device(cfg_id, dev)
    ds = engine.DeviceScan(None, s.scan.good_frames, s.w.w, s.m.mask, frames_dev=frames)
    u = ds.upload_u(s.u0.u)
    for sigma in (5.0, 1.0):
        uu = u.clone(); ds.smooth_displacement(uu, sigma); torch.cuda.synchronize()
        t = time.perf_counter(); ds.smooth_displacement(uu, sigma); torch.cuda.synchronize()
        print(f"cfg{cfg_id} smooth sigma={sigma}: {1e3*(time.perf_counter()-t):.3f} ms", flush=True)
    outs = {}
    for solver in ("cg", "mgcg"):
        uu = u.clone()
        ds.project_irrotational(uu.clone(), solver=solver); torch.cuda.synchronize()
        t = time.perf_counter(); info = ds.project_irrotational(uu, solver=solver)
        torch.cuda.synchronize()
        outs[solver] = uu
        print(f"cfg{cfg_id} project_irrotational[{solver}]: {1e3*(time.perf_counter()-t):.1f} ms, "
              f"{info.iterations} iterations, residual {info.residual:.3e}, converged {info.converged}",
              flush=True)
    d = (outs["cg"] - outs["mgcg"]).abs().max().item()
    print(f"cfg{cfg_id} max |u_cg - u_mgcg| = {d:.3e} px", flush=True)
    del frames, ds
    torch.cuda.empty_cache()

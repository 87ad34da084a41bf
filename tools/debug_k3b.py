import sys, os
sys.path.insert(0, '/root/repo')
os.environ["PXST_DEBUG"] = "1"
import numpy as np, torch
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan_device
c = int(sys.argv[1])
s, fr = make_scan_device(c, torch.device("cuda", 0))
ds = engine.DeviceScan(None, s.scan.good_frames, s.w.w, s.m.mask, frames_dev=fr)
u = ds.upload_u(s.u0.u); di, dj = ds.upload_t(s.t0.di, s.t0.dj)
ref = ds.object_map(u, di, dj)
v = ref.valid.cpu().numpy()
print("cfg", c, "ref", ref.shape, ref.origin, "invalid cells", int((v == 0).sum()), "interior invalid", int((v[20:-20, 20:-20] == 0).sum()), flush=True)
rows, cols = np.nonzero(v[20:-20, 20:-20] == 0)
print("first invalid interior cells", list(zip(rows[:10] + 20, cols[:10] + 20)))
ds.translation_search(ref, u, di, dj, s.cfg.t_half_ss, s.cfg.t_half_fs, s.cfg.t_subpixel_grid)
torch.cuda.synchronize()

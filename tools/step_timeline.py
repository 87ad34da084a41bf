"""Event timeline of the bench's steady-state step (config 1): where the
iteration's 1.2x ms go between the K2 call, the fused error pass and gaps."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
cfg = s.cfg
u, (di, dj) = ds.upload_u(s.u0.u), ds.upload_t(s.t0.di, s.t0.dj)
st = torch.cuda.current_stream()
geom = ds.geometry_async(u, di, dj)
pend = None
rows = []
for it in range(12):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record(st)
    dref = pend.resolve() if pend else ds.object_map(u, di, dj, geom=geom)
    ev[1].record(st)
    u1, _ = ds.pixel_map_search(dref, u, di, dj, cfg.half_ss, cfg.half_fs, None, True, geom=geom)
    ev[2].record(st)
    nxt = ds.geometry_async(u1, di, dj)
    ev[3].record(st)
    _, pend = ds.error_maps_and_next_object(dref, u1, di, dj, nxt)
    ev[4].record(st)
    u, geom = u1, nxt
    torch.cuda.synchronize()
    rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)] + [ev[0].elapsed_time(ev[4])])
r = np.array(rows[3:]) * 1e3
print("object(us) K2(us) geom-enqueue(us) fused(us) total(us)")
print(np.round(r.mean(axis=0), 1))

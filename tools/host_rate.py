"""Host enqueue time per bench step (config 1) against its device time: the
device queue is kept full by a leading spin kernel, so perf_counter around
step() measures the host's launch work alone.  python tools/host_rate.py"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2003_12726_b200 import engine
from paper_2003_12726_b200.synth import make_scan
s = make_scan(1)
ds = engine.DeviceScan(s.scan.frames, s.scan.good_frames, s.w.w, s.m.mask)
u_t = ds.upload_u(s.u0.u); di_t, dj_t = ds.upload_t(s.t0.di, s.t0.dj)
ds.ready(frame_stats=True); ds.absmax()
stream = torch.cuda.current_stream()
seq = bench.Sequence(ds, s.cfg, u_t, di_t, dj_t, stream)
for _ in range(30): seq.step()
torch.cuda.synchronize()
N = 60
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(20e-3 * 1.965e9))       # 20 ms head start for the host
host = []
a.record(stream)
for i in range(N):
    t0 = time.perf_counter(); seq.step(); host.append(time.perf_counter() - t0)
b.record(stream)
t_enq = sum(host)
torch.cuda.synchronize()
print("host enqueue per step: mean %.3f ms, median %.3f, max %.3f; device per step %.3f ms"
      % (np.mean(host) * 1e3, np.median(host) * 1e3, np.max(host) * 1e3, (a.elapsed_time(b) - 20) / N))
if len(sys.argv) > 1:
    import cProfile, pstats
    torch.cuda.synchronize()
    torch.cuda._sleep(int(20e-3 * 1.965e9))
    pr = cProfile.Profile()
    pr.enable()
    for i in range(60):
        seq.step()
    pr.disable()
    torch.cuda.synchronize()
    st = pstats.Stats(pr)
    st.sort_stats("cumulative").print_stats(45)

"""Pinned host->device bandwidth for a config-1-size stack: one copy vs chunks on 2 streams."""
import time, torch
n = 121 * 256 * 512
h = torch.empty(n, dtype=torch.float32, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device='cuda')
def run(chunks, streams):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize(); t = time.perf_counter()
    step = (n + chunks - 1) // chunks
    for i in range(chunks):
        with torch.cuda.stream(ss[i % streams]):
            d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
    torch.cuda.synchronize(); return time.perf_counter() - t
for c, s in [(1,1),(1,1),(4,2),(8,2),(8,4),(16,4)]:
    dt = min(run(c, s) for _ in range(5))
    print(f"chunks {c:2d} streams {s}: {dt*1e3:.3f} ms  {4*n/dt/1e9:.1f} GB/s")

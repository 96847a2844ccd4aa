"""Host overhead of one hull call (wall clock) vs its device time (CUDA events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1501_04706_b200 import dataio, hull
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
x, y = dataio.gen_uniform_device(n, 1)
torch.cuda.synchronize()
s = torch.cuda.current_stream().cuda_stream
out = tuple(torch.empty(max(n, 2), dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.int64))
for _ in range(5):
    hull.run_device(x, y, 1, stream=s, out=out)
for stats in (True, False):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    K = 50
    for _ in range(K):
        r = hull.run_device(x, y, 1, stream=s, out=out, stats=stats)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / K * 1e3
    print(f"n={n} stats={stats}: wall {wall:.3f} ms/call, events {e0.elapsed_time(e1)/K:.3f} ms/call", flush=True)
r = hull.run_device(x, y, 1, stream=s, out=out, timings=True)
print("device phases", r.kernels)

"""Profiling driver: R hulls of one device-resident workload (for ncu; never a bench number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1501_04706_b200 import dataio, hull  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "uniform"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 20_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if kind == "uniform":
    x, y = dataio.gen_uniform_device(n, 1)
elif kind == "disk":
    x, y = dataio.gen_disk_device(n, 1)
else:
    hx, hy = dataio.gen_circle(n, 1)
    x, y = torch.from_numpy(hx).cuda(), torch.from_numpy(hy).cuda()
torch.cuda.synchronize()
for _ in range(reps):
    r = hull.run_device(x, y, 1, timings=True)
    print(kind, n, "h", r.h, "rounds", r.rounds, r.kernels, r.phase_timings, flush=True)
    print("   round end (ms since K1 start):", [round(t, 4) for t in r.round_end_ms], flush=True)

"""Determinism of one hull call under another process sharing the GPU."""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1501_04706_b200 import dataio, hull
kind = sys.argv[1]; n = int(sys.argv[2]); reps = int(sys.argv[3])
hx, hy = dataio.gen_uniform(n, 5)
x, y = torch.from_numpy(hx).cuda(), torch.from_numpy(hy).cuda()
ids = torch.arange(n, dtype=torch.int32, device='cuda') * 3 + 7 if kind == 'ids' else None
ref = hull.run_device(x, y, 1, ids=ids, stats=False)
want = (ref.h, ref.x.cpu().numpy().tobytes())
bad = 0
for _ in range(reps):
    r = hull.run_device(x, y, 1, ids=ids, stats=False)
    if (r.h, r.x.cpu().numpy().tobytes()) != want: bad += 1
print(kind, n, "h", ref.h, "bad", bad, flush=True)

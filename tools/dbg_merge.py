import sys, torch, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_1501_04706_b200 import dataio, hull, shard
x, y = dataio.gen_uniform_device(40_000_000, 1)
whole = hull.run_device(x, y, 1, stats=False)
parts = []
for r in range(2):
    f, c = shard.shard_range(40_000_000, 2, r)
    f = r * 20_000_000; c = 20_000_000
    dh = hull.run_device(x[f:f+c].contiguous(), y[f:f+c].contiguous(), 1, stats=False)
    parts.append((dh.x.clone(), dh.y.clone(), dh.indices.to(torch.int64) + f))
    print("shard", r, dh.h)
for width in (0, 64, 512, 1024, 2048):
    w = width or max(p[0].shape[0] for p in parts)
    buf = torch.cat([shard.pack_shard_hull(px, py, pi, w) for px, py, pi in parts]).view(2, 3, w)
    mx = buf[:, 0, :].reshape(-1).contiguous(); my = buf[:, 1, :].reshape(-1).contiguous()
    mids = buf[:, 2, :].reshape(-1).to(torch.int64).to(torch.int32)
    m = hull.run_device(mx, my, 1, ids=mids, stats=False)
    print("width", w, "n", mx.numel(), "merged h", m.h, "whole", whole.h)

import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1501_04706_b200 import dataio, hull, shard
x, y = dataio.gen_uniform_device(40_000_000, 1)
whole = hull.run_device(x, y, 1, stats=False).h
sp = torch.cuda.current_stream().cuda_stream
parts = []
for r in range(2):
    f = r * 20_000_000
    dh = hull.run_device(x[f:f+20_000_000].contiguous(), y[f:f+20_000_000].contiguous(), 1, stats=False)
    parts.append((dh.x.clone(), dh.y.clone(), dh.indices.to(torch.int64) + f))
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 200):
    w = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    buf = torch.cat([shard.pack_shard_hull(px, py, pi, w) for px, py, pi in parts]).view(2, 3, w)
    mx = buf[:, 0, :].reshape(-1).contiguous(); my = buf[:, 1, :].reshape(-1).contiguous()
    mids = buf[:, 2, :].reshape(-1).to(torch.int64).to(torch.int32)
    m = hull.run_device(mx, my, 1, ids=mids, stream=sp, stats=False)
    if m.h != whole:
        bad += 1
print("whole", whole, "bad", bad, flush=True)

import time, numpy as np, torch, ctypes, sys
sys.path.insert(0, '/root/repo')
from paper_1501_04706_b200 import dataio, hull
x, y = dataio.gen_uniform(20_000_000, 1)
d = torch.empty(20_000_000, dtype=torch.float64, device='cuda')
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(torch.from_numpy(x)); torch.cuda.synchronize()
    print("pageable H2D 160MB: %.1f ms" % ((time.perf_counter() - t) * 1e3))
for rep in range(3):
    t = time.perf_counter(); r = hull.run_arrays(x, y, 1); print("run_arrays host pageable: %.1f ms h=%d" % ((time.perf_counter() - t) * 1e3, len(r)))

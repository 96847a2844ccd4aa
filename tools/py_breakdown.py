"""Where the Python API's per-call time goes (run_device on 20M device points)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1501_04706_b200 import _lib, dataio, hull
x, y = dataio.gen_uniform_device(20_000_000, 1)
out = tuple(torch.empty(20_000_000, dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.int64))
s = torch.cuda.current_stream().cuda_stream
for _ in range(5): hull.run_device(x, y, 1, stream=s, out=out)
K = 200
acc = {}
def t(name, f):
    t0 = time.perf_counter(); r = f(); acc[name] = acc.get(name, 0) + time.perf_counter() - t0; return r
for _ in range(K):
    xx, yy, ids, px, py, dx, n = t("prepare", lambda: hull._prepare(x, y, None))
    res = t("call(total)", lambda: hull._call(px, py, n, None, 1, _lib.SH_DEVICE_PTRS | _lib.SH_OUT_DEVICE, 0, s,
                                             out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), 20_000_000, 1 << 16))
    h = int(res[0].h)
    t("slices+DeviceHull", lambda: hull.DeviceHull(out[0][:h], out[1][:h], out[2][:h], h, res[1], res[2], res[3], 0, 0, 0))
for k, v in acc.items(): print(f"{k:20s} {v / K * 1e6:8.1f} us")

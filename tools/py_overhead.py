"""Python-side overhead of hull.run_device vs the bare C-ABI call (same inputs)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1501_04706_b200 import _lib, dataio, hull
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
x, y = dataio.gen_uniform_device(n, 1)
s = torch.cuda.current_stream().cuda_stream
out = tuple(torch.empty(n, dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.int64))
L = _lib.load()
req = _lib.sh_hull_request(); req.x = x.data_ptr(); req.y = y.data_ptr(); req.n = n; req.mode = 1
req.flags = _lib.SH_DEVICE_PTRS | _lib.SH_OUT_DEVICE; req.device = 0; req.stream = s
st = (_lib.sh_round_stat * 64)()
res = _lib.sh_hull_result(); res.x = out[0].data_ptr(); res.y = out[1].data_ptr(); res.idx = out[2].data_ptr()
res.cap = n; res.stats = ctypes.addressof(st); res.stats_cap = 64
def bare():
    assert L.sh_b200_hull_ex(ctypes.byref(req), ctypes.byref(res)) == 0
def api():
    hull.run_device(x, y, 1, stream=s, out=out)
def api_nostats():
    hull.run_device(x, y, 1, stream=s, out=out, stats=False)
for f in (bare, api, api_nostats, bare, api):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 100
    t0 = time.perf_counter(); e0.record()
    for _ in range(K): f()
    e1.record(); torch.cuda.synchronize()
    print(f"{f.__name__:12s} wall {1e3*(time.perf_counter()-t0)/K:.4f} ms  events {e0.elapsed_time(e1)/K:.4f} ms", flush=True)

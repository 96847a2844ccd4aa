"""Device hull::preprocess (sh_b200_preprocess) vs the reference's preprocess on
the host cores: 20M uniform, device-resident input.  Roofline: K1 reads 16 B/pt,
the compaction reads 16 B/pt and writes 16 B per survivor.
    python tools/bench_preprocess.py [--json-out F]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1501_04706_b200 import dataio, hull

n = 20_000_000
x, y = dataio.gen_uniform_device(n, 1)
torch.cuda.synchronize()
for _ in range(3):
    kx, ky, d = hull.preprocess_device(x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
e0.record()
for _ in range(K):
    kx, ky, d = hull.preprocess_device(x, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
kept = n - d
alg = 32 * n + 16 * kept
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
line = {"op": "hull::preprocess (device API)", "n": n, "kept": kept, "discarded": d,
        "ms": ms, "Mpoints_per_s": n / ms / 1e3, "alg_bytes": alg,
        "GB_per_s": alg / ms / 1e6, "hbm_peak_GB_per_s": peak, "frac": alg / ms / 1e6 / peak}
try:
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    import oracle
    if oracle.ref_available():
        hx, hy = x.cpu().numpy(), y.cpu().numpy()
        t = time.perf_counter(); oracle.ref_preprocess(hx, hy); t = time.perf_counter() - t
        line["cpu_reference_ms"] = t * 1e3
        line["cpu_reference"] = "hull::preprocess(Backend::Sequential) from oracle/_ref, 1 core"
except Exception as ex:  # noqa: BLE001
    line["cpu_reference_error"] = repr(ex)
print(json.dumps(line))
if len(sys.argv) > 2 and sys.argv[1] == "--json-out":
    open(sys.argv[2], "w").write(json.dumps(line) + "\n")

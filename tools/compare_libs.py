"""Time the pipeline with several library builds in ONE process per build, same box.
    [KIND=uniform|disk|circle N=2e7] python tools/compare_libs.py build_var/lib_*.so"""
import os, subprocess, sys, json
code = r'''
import os, sys, statistics, json
sys.path.insert(0, os.getcwd())
import torch
from paper_1501_04706_b200 import dataio, hull
n = int(float(os.environ.get("N", "2e7")))
kind = os.environ.get("KIND", "uniform")
if kind == "uniform":
    x, y = dataio.gen_uniform_device(n, 1)
elif kind == "disk":
    x, y = dataio.gen_disk_device(n, 1)
else:
    hx, hy = dataio.gen_circle(n, 1)
    x, y = torch.from_numpy(hx).cuda(), torch.from_numpy(hy).cuda()
torch.cuda.synchronize()
ks = []
for i in range(12):
    r = hull.run_device(x, y, 1, timings=True)
    if i >= 2: ks.append(r.kernels)
med = lambda f: statistics.median(f(k) for k in ks) * 1e3
print(json.dumps({"k1": med(lambda k: k.extremes_ms), "k2": med(lambda k: k.filter_ms),
                  "k3": med(lambda k: k.first_round_ms), "kr": med(lambda k: k.rounds_ms),
                  "tot": med(lambda k: k.extremes_ms + k.filter_ms + k.first_round_ms + k.rounds_ms)}))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SHB_LIB=lib)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
    try:
        d = json.loads(line)
        print(f"{os.path.basename(lib):12s} " + "  ".join(f"{k} {v:7.1f}" for k, v in d.items()), flush=True)
    except Exception:
        print(lib, "FAILED", line, flush=True)

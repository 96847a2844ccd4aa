"""Sweep the pageable staging ring (SHB_H2D_CHUNK_MB / SHB_H2D_NBUF / SHB_H2D_THREADS):
ms per 20M-point hull from pageable numpy input through hull.run_arrays (one process per
setting, same box).  Also reports pinned input and a bare host memcpy rate for reference."""
import itertools
import json
import os
import subprocess
import sys

CODE = r'''
import os, sys, time, statistics, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1501_04706_b200 import dataio, hull
x, y = dataio.gen_uniform(20_000_000, 1)
pin = os.environ.get("PIN") == "1"
if pin:
    x = torch.from_numpy(x).pin_memory(); y = torch.from_numpy(y).pin_memory()
for _ in range(3): hull.run_arrays(x, y, 1)
ts = []
for _ in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hull.run_arrays(x, y, 1)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
print(json.dumps({"ms": statistics.median(ts), "min": min(ts)}))
'''


def run(env):
    e = dict(os.environ, **{k: str(v) for k, v in env.items()})
    out = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=e)
    try:
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": out.stderr[-300:]}


print("pinned", run({"PIN": "1"}), flush=True)
for chunk, nbuf, th in itertools.product([4, 8, 16], [4, 8], [8, 12, 16]):
    print(f"chunk {chunk:2d} MB nbuf {nbuf} threads {th:2d}",
          run({"SHB_H2D_CHUNK_MB": chunk, "SHB_H2D_NBUF": nbuf, "SHB_H2D_THREADS": th}), flush=True)

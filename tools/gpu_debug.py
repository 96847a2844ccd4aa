"""Quick GPU shake-out: runs the sm_100a hull on growing inputs vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from paper_1501_04706_b200 import dataio, hull

def cmp(name, x, y, mode):
    try:
        ref = oracle.hull_run(x, y, mode)
    except oracle.OracleError as e:
        ref = e
    t = time.time()
    try:
        r = hull.run_arrays(x, y, mode, timings=True)
    except Exception as e:
        print(f"{name} m{mode}: GPU raised {type(e).__name__}: {e}; ref={ref if isinstance(ref, Exception) else ref.h}", flush=True)
        return isinstance(ref, Exception)
    dt = time.time() - t
    if isinstance(ref, Exception):
        print(f"{name} m{mode}: ref raised {ref}, GPU returned h={len(r)}", flush=True); return False
    ok = len(r) == ref.h and np.array_equal(r.x.view(np.uint64), ref.x.view(np.uint64)) and np.array_equal(r.y.view(np.uint64), ref.y.view(np.uint64))
    st = [(s.iteration, s.segments, s.points_remaining, s.points_removed) for s in r.stats]
    sok = st == [tuple(s) for s in ref.stats]
    if not (ok and sok):
        print(f"{name} m{mode}: MISMATCH h={len(r)} ref_h={ref.h} coords_ok={ok} stats_ok={sok} kept={r.kept}/{ref.kept}")
        print("  gpu stats", st[:12]); print("  ref stats", ref.stats[:12])
        if len(r) < 20: print("  gpu", list(zip(r.x, r.y))); print("  ref", list(zip(ref.x, ref.y)))
    else:
        print(f"{name} m{mode}: ok h={len(r)} rounds={r.rounds} wall={dt*1e3:.2f}ms ph={r.phase_timings} launches={r.kernel_launches}", flush=True)
    return ok and sok

from cases import kat_cases, random_cases
allok = True
for k, (x, y) in kat_cases().items():
    for m in (1, 2): allok &= cmp(k, x, y, m)
for name, x, y in random_cases(60, 5):
    for m in (1, 2): allok &= cmp(name, x, y, m)
for n, s in [(1000, 1), (100000, 42), (1000000, 1)]:
    x, y = dataio.gen_uniform(n, s)
    for m in (1, 2): allok &= cmp(f"uniform{n}", x, y, m)
x, y = dataio.gen_circle(200000, 3)
allok &= cmp("circle200k", x, y, 1)
allok &= cmp("circle200k", x, y, 2)
x, y = dataio.gen_circle(1_000_000, 1)
allok &= cmp("circle1M", x, y, 1)
x, y = oracle.gen_disk(2_000_000, 1)
allok &= cmp("disk2M", x, y, 1)
rng = np.random.default_rng(5)
g = rng.integers(0, 40, size=(300000, 2)).astype(np.float64)
allok &= cmp("grid40_300k", g[:, 0].copy(), g[:, 1].copy(), 1)
allok &= cmp("grid40_300k", g[:, 0].copy(), g[:, 1].copy(), 2)
x, y = dataio.gen_uniform(20_000_000, 1)
for i in range(3): allok &= cmp("uniform20M", x, y, 1)
print("ALL OK" if allok else "FAILURES")

"""Parity at extreme coordinate scales: the device hull vs the compiled reference, per factor and size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1501_04706_b200 import dataio, hull

for f in (1e-300, 1e-200, 1e-100, 1e100, 1e200, 1e300):
    for n in (10, 104, 7252, 105360):
        x, y = dataio.gen_uniform(n, 5)
        x, y = x * f, y * f
        for mode in (1, 2):
            ref = oracle.ref_hull_run(x, y, mode=mode, backend=1)
            r = hull.run_arrays(x, y, mode)
            same_h = len(r) == ref.h
            same_xy = same_h and np.array_equal(r.x.view(np.uint64), ref.x.view(np.uint64)) and \
                np.array_equal(r.y.view(np.uint64), ref.y.view(np.uint64))
            ours_st = [tuple(vars(s).values()) for s in r.stats]
            ref_st = [tuple(s) for s in ref.stats]
            same_idx = same_h and np.array_equal(r.indices, oracle.canonical_index(x, y, ref.x, ref.y))
            ok = same_xy and ours_st == ref_st and same_idx
            print(f"f={f:g} n={n} mode={mode}: h ours {len(r)} ref {ref.h} xy {same_xy} stats {ours_st == ref_st} "
                  f"idx {same_idx} kept ours {r.kept}", "ok" if ok else "DIFF", flush=True)
            if not ok:
                print("   ours", ours_st[:6], "\n   ref ", ref_st[:6])
                print("   ours xy", list(zip(r.x[:6], r.y[:6])), "\n   ref  xy", list(zip(ref.x[:6], ref.y[:6])))

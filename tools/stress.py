"""Randomised parity stress: many shapes and sizes, both modes, optional ids,
host and device inputs -- the sm_100a hull vs the compiled reference
(oracle/_ref: seghull::hull::run, Sequential) or, with --port, the C restatement.
Every 4th case also runs the multi-GPU entry point (sh_b200_hull_multi, 3 shards on
one device) against the same expected hull.
    python tools/stress.py [cases] [seed] [--port]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import oracle
from paper_1501_04706_b200 import dataio, hull

argv = [a for a in sys.argv[1:] if not a.startswith("--")]
cases = int(argv[0]) if len(argv) > 0 else 120
rng = np.random.default_rng(int(argv[1]) if len(argv) > 1 else 2024)
use_ref = "--port" not in sys.argv and oracle.ref_available()
print("expected hulls from", "the compiled reference (oracle/_ref)" if use_ref else "the C restatement",
      flush=True)


def shape(kind, n):
    if kind == "uniform":
        return dataio.gen_uniform(n, int(rng.integers(1 << 30)))
    if kind == "disk":
        return oracle.gen_disk(n, int(rng.integers(1 << 30)))
    if kind == "circle":
        return dataio.gen_circle(n, int(rng.integers(1 << 30)))
    if kind == "gauss":
        return rng.normal(size=n), rng.normal(size=n) * rng.uniform(0.01, 10)
    if kind == "clusters":
        c = rng.normal(size=(8, 2)) * 10
        k = rng.integers(0, 8, n)
        return c[k, 0] + rng.normal(size=n) * 0.1, c[k, 1] + rng.normal(size=n) * 0.1
    if kind == "lattice":
        m = int(rng.integers(2, 200))
        return rng.integers(0, m, n).astype(np.float64), rng.integers(0, m, n).astype(np.float64)
    if kind == "line":
        t = rng.uniform(-1, 1, n)
        return t, 3 * t - 1 + (rng.random(n) < 0.001) * 1e-9
    if kind == "annulus":
        th = rng.uniform(0, 2 * np.pi, n)
        r = 1 - rng.uniform(0, 1e-6, n)
        return r * np.cos(th), r * np.sin(th)
    if kind == "dups":
        bx, by = dataio.gen_uniform(max(1, n // 50), int(rng.integers(1 << 30)))
        k = rng.integers(0, bx.size, n)
        return bx[k].copy(), by[k].copy()
    if kind == "offset":  # large coordinates, small extent (cancellation in every difference)
        x, y = dataio.gen_uniform(n, int(rng.integers(1 << 30)))
        return x + 1e8, y * 1e-3 - 3e7
    if kind == "scaled":  # extreme magnitudes (the screen's range guards)
        x, y = dataio.gen_uniform(n, int(rng.integers(1 << 30)))
        f = [1e-300, 1e-100, 1e100, 1e300][int(rng.integers(4))]
        return x * f, y * f
    raise ValueError(kind)


kinds = ["uniform", "disk", "circle", "gauss", "clusters", "lattice", "line", "annulus", "dups",
         "offset", "scaled"]
bad = 0
multi = 0
multi_nonexact = 0
t0 = time.time()
for i in range(cases):
    kind = kinds[i % len(kinds)]
    n = int(np.exp(rng.uniform(np.log(3), np.log(3_000_000))))
    x, y = shape(kind, n)
    x, y = np.ascontiguousarray(x, np.float64), np.ascontiguousarray(y, np.float64)
    use_ids = rng.random() < 0.3
    dev = rng.random() < 0.5
    for mode in (1, 2):
        try:
            ref = oracle.ref_hull_run(x, y, mode=mode, backend=1) if use_ref else oracle.hull_run(x, y, mode)
        except oracle.OracleError as e:
            ref = e
        ids = None
        xx, yy = x, y
        if use_ids:
            perm = rng.permutation(n)
            xx, yy, ids = x[perm].copy(), y[perm].copy(), perm.astype(np.uint32)
        try:
            if dev:
                r = hull.run_arrays(torch.from_numpy(xx).cuda(), torch.from_numpy(yy).cuda(), mode,
                                    ids=None if ids is None else torch.from_numpy(ids.view(np.int32)).cuda())
            else:
                r = hull.run_arrays(xx, yy, mode, ids=ids)
        except hull.Error as e:
            ok = isinstance(ref, oracle.OracleError)
            if not ok:
                bad += 1
                print(f"FAIL {kind} n={n} m{mode}: GPU raised {e}", flush=True)
            continue
        if isinstance(ref, Exception):
            bad += 1
            print(f"FAIL {kind} n={n} m{mode}: oracle raised {ref}, GPU h={len(r)}", flush=True)
            continue
        ok = (len(r) == ref.h and np.array_equal(r.x.view(np.uint64), ref.x.view(np.uint64))
              and np.array_equal(r.y.view(np.uint64), ref.y.view(np.uint64))
              and [tuple(vars(s).values()) for s in r.stats] == [tuple(s) for s in ref.stats]
              and np.array_equal(r.indices, oracle.canonical_index(x, y, ref.x, ref.y)))
        if not ok:
            bad += 1
            print(f"FAIL {kind} n={n} m{mode} ids={use_ids} dev={dev}: h {len(r)} vs {ref.h}", flush=True)
        if i % 4 == 0 and mode == 1 and not use_ids and n >= 3:
            # the multi-GPU entry (3 contiguous shards on this device) against the
            # reference's own sharded route: hull::run of the union of the 3 shard
            # hulls.  In general position that IS the whole-input hull;
            # for near-collinear inputs the reference's sharded route itself differs
            # from its whole-input hull (FP predicates), and the device must match
            # the sharded route
            m = hull.run_multi(x, y, [0, 0, 0], mode)
            if use_ref:
                parts = []
                for g in range(3):
                    a, b = n * g // 3, n * (g + 1) // 3
                    if b > a:
                        try:
                            rr = oracle.ref_hull_run(x[a:b], y[a:b], mode=1, backend=0)
                            parts.append((rr.x, rr.y))
                        except oracle.OracleError:
                            pass
                sh = oracle.ref_hull_run(np.concatenate([p[0] for p in parts]),
                                         np.concatenate([p[1] for p in parts]), mode=1, backend=0)
            else:
                sh = ref
            okm = (len(m) == sh.h and np.array_equal(m.x.view(np.uint64), sh.x.view(np.uint64))
                   and np.array_equal(m.y.view(np.uint64), sh.y.view(np.uint64))
                   and np.array_equal(m.indices, oracle.canonical_index(x, y, sh.x, sh.y)))
            multi += 1
            if not (sh.h == ref.h and np.array_equal(sh.x.view(np.uint64), ref.x.view(np.uint64))):
                multi_nonexact += 1
            if not okm:
                bad += 1
                print(f"FAIL multi {kind} n={n}: h {len(m)} vs sharded reference {sh.h}", flush=True)
print(f"{cases} cases x 2 modes (+{multi} multi-GPU-entry checks vs the reference's sharded route, "
      f"{multi_nonexact} of them near-collinear inputs where that route differs from the whole-input "
      f"hull): {bad} failures ({time.time() - t0:.0f} s)", flush=True)

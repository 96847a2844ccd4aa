"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run here (where /root/reference exists) after `make -C oracle`:

    PYTHONPATH=. python tests/golden/make_golden.py

Every expected output is produced by the unmodified reference core compiled
from /root/reference sources (oracle/_ref/libseghull_ref.so, built by
oracle/Makefile) -- never by our own restatement and never by the CUDA path.
The fixtures then travel to the GPU box, where /root/reference does not.

Outputs
  small.npz      inputs + reference hulls (both modes, Sequential backend) +
                 per-round SegmentStats for the KAT and random corpora.
  configs.json   the BASELINE.json configs at full size: h, k (Mode-1 filter
                 survivors), per-round stats, FNV-1a of the vertex bits, and the
                 vertices themselves (hex floats) with canonical input indices
                 when the hull is small.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from cases import kat_cases, random_cases  # noqa: E402


def ref_or_error(x, y, mode):
    try:
        r = oracle.ref_hull_run(x, y, mode=mode, backend=0)
        return 0, r.x, r.y, r.stats
    except oracle.OracleError as e:
        return e.code, np.zeros(0), np.zeros(0), []


def small():
    names, xs, ys = [], [], []
    for k, (x, y) in kat_cases().items():
        names.append(k)
        xs.append(x)
        ys.append(y)
    for name, x, y in random_cases():
        names.append(name)
        xs.append(x)
        ys.append(y)
    # plus a few inputs with the error paths of hull.cpp:221-227
    names += ["empty", "nan_at_1", "inf_at_2"]
    xs += [np.zeros(0), np.array([0.0, 1.0, 2.0]), np.array([0.0, 1.0, np.inf])]
    ys += [np.zeros(0), np.array([0.0, np.nan, 1.0]), np.array([0.0, 1.0, 2.0])]

    rec = {"names": np.array(names)}
    in_off = np.cumsum([0] + [len(v) for v in xs])
    rec["in_off"] = in_off
    rec["in_x"] = np.concatenate(xs)
    rec["in_y"] = np.concatenate(ys)
    for mode in (1, 2):
        hx, hy, hidx, codes, st, st_off = [], [], [], [], [], [0]
        for x, y in zip(xs, ys):
            code, vx, vy, stats = ref_or_error(x, y, mode)
            codes.append(code)
            hx.append(vx)
            hy.append(vy)
            hidx.append(oracle.canonical_index(x, y, vx, vy) if vx.size else np.zeros(0, np.int64))
            st.extend(stats)
            st_off.append(len(st))
        rec[f"m{mode}_code"] = np.array(codes, np.int32)
        rec[f"m{mode}_off"] = np.cumsum([0] + [len(v) for v in hx])
        rec[f"m{mode}_x"] = np.concatenate(hx)
        rec[f"m{mode}_y"] = np.concatenate(hy)
        rec[f"m{mode}_idx"] = np.concatenate(hidx)
        rec[f"m{mode}_stats"] = np.array(st, np.uint64).reshape(-1, 4)
        rec[f"m{mode}_stats_off"] = np.array(st_off, np.int64)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **rec)
    print("small.npz:", len(names), "cases")


CONFIGS = [
    # name, generator, n, seed
    ("uniform_100k_s42", "uniform", 100_000, 42),
    ("uniform_1m_s1", "uniform", 1_000_000, 1),
    ("uniform_1m_s2", "uniform", 1_000_000, 2),
    ("circle_200k_s3", "circle", 200_000, 3),
    ("uniform_20m_s1", "uniform", 20_000_000, 1),
    ("disk_20m_s1", "disk", 20_000_000, 1),
    ("circle_4m_s1", "circle", 4_000_000, 1),
]


def gen(kind, n, seed):
    if kind == "uniform":
        return oracle.ref_gen_uniform(n, seed)
    if kind == "circle":
        return oracle.ref_gen_circle(n, seed)
    return oracle.gen_disk(n, seed)  # not in the reference: SURVEY.md section 8d


def configs():
    out = {"discards_uniform_100000_42": oracle.ref_preprocess_discards(
        *oracle.ref_gen_uniform(100_000, 42))}
    for name, kind, n, seed in CONFIGS:
        x, y = gen(kind, n, seed)
        ent = {"generator": kind, "n": n, "seed": seed}
        for mode in (1, 2):
            r = oracle.ref_hull_run(x, y, mode=mode, backend=1)
            e = {"h": r.h, "rounds": len(r.stats), "stats": [list(s) for s in r.stats],
                 "fnv1a": oracle.fnv1a(r.x, r.y),
                 "first": [float(r.x[0]).hex(), float(r.y[0]).hex()]}
            if r.h <= 5000:
                e["vx"] = [float(v).hex() for v in r.x]
                e["vy"] = [float(v).hex() for v in r.y]
                e["idx"] = [int(i) for i in oracle.canonical_index(x, y, r.x, r.y)]
            ent[f"mode{mode}"] = e
            print(name, mode, r.h, len(r.stats), flush=True)
        ent["kept"] = n - oracle.ref_preprocess_discards(x, y)
        out[name] = ent
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    small()
    configs()

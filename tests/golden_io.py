"""Helpers to walk tests/golden/small.npz (written by tests/golden/make_golden.py)."""
import numpy as np


def iter_small(g, mode):
    names = g["names"]
    io = g["in_off"]
    ho = g[f"m{mode}_off"]
    so = g[f"m{mode}_stats_off"]
    for k, name in enumerate(names):
        yield dict(
            name=str(name),
            x=g["in_x"][io[k]:io[k + 1]].copy(),
            y=g["in_y"][io[k]:io[k + 1]].copy(),
            code=int(g[f"m{mode}_code"][k]),
            hx=g[f"m{mode}_x"][ho[k]:ho[k + 1]],
            hy=g[f"m{mode}_y"][ho[k]:ho[k + 1]],
            idx=g[f"m{mode}_idx"][ho[k]:ho[k + 1]],
            stats=[tuple(int(v) for v in row) for row in g[f"m{mode}_stats"][so[k]:so[k + 1]]],
        )


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def fromhex(lst):
    return np.array([float.fromhex(v) for v in lst], dtype=np.float64)

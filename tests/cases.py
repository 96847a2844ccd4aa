"""Deterministic small-input corpus shared by the golden generator and tests.

The shapes mirror the reference's own randomized suites:
tests/test_hull.cpp:376-403 (uniform / circle, n <= 400),
tests/acceptance.cpp:140-167 (12x12 integer grid with duplicates) and the
degenerate suite at acceptance.cpp:271-323 (collinear, identical, duplicated
corners).  Inputs are generated with our own SplitMix64 so they do not depend
on numpy's RNG stream, and the golden file stores them anyway.
"""
from __future__ import annotations

import numpy as np

MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


class SM64:
    def __init__(self, seed: int):
        self.s = seed & MASK

    def next(self) -> int:
        self.s = (self.s + GAMMA) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def below(self, k: int) -> int:
        return self.next() % k

    def unit(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53


def kat_cases():
    """Hand-written inputs from the reference's unit/acceptance tests."""
    P = lambda pts: (np.array([p[0] for p in pts], float), np.array([p[1] for p in pts], float))
    cases = {
        "square_center": P([(0, 0), (1, 0), (1, 1), (0, 1), (0.5, 0.5)]),       # test_hull.cpp:316
        "three_points": P([(3, 1), (0, 2), (1, 0)]),                           # test_hull.cpp:325
        "first_split_4": P([(0, 0), (2, 0), (1, 1), (1, -1)]),                 # test_hull.cpp:88
        "collinear_upper": P([(0, 0), (1, 0), (2, 0), (1, 2)]),                # test_hull.cpp:103
        "one": P([(2, 3)]),                                                    # test_hull.cpp:345
        "two": P([(5, 5), (2, 3)]),                                            # test_hull.cpp:348
        "same3": P([(1, 1), (1, 1), (1, 1)]),                                  # test_hull.cpp:352
        "collinear4": P([(0, 0), (2, 2), (1, 1), (3, 3)]),                     # test_hull.cpp:356
        "dup_corners": P([(0, 0), (1, 0), (1, 1), (0, 1), (0, 0), (1, 1), (1, 0),
                          (0.25, 0.5), (1, 1)]),                               # test_hull.cpp:367
        "acc_one": P([(3.5, -1.25)]),                                          # acceptance.cpp:283
        "acc_two": P([(4, 4), (-1, 2)]),                                       # acceptance.cpp:290
        "acc_identical": P([(2, 2)] * 9),                                      # acceptance.cpp:298
        "acc_collinear": P([(i % 7, 2 * (i % 7)) for i in range(11)]),         # acceptance.cpp:305
        "acc_dup_corners": P([(0, 0), (2, 0), (2, 2), (0, 2)] * 3 + [(1, 1)]),  # acceptance.cpp:313
        "vertical_line": P([(1, 0), (1, 3), (1, 1), (1, 2)]),
        "horizontal_line": P([(0, 5), (3, 5), (1, 5)]),
        "neg_slope": P([(0, 2), (1, 1), (2, 0), (0.5, 1.5)]),
    }
    return cases


def random_cases(count: int = 400, seed: int = 2024):
    """(name, x, y) tuples: uniform, circle-like, integer grids, folded lines."""
    import oracle  # test infrastructure only

    rng = SM64(seed)
    out = []
    for t in range(count):
        kind = t % 5
        n = 1 + rng.below(300)
        s = rng.next()
        if kind == 0:
            x, y = oracle.gen_uniform(n, s)
        elif kind == 1:
            x, y = oracle.gen_circle(n, s)
        elif kind == 2:   # 12x12 grid with duplicates, acceptance.cpp:150-156
            x = np.array([float(rng.below(12)) for _ in range(n)])
            y = np.array([float(rng.below(12)) for _ in range(n)])
        elif kind == 3:   # 4x50 grid: many exact ties in distance and lex order
            x = np.array([float(rng.below(4)) for _ in range(n)])
            y = np.array([float(rng.below(50)) for _ in range(n)])
        else:             # folded collinear line plus a few off-line points
            k = np.array([float(rng.below(40)) for _ in range(n)])
            x = k.copy()
            y = 3.0 * k - 7.0
            for _ in range(rng.below(3)):
                j = rng.below(n)
                y[j] += rng.unit() * 4 - 2
        out.append((f"rand{t}_k{kind}_n{n}", np.ascontiguousarray(x), np.ascontiguousarray(y)))
    return out

"""GPU: the per-phase device API (hull.hpp:61-91).

The reference's per-stage tests (tests/test_hull.cpp:88-314) restated against
the device HullState, plus a step-by-step comparison with the reference's own
HullState (oracle/_ref, RefHullState): after EVERY phase of every round, every
column of the device state must equal the reference's, bit for bit.
"""
import numpy as np
import pytest

import oracle
from golden_io import bits
from paper_1501_04706_b200 import dataio, hull
from paper_1501_04706_b200.hull import SegmentMax

pytestmark = pytest.mark.gpu


def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def pts(*p):
    a = np.array(p, np.float64)
    return a[:, 0].copy(), a[:, 1].copy()


def col(st, k):
    return list(st.columns()[k])


def advance_one_round(s):  # tests/test_hull.cpp:21-33
    hull.compute_distances(s)
    far = hull.find_farthest(s)
    splittable = any(f.value > 0.0 for f in far)
    if not splittable and s.size() == len(far):
        return False
    hull.split_segments(s, far)
    hull.mark_interior(s)
    hull.compact(s)
    return True


def valid_hull_state(s):  # tests/helpers.hpp valid_hull_state
    c = s.columns()
    n = s.size()
    if n == 0:
        return True
    head, keys = c["head"], c["keys"]
    if head[0] != 1 or not np.isin(head, [0, 1]).all():
        return False
    if keys[0] != 0 or not np.isin(np.diff(keys), [0, 1]).all():
        return False
    if not np.array_equal(keys, np.cumsum(head) - 1):
        return False
    first = np.maximum.accumulate(np.where(head != 0, np.arange(n), 0))
    if not np.array_equal(c["first_pts"], first):
        return False
    x, y = c["x"], c["y"]
    starts = list(np.flatnonzero(head)) + [n]
    for a, b in zip(starts[:-1], starts[1:]):
        asc = desc = True
        for j in range(a + 1, b):
            less = x[j - 1] < x[j] if x[j - 1] != x[j] else y[j - 1] < y[j]
            greater = x[j - 1] > x[j] if x[j - 1] != x[j] else y[j - 1] > y[j]
            desc &= not less
            asc &= not greater
        if not asc and not desc:
            return False
    return True


def test_first_split_ccw_layout():  # test_hull.cpp:88-101
    torch_cuda()
    s = hull.first_split(*pts((0, 0), (2, 0), (1, 1), (1, -1)))
    assert s.size() == 4
    assert [s.point(i) for i in range(4)] == [hull.Point(0, 0), hull.Point(1, -1),
                                              hull.Point(2, 0), hull.Point(1, 1)]
    assert col(s, "head") == [1, 0, 1, 0]
    assert col(s, "keys") == [0, 0, 1, 1]
    assert col(s, "first_pts") == [0, 0, 2, 2]
    assert col(s, "flag") == [1, 1, 1, 1]
    assert valid_hull_state(s)


def test_first_split_collinear_goes_upper():  # test_hull.cpp:103-121
    torch_cuda()
    x, y = pts((0, 0), (1, 0), (2, 0), (1, 2))
    s = hull.first_split(x, y)
    assert [s.point(i) for i in range(4)] == [hull.Point(0, 0), hull.Point(2, 0),
                                              hull.Point(1, 2), hull.Point(1, 0)]
    assert col(s, "head") == [1, 1, 0, 0]
    ex, ey = oracle.monotone_chain(x, y)
    for mode in (1, 2):
        r = hull.run_arrays(x, y, mode)
        assert np.array_equal(bits(r.x), bits(ex)) and np.array_equal(bits(r.y), bits(ey))


def test_first_split_random_valid():  # test_hull.cpp:123-130
    torch_cuda()
    s = hull.first_split(*dataio.gen_uniform(100, 7))
    assert valid_hull_state(s)


def test_first_split_errors():  # test_hull.cpp:132-138
    torch_cuda()
    with pytest.raises(hull.Error) as ei:
        hull.first_split(*pts((1, 1), (1, 1), (1, 1)))
    assert ei.value.code() == hull.Errc.DegenerateInput
    with pytest.raises(hull.Error) as ei:
        hull.first_split(np.zeros(0), np.zeros(0))
    assert ei.value.code() == hull.Errc.EmptyInput


def test_distances_against_base_line():  # test_hull.cpp:140-148
    torch_cuda()
    s = hull.first_split(*pts((0, 0), (2, 0), (1, 1), (1, -1)))
    hull.compute_distances(s)
    d = col(s, "dist")
    assert d[1] == 2.0 and d[0] == 0.0 and d[2] == 0.0 and d[3] == 2.0


def test_distances_scalar_recomputation():  # test_hull.cpp:150-169
    torch_cuda()
    s = hull.first_split(*dataio.gen_uniform(50, 12))
    advance_one_round(s)
    hull.compute_distances(s)
    c = s.columns()
    heads = list(np.flatnonzero(c["head"]))
    n = s.size()
    for i in range(n):
        seg = 0
        while seg + 1 < len(heads) and heads[seg + 1] <= i:
            seg += 1
        f = heads[seg]
        l = heads[seg + 1] if seg + 1 < len(heads) else 0
        cr = (c["x"][l] - c["x"][f]) * (c["y"][i] - c["y"][f]) - \
             (c["y"][l] - c["y"][f]) * (c["x"][i] - c["x"][f])
        assert c["dist"][i] == -cr


def test_find_farthest_maxima():  # test_hull.cpp:171-210
    torch_cuda()
    s = hull.HullState.from_columns(x=[0, 1, 2], y=[0, 0, 0], dist=[0, 3, 1], head=[1, 0, 0],
                                    keys=[0, 0, 0], first_pts=[0, 0, 0], flag=[1, 1, 1])
    far = hull.find_farthest(s)
    assert list(far) == [SegmentMax(0, 3.0, 1)]
    s2 = hull.HullState.from_columns(x=[0, 1, 2], y=[0, 0, 0], dist=[0, 0, 0], head=[1, 0, 0],
                                     keys=[0, 0, 0], first_pts=[0, 0, 0], flag=[1, 1, 1])
    far = hull.find_farthest(s2)
    assert len(far) == 1 and far[0].value == 0.0
    t = hull.first_split(*pts((0, 0), (1, -2), (2, -1), (4, 0), (3, 2), (1, 1)))
    hull.compute_distances(t)
    res = hull.find_farthest(t)
    assert len(res) == 2
    c = t.columns()
    for e in res:
        best, arg = -1.0, 0
        for i in range(t.size()):
            if c["keys"][i] == e.key and c["dist"][i] > best:
                best, arg = c["dist"][i], i
        assert e.value == best and e.index == arg


def test_split_segments_promotes():  # test_hull.cpp:212-236
    torch_cuda()
    s = hull.HullState.from_columns(x=[0, 1, 2, 3, 4], y=[0] * 5, dist=[0, 3, 1, 0, 0],
                                    head=[1, 0, 0, 1, 0], keys=[0, 0, 0, 1, 1],
                                    first_pts=[0, 0, 0, 3, 3], flag=[1] * 5)
    hull.split_segments(s, [SegmentMax(0, 3.0, 1), SegmentMax(1, 0.0, 3)])
    assert col(s, "head") == [1, 1, 0, 1, 0]
    assert col(s, "keys") == [0, 1, 1, 2, 2]
    assert col(s, "first_pts") == [0, 1, 1, 3, 3]
    before = s.columns()
    hull.split_segments(s, [SegmentMax(0, 0.0, 0), SegmentMax(1, 0.0, 1), SegmentMax(2, 0.0, 3)])
    after = s.columns()
    for k in ("head", "keys", "first_pts"):
        assert np.array_equal(after[k], before[k])


def test_split_keeps_keys_valid():  # test_hull.cpp:238-250
    torch_cuda()
    for trial in range(20):
        s = hull.first_split(*dataio.gen_uniform(20, 100 + trial))
        hull.compute_distances(s)
        hull.split_segments(s, hull.find_farthest(s))
        c = s.columns()
        assert np.array_equal(c["keys"], np.cumsum(c["head"]) - 1)


def test_mark_interior_triangle():  # test_hull.cpp:252-282
    torch_cuda()

    def build(px, py):
        return hull.HullState.from_columns(x=[0, px, 2, 4], y=[0, py, -2, 0], dist=[0] * 4,
                                           head=[1, 0, 1, 1], keys=[0, 0, 1, 2],
                                           first_pts=[0, 0, 2, 3], flag=[1] * 4)
    inside = build(1, -0.5)
    hull.mark_interior(inside)
    assert col(inside, "flag")[1] == 0
    outside = build(1, -1.5)
    hull.mark_interior(outside)
    assert col(outside, "flag")[1] == 1
    on_line = build(1, -1)
    hull.mark_interior(on_line)
    assert col(on_line, "flag")[1] == 0
    f = col(inside, "flag")
    assert f[0] == 1 and f[2] == 1 and f[3] == 1


def test_compact_rows_and_first_pts():  # test_hull.cpp:284-301
    torch_cuda()
    x, y = dataio.gen_uniform(60, 19)
    s = hull.first_split(x, y)
    c0 = s.columns()
    copy = hull.first_split(x, y)
    assert hull.compact(copy) == 0
    c1 = copy.columns()
    assert np.array_equal(bits(c1["x"]), bits(c0["x"])) and np.array_equal(c1["head"], c0["head"])
    hull.compute_distances(s)
    hull.split_segments(s, hull.find_farthest(s))
    segments = s.segments()
    s.flag[:s.size()].copy_(s.head[:s.size()])
    hull.compact(s)
    assert s.size() == segments
    assert valid_hull_state(s)


def test_compact_invariants_random_pipelines():  # test_hull.cpp:303-314
    torch_cuda()
    for trial in range(0, 100, 7):
        n = 3 + trial * 3
        x, y = dataio.gen_circle(n, trial) if trial % 3 == 2 else dataio.gen_uniform(n, trial)
        s = hull.first_split(x, y)
        for _ in range(4):
            if not advance_one_round(s):
                break
            assert valid_hull_state(s), (trial, n)


def _same_state(dev, ref, where):
    a, b = dev.columns(), ref.columns()
    for k in oracle.STATE_COLUMNS:
        if k in ("x", "y", "dist"):
            assert np.array_equal(bits(a[k]), bits(b[k])), (where, k)
        else:
            assert np.array_equal(a[k], b[k]), (where, k)


def _inputs():
    yield "uniform_5k", dataio.gen_uniform(5_000, 3)
    yield "circle_3k", dataio.gen_circle(3_000, 4)
    rng = np.random.default_rng(5)
    g = rng.integers(0, 12, size=(4_000, 2)).astype(np.float64)  # duplicates and collinear runs
    yield "grid_12", (g[:, 0].copy(), g[:, 1].copy())
    yield "uniform_300k", dataio.gen_uniform(300_000, 8)
    z = rng.integers(-2, 3, size=(2_000, 2)).astype(np.float64)
    z[z == 0] = -0.0  # signed zeros: equal under the reference's comparisons
    yield "signed_zero_grid", (z[:, 0].copy(), z[:, 1].copy())


@pytest.mark.parametrize("name,xy", list(_inputs()), ids=lambda v: v if isinstance(v, str) else "")
def test_every_phase_equals_reference_state(name, xy):
    """Drive the device state and the reference's HullState through the same
    rounds; compare all seven columns after every phase."""
    torch_cuda()
    x, y = xy
    dev = hull.first_split(x, y)
    ref = oracle.RefHullState.first_split(x, y)
    if name != "signed_zero_grid":  # std::sort may order +0/-0 duplicates either way
        _same_state(dev, ref, "first_split")
    else:  # re-seed the device from the reference's layout
        dev = hull.HullState.from_columns(**ref.columns())
    for rnd in range(1, 200):
        hull.compute_distances(dev)
        ref.compute_distances()
        _same_state(dev, ref, (rnd, "compute_distances"))
        far = hull.find_farthest(dev)
        rk, rv, ri = ref.find_farthest()
        assert [e.key for e in far] == list(rk) and [e.index for e in far] == list(ri), rnd
        assert np.array_equal(bits(np.array([e.value for e in far])), bits(rv)), rnd
        if not any(e.value > 0.0 for e in far) and dev.size() == len(far):
            break
        hull.split_segments(dev, far)
        ref.split_segments(rk, rv, ri)
        _same_state(dev, ref, (rnd, "split_segments"))
        hull.mark_interior(dev)
        ref.mark_interior()
        _same_state(dev, ref, (rnd, "mark_interior"))
        assert hull.compact(dev) == ref.compact(), rnd
        _same_state(dev, ref, (rnd, "compact"))
    # the stages drove to the hull: the state's rows are the reference hull
    r = oracle.ref_hull_run(x, y, mode=2, backend=0)
    c = dev.columns()
    assert np.array_equal(bits(c["x"]), bits(r.x)) and np.array_equal(bits(c["y"]), bits(r.y))

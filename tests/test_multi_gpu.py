"""GPU: the multi-GPU entry points of the C-ABI, the 1B config, the segment-table
regrow path and concurrent callers.

* sh_b200_hull_multi / sh_b200_hull_shards with several shards on ONE device
  (devices = {0,0,0,0}: one host thread, workspace, stream and pinned ring per
  shard, the payload blocks written into the root's gather buffer) must give
  the same vertices and canonical GLOBAL indices as the single-device hull
  (SURVEY.md section 8e parity: coordinates bit-exact, indices canonical).
* pack_device + hull_gathered (the one-process-per-GPU path of bench.py) with
  a block smaller than the shard hull: the overflow marker and the retry.
* BASELINE.json configs[4] (1B uniform points): on one GPU whole, and as 8
  device-generated shards merged by sh_b200_hull_shards, against the reference
  golden of tests/golden/make_golden_1b.py.
* SHB_SEG_CAP forces ST_OVERFLOW: the regrow-and-rerun path (with the pool
  stream, the default for host inputs).
* two host threads with pageable inputs at once (per-workspace pinned rings).
"""
import ctypes
import os
import threading

import numpy as np
import pytest

import oracle
from golden_io import bits, fromhex
from paper_1501_04706_b200 import _lib, dataio, hull, shard

pytestmark = pytest.mark.gpu


def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def inputs(kind):
    if kind == "uniform":
        return dataio.gen_uniform(2_000_000, 9)
    if kind == "circle":
        return dataio.gen_circle(300_000, 2)
    rng = np.random.default_rng(3)  # duplicates within and across shards
    g = rng.integers(0, 25, size=(90_000, 2)).astype(np.float64)
    return g[:, 0].copy(), g[:, 1].copy()


def same_hull(r, ref_x, ref_y, ref_idx, name=""):
    rx = r.x.cpu().numpy() if hasattr(r.x, "cpu") else np.asarray(r.x)
    ry = r.y.cpu().numpy() if hasattr(r.y, "cpu") else np.asarray(r.y)
    ri = r.indices.cpu().numpy() if hasattr(r.indices, "cpu") else np.asarray(r.indices)
    assert rx.size == ref_x.size, (name, rx.size, ref_x.size)
    assert np.array_equal(bits(rx), bits(ref_x)), name
    assert np.array_equal(bits(ry), bits(ref_y)), name
    assert np.array_equal(ri, np.asarray(ref_idx, np.int64)), name


@pytest.mark.parametrize("kind", ["uniform", "circle", "grid"])
@pytest.mark.parametrize("ndev", [4, 3])
def test_hull_multi_same_device_bit_exact(kind, ndev):
    torch_cuda()
    x, y = inputs(kind)
    whole = hull.run_arrays(x, y, 1)
    ref = oracle.hull_run(x, y, 1)
    assert np.array_equal(bits(whole.x), bits(ref.x))
    idx = oracle.canonical_index(x, y, ref.x, ref.y)
    m = hull.run_multi(x, y, [0] * ndev, 1)
    same_hull(m, ref.x, ref.y, idx, f"{kind} x{ndev}")
    assert m.kernels.shards == ndev
    md = hull.run_multi(x, y, [0] * ndev, 2, out_device=True)  # Mode 2, device outputs
    same_hull(md, ref.x, ref.y, idx, f"{kind} x{ndev} mode 2")


def test_hull_multi_circle_overflows_first_block_and_repacks():
    """Shard hulls of ~100K vertices exceed the 2048-vertex first-pass block:
    the library re-packs them from the retained head tables."""
    torch_cuda()
    x, y = dataio.gen_circle(400_000, 4)
    ref = oracle.hull_run(x, y, 1)
    m = hull.run_multi(x, y, [0, 0, 0, 0], 1)
    same_hull(m, ref.x, ref.y, oracle.canonical_index(x, y, ref.x, ref.y), "circle repack")
    assert m.kernels.block_cap > 2048


def test_hull_shards_device_resident_and_errors():
    torch = torch_cuda()
    x, y = inputs("uniform")
    ref = oracle.hull_run(x, y, 1)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    parts = []
    for r in range(5):
        f, c = shard.shard_range(x.size, 5, r)
        parts.append((dx[f:f + c], dy[f:f + c], f))
    m = hull.run_shards(parts, 1)
    same_hull(m, ref.x, ref.y, oracle.canonical_index(x, y, ref.x, ref.y), "shards")
    # non-finite input: the GLOBAL first bad index (hull.cpp:222-227)
    x2 = x.copy()
    x2[1_234_567] = np.nan
    x2[1_900_000] = np.inf
    with pytest.raises(hull.Error) as ei:
        hull.run_multi(x2, y, [0, 0, 0], 1)
    assert ei.value.code() == hull.Errc.NonFiniteInput
    assert "index 1234567" in str(ei.value)
    with pytest.raises(hull.Error) as ei:
        hull.run_multi(np.zeros(0), np.zeros(0), [0, 0], 1)
    assert ei.value.code() == hull.Errc.EmptyInput


def test_pack_and_gathered_merge_with_overflow_retry():
    """bench.py's N-rank step on one device: each 'rank' packs its shard hull
    into a block, the blocks are concatenated as an all-gather would, the
    library merges.  A 64-vertex block overflows on a circle: the merge
    reports the capacity needed and the retry is exact."""
    torch = torch_cuda()
    for kind, cap in [("uniform", shard.HMAX), ("circle", 64), ("grid", 8)]:
        x, y = inputs(kind)
        ref = oracle.hull_run(x, y, 1)
        idx = oracle.canonical_index(x, y, ref.x, ref.y)
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        world = 4

        def gather(out, inp, _w=world, _x=dx, _y=dy):
            blocks = []
            cap_ = inp.numel() // 3
            for r in range(_w):
                f, c = shard.shard_range(_x.shape[0], _w, r)
                b = torch.empty(3 * cap_, dtype=torch.float64, device="cuda")
                hull.pack_device(_x[f:f + c], _y[f:f + c], b, first=f)
                blocks.append(b)
            out.copy_(torch.cat(blocks))

        f0, c0 = shard.shard_range(x.size, world, 0)
        (mx, my, mi), h = shard.merged_hull(dx[f0:f0 + c0], dy[f0:f0 + c0], f0, x.size, world,
                                            gather, block_cap=cap)
        assert h == ref.h, kind
        assert np.array_equal(bits(mx.cpu().numpy()), bits(ref.x)), kind
        assert np.array_equal(bits(my.cpu().numpy()), bits(ref.y)), kind
        assert np.array_equal(mi.cpu().numpy(), idx), kind


def test_pack_degenerate_shards():
    """Shards whose hull is one point or two points (hull.cpp:234-248) pack
    their extremes; the merge of such blocks equals the whole hull."""
    torch = torch_cuda()
    x = np.array([2.0, 2.0, 2.0, 0.0, 1.0, 3.0, 5.0, 5.0, 5.0])
    y = np.array([2.0, 2.0, 2.0, 0.0, 1.0, 3.0, 1.0, 1.0, 1.0])
    ref = oracle.hull_run(x, y, 1)
    m = hull.run_multi(x, y, [0, 0, 0], 1)
    same_hull(m, ref.x, ref.y, oracle.canonical_index(x, y, ref.x, ref.y), "degenerate")


@pytest.mark.slow
def test_uniform_1b_one_gpu_matches_reference(golden_configs):
    """BASELINE.json configs[4] on one B200: gen_uniform(1e9, 1) generated on
    the device, hulled whole; vertices, canonical indices and per-round
    SegmentStats equal the reference's whole-input run."""
    torch = torch_cuda()
    g = golden_configs["uniform_1b_s1"]
    e = g["mode1"]
    _lib.load().sh_b200_release_pool()
    x, y = dataio.gen_uniform_device(g["n"], g["seed"])
    r = hull.run_arrays(x, y, 1)
    same_hull(r, fromhex(e["vx"]), fromhex(e["vy"]), e["idx"], "1B")
    assert [(s.iteration, s.segments, s.points_remaining, s.points_removed) for s in r.stats] == \
        [tuple(s) for s in e["stats"]]
    assert oracle.fnv1a(r.x, r.y) == e["fnv1a"]
    del x, y
    torch.cuda.empty_cache()
    _lib.load().sh_b200_release_pool()


@pytest.mark.slow
def test_uniform_1b_eight_shards_matches_reference(golden_configs):
    """The 8-GPU decomposition of configs[4] on one GPU: 8 device-generated
    shards of 125M points hulled by 8 host threads, merged by the library."""
    torch = torch_cuda()
    g = golden_configs["uniform_1b_s1"]
    e = g["mode1"]
    _lib.load().sh_b200_release_pool()
    n, w = g["n"], 8
    parts = []
    for r in range(w):
        f, c = shard.shard_range(n, w, r)
        sx, sy = dataio.gen_uniform_device(c, g["seed"], first=f)
        parts.append((sx, sy, f))
    m = hull.run_shards(parts, 1)
    same_hull(m, fromhex(e["vx"]), fromhex(e["vy"]), e["idx"], "1B x8")
    del parts
    torch.cuda.empty_cache()
    _lib.load().sh_b200_release_pool()


def test_segment_table_overflow_regrows_and_reruns(golden_configs):
    """n <= 2^27 never overflows the segment table in production; SHB_SEG_CAP
    shrinks it so the circle (every point a head) overflows at 8K segments.
    The call regrows the tables to n + 2 and reruns -- with host inputs, i.e.
    on the pool stream that the regrow replaces."""
    torch_cuda()
    L = _lib.load()
    g = golden_configs["circle_200k_s3"]
    x, y = dataio.gen_circle(g["n"], g["seed"])
    L.sh_b200_release_pool()
    os.environ["SHB_SEG_CAP"] = "5000"
    try:
        r = hull.run_arrays(x, y, 1)
    finally:
        del os.environ["SHB_SEG_CAP"]
        L.sh_b200_release_pool()
    e = g["mode1"]
    assert len(r) == e["h"]
    assert oracle.fnv1a(r.x, r.y) == e["fnv1a"]
    assert [(s.iteration, s.segments, s.points_remaining, s.points_removed) for s in r.stats] == \
        [tuple(s) for s in e["stats"]]


@pytest.mark.parametrize("name", ["uniform_1m_s1", "uniform_20m_s1"])
def test_live_set_overflow_regrows_and_reruns(golden_configs, name):
    """Inputs above 2^24 points start with live sets of 3n/8; SHB_LIVE_CAP
    shrinks them below round 1's survivors so K3's capped appends flag
    ST_OVERFLOW and the call reruns with full live sets."""
    torch_cuda()
    L = _lib.load()
    g = golden_configs[name]
    x, y = dataio.gen_uniform_device(g["n"], g["seed"])
    L.sh_b200_release_pool()
    os.environ["SHB_LIVE_CAP"] = str(g["mode1"]["stats"][0][2] // 2)
    try:
        r = hull.run_arrays(x, y, 1)
    finally:
        del os.environ["SHB_LIVE_CAP"]
        L.sh_b200_release_pool()
    e = g["mode1"]
    assert len(r) == e["h"]
    assert np.array_equal(bits(r.x), bits(fromhex(e["vx"])))
    assert np.array_equal(r.indices, np.asarray(e["idx"], np.int64))
    assert [(s.iteration, s.segments, s.points_remaining, s.points_removed) for s in r.stats] == \
        [tuple(s) for s in e["stats"]]


def test_concurrent_pageable_callers():
    """Two host threads at once, both with pageable numpy inputs large enough
    for the pinned ring (one a 1M-vertex hull read back through the ring):
    every result equals its single-threaded one."""
    torch_cuda()
    ux, uy = dataio.gen_uniform(6_000_000, 21)
    cx, cy = dataio.gen_circle(1_000_000, 22)
    ru = hull.run_arrays(ux, uy, 1)
    rc = hull.run_arrays(cx, cy, 1)
    errors = []

    def worker(x, y, ref, reps):
        try:
            for _ in range(reps):
                r = hull.run_arrays(x, y, 1)
                assert np.array_equal(bits(r.x), bits(ref.x))
                assert np.array_equal(r.indices, ref.indices)
        except BaseException as ex:  # noqa: BLE001
            errors.append(repr(ex))

    th = [threading.Thread(target=worker, args=(ux, uy, ru, 6)),
          threading.Thread(target=worker, args=(cx, cy, rc, 4))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


def test_hull_multi_near_collinear_matches_reference_sharded_route():
    """Nearly collinear input: the reference's own hull(union of shard hulls)
    differs from its whole-input hull (FP predicates see different neighbours;
    tests/test_oracle.py), so the multi-GPU entry is held to the reference's
    sharded route: 3 contiguous shards, hull::run of each, hull::run
    of their union."""
    torch_cuda()
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for n in (42, 7_428, 200_000):
        t = rng.uniform(-1, 1, n)
        x, y = t, 3 * t - 1 + (rng.random(n) < 0.001) * 1e-9
        px, py = [], []
        for g in range(3):
            a, b = n * g // 3, n * (g + 1) // 3
            r = oracle.ref_hull_run(x[a:b], y[a:b], mode=1)
            px.append(r.x)
            py.append(r.y)
        sh = oracle.ref_hull_run(np.concatenate(px), np.concatenate(py), mode=1)
        m = hull.run_multi(x, y, [0, 0, 0], 1)
        same_hull(m, sh.x, sh.y, oracle.canonical_index(x, y, sh.x, sh.y), f"line {n}")


def test_async_submission_matches_sync():
    """SH_ASYNC: several hulls in flight on one stream (each holding its own
    workspace), completed out of order, equal the synchronous results; a
    ticket is waited for once; the overflow regrow also runs on completion."""
    torch = torch_cuda()
    L = _lib.load()
    inputs_ = [dataio.gen_uniform_device(3_000_000, s) for s in (1, 2, 3)]
    circle = dataio.gen_circle(200_000, 3)
    inputs_.append((torch.from_numpy(circle[0]).cuda(), torch.from_numpy(circle[1]).cuda()))
    sync = [hull.run_device(x, y, 1) for x, y in inputs_]
    pend = [hull.run_device(x, y, 1, wait=False) for x, y in inputs_]
    for i in (2, 0, 3, 1):
        r = pend[i].result()
        assert r.h == sync[i].h and r.rounds == sync[i].rounds
        assert torch.equal(r.x, sync[i].x) and torch.equal(r.indices, sync[i].indices)
        assert [tuple(vars(s).values()) for s in r.stats] == [tuple(vars(s).values()) for s in sync[i].stats]
    res = _lib.sh_hull_result()
    assert L.sh_b200_hull_wait(pend[0]._res.ticket, ctypes.byref(res)) == 102  # already waited
    # host inputs cannot be asynchronous
    with pytest.raises(RuntimeError):
        hull.PendingHull(circle[0].ctypes.data, circle[1].ctypes.data, circle[0].size, None, 1,
                         _lib.SH_ASYNC | _lib.SH_OUT_DEVICE, 0, None, hull._multi_out(8, True, 0), 0, None)
    # the regrow-and-rerun path on completion
    L.sh_b200_release_pool()
    os.environ["SHB_SEG_CAP"] = "5000"
    try:
        r = hull.run_device(inputs_[3][0], inputs_[3][1], 1, wait=False).result()
    finally:
        del os.environ["SHB_SEG_CAP"]
        L.sh_b200_release_pool()
    assert r.h == sync[3].h and torch.equal(r.x, sync[3].x)
    assert r.kernel_launches > 0

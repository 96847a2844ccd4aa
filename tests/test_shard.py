"""Multi-GPU sharding logic on CPU: world_size 2, gloo.

The product path (bench.py --gpus N) runs one process per GPU over NCCL and
hulls the gathered shard hulls with the sm_100a library.  Here the same
host-side merge code (paper_1501_04706_b200.shard) runs on two CPU processes
over gloo, with the oracle standing in for the per-shard hull (there is no
GPU in this container).  Checked: hull(union of shard hulls) == hull(all),
bit-exact coordinates, canonical GLOBAL indices, for shards with duplicates
across ranks and with empty-looking pads (h differs per rank).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1501_04706_b200 import dataio, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Hull:
    def __init__(self, x, y, idx):
        self.x = torch.from_numpy(np.ascontiguousarray(x))
        self.y = torch.from_numpy(np.ascontiguousarray(y))
        self.indices = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int64))


def _oracle_hull(x, y, mode):
    r = oracle.hull_run(x, y, mode)
    return r.x, r.y, oracle.canonical_index(x, y, r.x, r.y)


def _oracle_hull_ids(mx, my, mids, mode):
    """The C-ABI's ids rule restated for the test: the hull of the gathered
    points, each vertex reported with the lowest id among equal coordinates.
    Non-finite input raises hull.Error(NonFiniteInput), like the C-ABI."""
    from paper_1501_04706_b200 import hull
    x, y, ids = mx.numpy(), my.numpy(), mids.numpy().astype(np.int64) & 0xFFFFFFFF
    if not (np.isfinite(x).all() and np.isfinite(y).all()):
        raise hull.Error(hull.Errc.NonFiniteInput, "non-finite input")
    hx, hy, _ = _oracle_hull(x, y, mode)
    out = []
    for a, b in zip(hx, hy):
        out.append(int(ids[(x == a) & (y == b)].min()))
    return _Hull(hx, hy, np.array(out, np.int64))


def _worker(rank, world, port, x, y, mode, q, hmax=shard.HMAX):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            first, cnt = shard.shard_range(x.size, world, rank)
            lx, ly, li = _oracle_hull(x[first:first + cnt], y[first:first + cnt], mode)
            m = shard.merged_hull(_Hull(lx, ly, li), first, world, dist.all_gather_into_tensor,
                                  lambda mx, my, mids: _oracle_hull_ids(mx, my, mids, mode),
                                  hmax=hmax)
            q.put((rank, m.x.numpy().copy(), m.y.numpy().copy(), m.indices.numpy().copy()))
        finally:
            dist.destroy_process_group()
    except BaseException as e:  # surface child failures instead of a queue timeout
        q.put((rank, "error", repr(e), None))


def _run(x, y, mode, world=2, hmax=shard.HMAX):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.environ["PYTHONPATH"] = os.pathsep.join(
        [root, os.path.join(root, "tests"), os.environ.get("PYTHONPATH", "")])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, y, mode, q, hmax))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert not (isinstance(r[1], str) and r[1] == "error"), r
    for p in procs:
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("mode", [1, 2])
def test_shard_merge_equals_full_hull(mode):
    x, y = dataio.gen_uniform(60_000, 5)
    ref = oracle.hull_run(x, y, mode)
    ref_idx = oracle.canonical_index(x, y, ref.x, ref.y)
    for rank, hx, hy, hi in _run(x, y, mode):
        assert np.array_equal(hx.view(np.uint64), ref.x.view(np.uint64)), rank
        assert np.array_equal(hy.view(np.uint64), ref.y.view(np.uint64)), rank
        assert np.array_equal(hi, ref_idx), rank


def test_shard_merge_fixed_gather_overflow_falls_back():
    """Shard hulls larger than the fixed gather (hmax) send NaN payloads; the
    merge then redoes the gather with exact sizes -- same result."""
    x, y = dataio.gen_circle(2_000, 3)  # every point is a hull vertex
    ref = oracle.hull_run(x, y, 1)
    for rank, hx, hy, hi in _run(x, y, 1, hmax=64):
        assert np.array_equal(hx.view(np.uint64), ref.x.view(np.uint64)), rank
        assert np.array_equal(hi, oracle.canonical_index(x, y, ref.x, ref.y)), rank


def test_shard_merge_duplicates_across_ranks():
    # the second half repeats the first: every hull vertex exists on both
    # ranks, the merged hull must report the rank-0 (lowest) global index
    x, y = dataio.gen_circle(3_000, 9)
    X, Y = np.concatenate([x, x]), np.concatenate([y, y])
    ref = oracle.hull_run(X, Y, 1)
    for rank, hx, hy, hi in _run(X, Y, 1):
        assert np.array_equal(hx.view(np.uint64), ref.x.view(np.uint64))
        assert np.array_equal(hi, oracle.canonical_index(X, Y, ref.x, ref.y))
        assert hi.max() < x.size


def test_shard_range_covers():
    for n, w in [(10, 3), (1_000_000_000, 8), (7, 8)]:
        seen = 0
        for r in range(w):
            f, c = shard.shard_range(n, w, r)
            assert f == seen or c == 0
            seen += c
        assert seen == n

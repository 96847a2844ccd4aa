"""Multi-GPU sharding glue on CPU: world_size 2, gloo.

The product path (bench.py --gpus N; shard.merged_hull) runs one process per
GPU: the library packs each shard hull into a fixed-size payload block
(sh_b200_hull_ex + SH_OUT_PAD), ONE all-gather moves the blocks, and the
library merges them (sh_b200_hull_gathered).  There is no GPU here, so the two
library steps are replaced by stand-ins that restate the payload contract of
include/seghull_b200.h on top of the oracle; what runs for real is the glue:
block sizing, the gloo all-gather, and the overflow protocol (a shard hull
larger than the block leaves a marker with its size; every rank retries with
blocks of that size).  The library steps themselves are GPU-tested
(tests/test_multi_gpu.py, tests/test_bench_gpu.py).
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


def _pack_standin(x, y, block, *, first, mode, stream=None):
    """SH_OUT_PAD restated: {x[cap] | y[cap] | int64 global index[cap]}, vertices
    then padding (copies of vertex 0 with index -1); h > cap -> NaN x and h in
    index[0]."""
    cap = block.numel() // 3
    r = oracle.hull_run(x, y, mode)
    idx = oracle.canonical_index(x, y, r.x, r.y) + first
    h = r.x.size
    bx, by = block[:cap], block[cap:2 * cap]
    bi = block[2 * cap:].view(torch.int64)
    if h > cap:
        bx.fill_(float("nan"))
        by.zero_()
        bi.zero_()
        bi[0] = h
        return h
    pad = lambda v: np.concatenate([v, np.full(cap - h, v[0], v.dtype)])
    bx.copy_(torch.from_numpy(pad(r.x)))
    by.copy_(torch.from_numpy(pad(r.y)))
    bi.copy_(torch.from_numpy(np.concatenate([idx.astype(np.int64),
                                              np.full(cap - h, -1, np.int64)])))
    return h


def _merge_standin(g, nblocks, n_total, mode, stream=None, out_device=True):
    """sh_b200_hull_gathered restated: unpack, report an overflow marker, else the
    hull of the gathered points with the lowest id among equal coordinates."""
    cap = g.numel() // (3 * nblocks)
    b = g.view(nblocks, 3, cap)
    x = b[:, 0, :].reshape(-1).numpy()
    y = b[:, 1, :].reshape(-1).numpy()
    ids = b[:, 2, :].reshape(-1).contiguous().view(torch.int64).numpy()
    if np.isnan(x).any():
        need = [int(b[k, 2, :].contiguous().view(torch.int64)[0]) for k in range(nblocks)
                if np.isnan(float(b[k, 0, 0]))]
        return None, max(need)
    real = ids >= 0  # padding dropped
    x, y, ids = x[real], y[real], ids[real]
    r = oracle.hull_run(x, y, mode)
    out = np.array([ids[(x == a) & (y == c)].min() for a, c in zip(r.x, r.y)], np.int64)
    return (r.x, r.y, out), r.x.size


def _worker(rank, world, port, x, y, mode, q, cap):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            first, cnt = shard.shard_range(x.size, world, rank)
            (mx, my, mi), h = shard.merged_hull(
                x[first:first + cnt], y[first:first + cnt], first, x.size, world,
                dist.all_gather_into_tensor, mode=mode, block_cap=cap,
                pack=_pack_standin, merge=_merge_standin)
            q.put((rank, mx.copy(), my.copy(), mi.copy()))
        finally:
            dist.destroy_process_group()
    except BaseException as e:  # surface child failures instead of a queue timeout
        q.put((rank, "error", repr(e), None))


def _run(x, y, mode, world=2, cap=shard.HMAX):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.environ["PYTHONPATH"] = os.pathsep.join(
        [root, os.path.join(root, "tests"), os.environ.get("PYTHONPATH", "")])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, y, mode, q, cap))
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


def _check(res, x, y, mode):
    ref = oracle.hull_run(x, y, mode)
    ref_idx = oracle.canonical_index(x, y, ref.x, ref.y)
    for rank, hx, hy, hi in res:
        assert np.array_equal(hx.view(np.uint64), ref.x.view(np.uint64)), rank
        assert np.array_equal(hy.view(np.uint64), ref.y.view(np.uint64)), rank
        assert np.array_equal(hi, ref_idx), rank


@pytest.mark.parametrize("mode", [1, 2])
def test_shard_merge_equals_full_hull(mode):
    x, y = dataio.gen_uniform(60_000, 5)
    _check(_run(x, y, mode), x, y, mode)


def test_shard_merge_overflow_retries_with_needed_capacity():
    """Shard hulls larger than the block leave the overflow marker; every rank
    sees it in the gathered payload and retries with the size needed."""
    x, y = dataio.gen_circle(2_000, 3)  # every point is a hull vertex
    _check(_run(x, y, 1, cap=64), x, y, 1)


def test_shard_merge_duplicates_across_ranks():
    # the second half repeats the first: every hull vertex exists on both
    # ranks, the merged hull must report the rank-0 (lowest) global index
    x, y = dataio.gen_circle(3_000, 9)
    X, Y = np.concatenate([x, x]), np.concatenate([y, y])
    res = _run(X, Y, 1)
    _check(res, X, Y, 1)
    assert all(r[3].max() < x.size for r in res)


def test_shard_range_covers():
    for n, w in [(10, 3), (1_000_000_000, 8), (7, 8)]:
        seen = 0
        for r in range(w):
            f, c = shard.shard_range(n, w, r)
            assert f == seen or c == 0
            seen += c
        assert seen == n

"""Multi-GPU sharding of the hull.

hull(union of S_g) == hull(union of hull(S_g)): every rank hulls its contiguous
shard of the point set, the per-shard hulls are all-gathered (NCCL over
NVLink on the GPU box; any torch.distributed backend works), and every rank
hulls the gathered vertices with their GLOBAL input indices as ids, so the
merged result carries canonical global indices (lowest input index among
exact duplicates, via the ids tie-break of the C-ABI).

This is the only exchange step of the path, and it moves ~50 vertices x 24 B
per rank for uniform inputs: it is latency-bound, so it is one pair of
all-gathers (counts, then a padded payload), not a fused compute+collective
kernel.
"""
from __future__ import annotations

from typing import Callable


def pack_shard_hull(x, y, global_idx, hmax: int):
    """(3, hmax) float64 payload: x, y and global index of a shard hull, padded
    with copies of vertex 0 (a duplicate carries the same id and coordinates,
    so it changes neither the merged hull nor its canonical indices)."""
    import torch
    h = int(x.shape[0])
    buf = torch.empty((3, hmax), dtype=torch.float64, device=x.device)
    buf[0, :h] = x
    buf[1, :h] = y
    buf[2, :h] = global_idx.to(torch.float64)  # exact: indices < 2^53
    if h < hmax:
        buf[:, h:] = buf[:, :1]
    return buf


def gather_shard_hulls(x, y, global_idx, world: int, all_gather_into_tensor: Callable):
    """All-gather the shard hulls of `world` ranks.  Returns (mx, my, mids):
    the concatenated vertices and their global ids (uint32-compatible int32
    tensor, as the C-ABI's ids expect)."""
    import torch
    cnt = torch.tensor([int(x.shape[0])], dtype=torch.int64, device=x.device)
    cnts = torch.empty(world, dtype=torch.int64, device=x.device)
    all_gather_into_tensor(cnts, cnt)
    hmax = max(1, int(cnts.max().item()))
    buf = pack_shard_hull(x, y, global_idx, hmax)
    allb = torch.empty((world * 3, hmax), dtype=torch.float64, device=x.device)
    all_gather_into_tensor(allb, buf)
    allb = allb.view(world, 3, hmax)
    mx = allb[:, 0, :].reshape(-1).contiguous()
    my = allb[:, 1, :].reshape(-1).contiguous()
    mids = allb[:, 2, :].reshape(-1).to(torch.int64)
    if int(mids.max().item()) >= 2 ** 32:
        raise ValueError("global indices exceed the 32-bit ids of the C-ABI")
    return mx, my, mids.to(torch.int32).contiguous()


def shard_range(n_total: int, world: int, rank: int):
    """Contiguous shard [first, first + count) of rank `rank`."""
    per = (n_total + world - 1) // world
    first = min(n_total, rank * per)
    return first, max(0, min(per, n_total - first))


HMAX = 2048  # shard-hull vertices sent in the single-collective fast path


def gather_shard_hulls_fixed(x, y, global_idx, world: int, all_gather_into_tensor: Callable,
                             hmax: int = HMAX):
    """ONE all-gather of fixed-size (3, hmax) payloads: no count exchange and no
    host synchronisation.  A shard hull larger than hmax sends NaN coordinates
    instead, so the merge hull of the gathered set fails with NonFiniteInput
    and the caller falls back to gather_shard_hulls (exact sizes)."""
    import torch
    h = int(x.shape[0])
    if h > hmax:
        buf = torch.full((3, hmax), float("nan"), dtype=torch.float64, device=x.device)
    else:
        buf = pack_shard_hull(x, y, global_idx, hmax)
    allb = torch.empty((world * 3, hmax), dtype=torch.float64, device=x.device)
    all_gather_into_tensor(allb, buf)
    allb = allb.view(world, 3, hmax)
    mx = allb[:, 0, :].reshape(-1).contiguous()
    my = allb[:, 1, :].reshape(-1).contiguous()
    mids = allb[:, 2, :].reshape(-1).nan_to_num(0.0).to(torch.int64).to(torch.int32)
    return mx, my, mids


def merged_hull(local_hull, first: int, world: int, all_gather_into_tensor: Callable,
                hull_with_ids: Callable, hmax: int = HMAX):
    """Final hull of the union from this rank's shard hull.

    local_hull    : object with .x, .y, .indices (local indices) -- e.g. a
                    hull.DeviceHull from run_device on the rank's shard
    hull_with_ids : f(mx, my, mids) -> hull of the gathered points using mids
                    as ids (hull.run_device(..., ids=mids) on the GPU)
    The common case is one fixed-size all-gather (gather_shard_hulls_fixed);
    only when some shard hull exceeds hmax vertices (every rank sees its NaN
    payload) does it redo the gather with exact sizes.  Global indices must be
    below 2^32 (the C-ABI's ids).
    """
    import torch
    from .hull import Errc, Error
    gidx = local_hull.indices.to(dtype=torch.int64) + first
    if hmax > 0:
        mx, my, mids = gather_shard_hulls_fixed(local_hull.x, local_hull.y, gidx, world,
                                                all_gather_into_tensor, hmax)
        try:
            return hull_with_ids(mx, my, mids)
        except Error as e:  # a shard hull did not fit hmax (NaN payload)
            if e.code() != Errc.NonFiniteInput:
                raise
    mx, my, mids = gather_shard_hulls(local_hull.x, local_hull.y, gidx, world,
                                      all_gather_into_tensor)
    return hull_with_ids(mx, my, mids)

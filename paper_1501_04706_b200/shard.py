"""Multi-GPU sharding of the hull, one process per GPU.

hull(union of S_g) == hull(union of hull(S_g)): every rank hulls its contiguous
shard, the per-shard hulls are all-gathered (NCCL over NVLink on the GPU box;
any torch.distributed backend works), and every rank hulls the gathered
vertices with their GLOBAL input indices as ids, so the merged result carries
canonical global indices (lowest input index among exact duplicates).

Everything on the data path is the library's (include/seghull_b200.h):
  * the shard hull is written by the GPU as ONE fixed-size payload block
    (``hull.pack_device`` -> sh_b200_hull_ex with SH_OUT_PAD: x | y | global
    index, padded with copies of vertex 0, global index = first + local);
  * ONE all-gather of the blocks -- no count exchange, no host sync, no torch
    packing;
  * the merge (``hull.hull_gathered`` -> sh_b200_hull_gathered) unpacks the
    blocks on the device and hulls them with the global ids.
A shard hull larger than the block leaves an overflow marker carrying its
size; every rank sees the same gathered payload, so every rank takes the same
fallback: redo the step with blocks of exactly the size needed.

The in-process variant (one host thread per GPU, P2P stores into the root's
gather buffer) is ``hull.run_multi`` / ``hull.run_shards``.
"""
from __future__ import annotations

from typing import Callable

HMAX = 2048  # shard-hull vertices per payload block in the first pass


def shard_range(n_total: int, world: int, rank: int):
    """Contiguous shard [first, first + count) of rank `rank`."""
    per = (n_total + world - 1) // world
    first = min(n_total, rank * per)
    return first, max(0, min(per, n_total - first))


def merged_hull(x, y, first: int, n_total: int, world: int,
                all_gather_into_tensor: Callable, *, mode: int = 1, block_cap: int = HMAX,
                out_device: bool = True, stream=None, pack=None, merge=None):
    """Final hull of the union from this rank's shard (x, y: CUDA float64
    tensors, or host arrays -- then the H2D copy is part of the call).

    Returns ((mx, my, midx), h, launches): the merged vertices and their
    canonical global indices (device tensors when out_device).  ``pack`` and
    ``merge`` default to the library (hull.pack_device / hull.hull_gathered);
    tests on machines without a GPU inject stand-ins.
    Every rank must own at least one point (shard_range gives each rank
    points whenever n_total >= world).
    """
    import torch

    from . import hull
    pack = pack or hull.pack_device
    merge = merge or hull.hull_gathered
    if len(x) == 0:
        raise ValueError("merged_hull: this rank's shard is empty")
    if hasattr(x, "is_cuda") and x.is_cuda:
        dev = x.device
    elif torch.cuda.is_available():
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cpu")
    if n_total >= 2 ** 32 - 16:
        raise ValueError("global indices exceed the 32-bit ids of the C-ABI")
    cap = block_cap
    while True:
        # the block, the gathered payload and the merge outputs are reused
        # from step to step (a repeated step allocates nothing)
        key = (str(dev), cap, world, bool(out_device))
        bufs = _BUFS.get(key)
        if bufs is None:
            mo = None
            if out_device and dev.type == "cuda":
                mo = tuple(torch.empty(world * cap, dtype=dt, device=dev)
                           for dt in (torch.float64, torch.float64, torch.int64))
            bufs = _BUFS[key] = (torch.empty(3 * cap, dtype=torch.float64, device=dev),
                                 torch.empty(world * 3 * cap, dtype=torch.float64, device=dev), mo)
        block, gathered, mo = bufs
        pack(x, y, block, first=first, mode=mode, stream=stream)
        all_gather_into_tensor(gathered, block)
        kw = {"out": mo} if mo is not None else {}
        res, k = merge(gathered, world, n_total, mode, stream=stream, out_device=out_device, **kw)
        if res is not None:
            return res, k
        if k <= cap:
            raise RuntimeError(f"merge reported capacity {k} <= block capacity {cap}")
        cap = k  # some shard hull outgrew the block: every rank retries with its size


_BUFS: dict = {}

"""Host-side mirror of the reference's hull interface, backed by the sm_100a library.

Mirrors /root/reference/proj/core/include/seghull/hull.hpp:35-95 and
error.hpp:8-48 name for name so callers (and our parity tests) read like the
reference's own tests (tests/test_hull.cpp):

    result = hull.run(points, Mode.WithPreprocess, Backend.B200)
    result.vertices      # CCW from the leftmost vertex (hull.hpp:53-59)
    result.stats         # one SegmentStats per refinement round (hull.hpp:35-40)
    result.phase_timings # PhaseTimings (hull.hpp:42-46), device time per phase

Additions the reference does not have: ``result.indices`` (canonical input
index of each vertex), ``result.kept`` (Mode-1 filter survivors) and the
device-pointer / stream / ids options of :func:`run_arrays`.

Every compute call goes through libseghull_b200.so; there is no CPU path.
"""
from __future__ import annotations

import collections.abc
import ctypes
import enum
import threading
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib


class Errc(enum.IntEnum):
    """error.hpp:8-19"""
    EmptyInput = 0
    NonFiniteInput = 1
    DegenerateInput = 2
    InputTooLarge = 3
    InternalError = 4
    FileNotFound = 5
    ParseError = 6
    UnsupportedFormat = 7
    IoError = 8
    VerificationFailed = 9


class Error(RuntimeError):
    """error.hpp:39-48 -- single exception type; ``code()`` gives the Errc."""

    def __init__(self, code: Errc, what: str):
        super().__init__(what)
        self._code = code

    def code(self) -> Errc:
        return self._code


class CudaError(RuntimeError):
    """The CUDA runtime failed (no device, out of memory, launch failure)."""


class CapacityError(RuntimeError):
    """SH_CAP_TOO_SMALL: an output buffer is smaller than the hull."""


class Mode(enum.IntEnum):
    """hull.hpp:48-51"""
    WithPreprocess = 1
    WithoutPreprocess = 2


class Backend(enum.IntEnum):
    """primitives.hpp:14 plus the enumerator this library adds."""
    Sequential = 0
    Multicore = 1
    B200 = 2


@dataclass(frozen=True)
class Point:
    """geometry.hpp:8-13"""
    x: float
    y: float


@dataclass
class PointSet:
    """dataio.hpp:14-30 -- structure of arrays."""
    x: np.ndarray
    y: np.ndarray

    def __post_init__(self):
        self.x = np.ascontiguousarray(self.x, dtype=np.float64)
        self.y = np.ascontiguousarray(self.y, dtype=np.float64)
        if self.x.shape != self.y.shape or self.x.ndim != 1:
            raise ValueError("PointSet: x and y must be 1-D arrays of equal length")

    @classmethod
    def from_points(cls, pts: Sequence) -> "PointSet":
        return cls(np.array([float(p[0]) for p in pts]), np.array([float(p[1]) for p in pts]))

    def size(self) -> int:
        return int(self.x.size)

    def empty(self) -> bool:
        return self.x.size == 0

    def point(self, i: int) -> Point:
        return Point(float(self.x[i]), float(self.y[i]))


@dataclass(frozen=True)
class SegmentStats:
    """hull.hpp:35-40"""
    iteration: int
    segments: int
    points_remaining: int
    points_removed: int


@dataclass(frozen=True)
class PhaseTimings:
    """hull.hpp:42-46 (device milliseconds from CUDA events); total_ms is ours."""
    pre_ms: float = 0.0
    split_ms: float = 0.0
    recurse_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class HullResult:
    """hull.hpp:53-59, plus canonical input indices of the vertices."""
    x: np.ndarray
    y: np.ndarray
    indices: np.ndarray
    stats: list = field(default_factory=list)
    phase_timings: PhaseTimings = PhaseTimings()
    kept: int = 0
    rounds: int = 0
    kernel_launches: int = 0
    kernels: object = None
    round_end_ms: list = field(default_factory=list)  # device time at the end of each round
    round_phases_ms: list = field(default_factory=list)  # (table end, points end, round end)

    @property
    def vertices(self) -> list:
        return [Point(float(a), float(b)) for a, b in zip(self.x, self.y)]

    def __len__(self) -> int:
        return int(self.x.size)


_ERRC_OF_STATUS = {1 + int(e): e for e in Errc}  # status = 1 + Errc (include/seghull_b200.h)


def _raise(rc: int, msg: str):
    if rc in _ERRC_OF_STATUS:
        raise Error(_ERRC_OF_STATUS[rc], msg)
    if rc == 101:
        raise CudaError(msg or "CUDA error")
    if rc == 100:
        raise CapacityError(msg or "output capacity too small")
    raise RuntimeError(f"sh_b200_hull_ex failed with status {rc}: {msg}")


def _ptr_of(a):
    """(device_pointer, is_device) for a numpy array or a CUDA torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data, False
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
        if not a.is_contiguous():
            raise ValueError("tensor inputs must be contiguous")
        return a.data_ptr(), bool(a.is_cuda)
    raise TypeError(f"unsupported array type {type(a)!r}")


@dataclass(frozen=True)
class KernelTimings:
    """Per-kernel device milliseconds of one call (sh_kernel_ms)."""
    h2d_ms: float = 0.0
    extremes_ms: float = 0.0
    filter_ms: float = 0.0
    first_round_ms: float = 0.0
    rounds_ms: float = 0.0
    d2h_ms: float = 0.0


_ZERO_KT = KernelTimings()


def _prepare(x, y, ids):
    if isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        if ids is not None:
            if not isinstance(ids, np.ndarray):
                raise TypeError("ids must be a host array when x and y are")
            if ids.dtype != np.uint32:
                ids = np.asarray(ids)
                if ids.size and (ids.min() < 0 or ids.max() >= 2 ** 32):
                    raise ValueError("ids must lie in [0, 2^32)")
            ids = np.ascontiguousarray(ids, dtype=np.uint32)
    else:
        import torch
        if x.dtype != torch.float64 or y.dtype != torch.float64:
            raise TypeError("tensor inputs must be float64")
        if ids is not None:
            if not (hasattr(ids, "is_cuda") and ids.is_cuda == x.is_cuda
                    and (not x.is_cuda or ids.device == x.device)):
                raise ValueError("ids must live on the same device as x and y")
            if ids.dtype not in (torch.int32, torch.uint32):
                raise TypeError("tensor ids must be 32-bit integers")
    px, dx = _ptr_of(x)
    py, dy = _ptr_of(y)
    if dx != dy:
        raise ValueError("x and y must both be host arrays or both device tensors")
    n = int(x.shape[0])
    if int(y.shape[0]) != n:
        raise ValueError("x and y differ in length")
    if ids is not None and tuple(ids.shape) != (n,):
        raise ValueError(f"ids must have shape ({n},), got {tuple(ids.shape)}")
    return x, y, ids, px, py, dx, n


_tls = threading.local()


def _stats_buffer(cap: int):
    """Per-thread reusable stats array (the library writes min(rounds, cap) rows)."""
    buf = getattr(_tls, "stats", None)
    if buf is None or len(buf) < cap:
        buf = (_lib.sh_round_stat * max(cap, 64))()
        _tls.stats = buf
    return buf


class RoundList(collections.abc.Sequence):
    """Per-round records of one call, parsed on first access from a copy of the
    library's sh_round_stat rows: kind 0 = SegmentStats (hull.hpp:35-40),
    1 = device time at the end of each round (ms since K1 started),
    2 = (table phase end, point phase end, round end) in ms."""
    __slots__ = ("_raw", "_kind", "_items")

    def __init__(self, raw: bytes = b"", kind: int = 0):
        self._raw = raw
        self._kind = kind
        self._items = None

    def _get(self) -> list:
        if self._items is None:
            a = np.frombuffer(self._raw, dtype=np.uint64).reshape(-1, 7).tolist()
            if self._kind == 0:
                self._items = [SegmentStats(r[0], r[1], r[2], r[3]) for r in a]
            elif self._kind == 1:
                self._items = [r[4] * 1e-6 for r in a]
            else:
                self._items = [(r[5] * 1e-6, r[6] * 1e-6, r[4] * 1e-6) for r in a]
        return self._items

    def __getitem__(self, i):
        return self._get()[i]

    def __len__(self) -> int:
        return len(self._raw) // _ROW

    def __eq__(self, other) -> bool:
        return list(self) == list(other)

    def __repr__(self) -> str:
        return repr(self._get())


_ROW = ctypes.sizeof(_lib.sh_round_stat)


_ZERO_PH = PhaseTimings()


def _call(px, py, n, pids, mode, flags, device, stream, ox, oy, oi, capacity, stats_cap,
          id_base=0):
    L = _lib.load()
    io = getattr(_tls, "io", None)  # per-thread request/result structs, reused
    if io is None:
        io = _tls.io = (_lib.sh_hull_request(), _lib.sh_hull_result())
    req, res = io
    req.x = px
    req.y = py
    req.n = n
    req.ids = pids
    req.mode = int(mode)
    req.flags = flags
    req.device = int(device)
    req.stream = _lib.stream_handle(stream)
    req.id_base = int(id_base)
    st = _stats_buffer(stats_cap)
    res.idx = oi
    res.x = ox
    res.y = oy
    res.cap = capacity
    res.stats = ctypes.addressof(st) if stats_cap else None
    res.stats_cap = stats_cap
    rc = L.sh_b200_hull_ex(ctypes.byref(req), ctypes.byref(res))
    if rc != 0:
        _raise(rc, res.err.decode(errors="replace"))
    nst = min(int(res.rounds), stats_cap)
    raw = ctypes.string_at(ctypes.addressof(st), nst * _ROW) if nst else b""
    sts, ends, phases = RoundList(raw, 0), RoundList(raw, 1), RoundList(raw, 2)
    if flags & _lib.SH_PHASE_TIMINGS:
        ph = PhaseTimings(res.phases.pre_ms, res.phases.split_ms, res.phases.recurse_ms,
                          res.phases.total_ms)
        k = res.kernels
        kt = KernelTimings(k.h2d_ms, k.extremes_ms, k.filter_ms, k.first_round_ms, k.rounds_ms,
                           k.d2h_ms)
    else:
        ph, kt = _ZERO_PH, _ZERO_KT
    return res, sts, ph, kt, (ends, phases)


def run_arrays(x, y, mode: int = Mode.WithPreprocess, *, ids=None, device: int | None = None,
               stream: int | None = None, timings: bool = False, stats: bool = True,
               cap: int | None = None) -> HullResult:
    """Hull of (x[i], y[i]).  x/y: float64 numpy arrays or CPU tensors (host; the
    H2D copy happens inside the call) or CUDA tensors (device-resident, no H2D).
    ``ids``: optional uint32 ids (same kind as x) used for duplicate tie-breaks
    and returned as ``indices``.  The result is returned in host memory."""
    x, y, ids, px, py, dx, n = _prepare(x, y, ids)
    if device is None:
        device = int(x.device.index) if dx else 0
    if dx and stream is None:  # order the hull after torch's queued work on these tensors
        import torch
        stream = torch.cuda.current_stream(x.device).cuda_stream
    capacity = max(int(cap if cap is not None else max(n, 2)), 2)
    ox = np.empty(capacity, np.float64)
    oy = np.empty(capacity, np.float64)
    oi = np.empty(capacity, np.int64)
    flags = (_lib.SH_DEVICE_PTRS if dx else _lib.SH_HOST_PTRS) | (
        _lib.SH_PHASE_TIMINGS if timings else 0)
    res, sts, ph, kt, ends = _call(px, py, n, _ptr_of(ids)[0] if ids is not None else None, mode,
                             flags, device, stream, ox.ctypes.data, oy.ctypes.data,
                             oi.ctypes.data, capacity, (1 << 16) if stats else 0)
    h = int(res.h)
    if 2 * h < capacity:  # return compact arrays, not views of the n-sized buffers
        ox, oy, oi = ox[:h].copy(), oy[:h].copy(), oi[:h].copy()
    else:                 # most points are on the hull (the circle): views, no second pass
        ox, oy, oi = ox[:h], oy[:h], oi[:h]
    r = HullResult(ox, oy, oi, sts, ph, int(res.kept),
                   int(res.rounds), int(res.kernel_launches))
    r.kernels = kt
    r.round_end_ms, r.round_phases_ms = ends
    return r


class DeviceHull:
    """A hull whose vertices stay in HBM (SH_OUT_DEVICE): torch CUDA tensors.
    x, y, indices are views of the output buffers, created on first access
    (slicing three tensors costs more host time than the rest of the wrapper)."""
    __slots__ = ("_bufs", "_views", "h", "stats", "phase_timings", "kernels", "kept", "rounds",
                 "kernel_launches", "round_end_ms", "round_phases_ms")

    def __init__(self, x, y, indices, h: int, stats, phase_timings, kernels, kept: int,
                 rounds: int, kernel_launches: int, round_end_ms=(), round_phases_ms=()):
        self._bufs = (x, y, indices)  # full buffers (or already the views)
        self._views = None
        self.h = h
        self.stats = stats
        self.phase_timings = phase_timings
        self.kernels = kernels
        self.kept = kept
        self.rounds = rounds
        self.kernel_launches = kernel_launches
        self.round_end_ms = round_end_ms
        self.round_phases_ms = round_phases_ms

    def _v(self, i):
        if self._views is None:
            self._views = tuple(b[:self.h] for b in self._bufs)
        return self._views[i]

    x = property(lambda self: self._v(0))
    y = property(lambda self: self._v(1))
    indices = property(lambda self: self._v(2))

    def __repr__(self) -> str:
        return (f"DeviceHull(h={self.h}, rounds={self.rounds}, kept={self.kept}, "
                f"kernel_launches={self.kernel_launches})")


def run_device(x, y, mode: int = Mode.WithPreprocess, *, ids=None, stream: int | None = None,
               timings: bool = False, stats: bool = True, out=None, wait: bool = True):
    """Hull of device-resident float64 CUDA tensors; the vertices are written to
    device tensors (``out`` = (x, y, idx) buffers of equal capacity, else
    allocated at len(x)).  Only h, the stats and timings cross to the host.
    ``wait=False`` (SH_ASYNC) only enqueues the call on the stream and returns a
    :class:`PendingHull`; its ``result()`` completes it.  The host work of the
    next call then overlaps this call's device work."""
    import torch
    x, y, ids, px, py, dx, n = _prepare(x, y, ids)
    if not dx:
        raise ValueError("run_device needs CUDA tensors")
    device = int(x.device.index)
    if out is None:
        cap = max(n, 2)
        out = (torch.empty(cap, dtype=torch.float64, device=x.device),
               torch.empty(cap, dtype=torch.float64, device=x.device),
               torch.empty(cap, dtype=torch.int64, device=x.device))
    ox, oy, oi = out
    if stream is None:
        stream = torch.cuda.current_stream(x.device).cuda_stream
    flags = _lib.SH_DEVICE_PTRS | _lib.SH_OUT_DEVICE | (_lib.SH_PHASE_TIMINGS if timings else 0)
    if not wait:
        return PendingHull(px, py, n, ids, mode, flags | _lib.SH_ASYNC
                           | (0 if stats else _lib.SH_NO_STATS), device, stream, out,
                           (1 << 16) if stats else 0, (x, y))
    res, sts, ph, kt, ends = _call(px, py, n, ids.data_ptr() if ids is not None else None, mode, flags,
                             device, stream, ox.data_ptr(), oy.data_ptr(), oi.data_ptr(),
                             int(ox.shape[0]), (1 << 16) if stats else 0)
    h = int(res.h)
    return DeviceHull(ox, oy, oi, h, sts, ph, kt, int(res.kept), int(res.rounds),
                      int(res.kernel_launches), ends[0], ends[1])


class PendingHull:
    """An SH_ASYNC hull (run_device(..., wait=False)): enqueued on its stream,
    completed by result().  Keeps its inputs and outputs alive until then."""

    def __init__(self, px, py, n, ids, mode, flags, device, stream, out, stats_cap, keep):
        L = _lib.load()
        self._req, self._res = _lib.sh_hull_request(), _lib.sh_hull_result()
        req, res = self._req, self._res
        req.x, req.y, req.n = px, py, n
        req.ids = ids.data_ptr() if ids is not None else None
        req.mode, req.flags, req.device = int(mode), flags, int(device)
        req.stream = _lib.stream_handle(stream)
        ox, oy, oi = out
        res.x, res.y, res.idx, res.cap = ox.data_ptr(), oy.data_ptr(), oi.data_ptr(), int(ox.shape[0])
        self._stats_cap = stats_cap
        self._out, self._keep, self._done = out, keep, None
        self._flags = flags
        rc = L.sh_b200_hull_ex(ctypes.byref(req), ctypes.byref(res))
        if rc != 0:
            _raise(rc, res.err.decode(errors="replace"))

    def result(self) -> "DeviceHull":
        if self._done is not None:
            return self._done
        L = _lib.load()
        res = self._res
        st = (_lib.sh_round_stat * max(self._stats_cap, 1))() if self._stats_cap else None
        res.stats = ctypes.addressof(st) if st is not None else None
        res.stats_cap = self._stats_cap
        rc = L.sh_b200_hull_wait(res.ticket, ctypes.byref(res))
        if rc != 0:
            _raise(rc, res.err.decode(errors="replace"))
        nst = min(int(res.rounds), self._stats_cap)
        raw = ctypes.string_at(ctypes.addressof(st), nst * _ROW) if nst else b""
        if self._flags & _lib.SH_PHASE_TIMINGS:
            ph = PhaseTimings(res.phases.pre_ms, res.phases.split_ms, res.phases.recurse_ms,
                              res.phases.total_ms)
            k = res.kernels
            kt = KernelTimings(k.h2d_ms, k.extremes_ms, k.filter_ms, k.first_round_ms,
                               k.rounds_ms, k.d2h_ms)
        else:
            ph, kt = _ZERO_PH, _ZERO_KT
        ox, oy, oi = self._out
        self._done = DeviceHull(ox, oy, oi, int(res.h), RoundList(raw, 0), ph, kt, int(res.kept),
                                int(res.rounds), int(res.kernel_launches), RoundList(raw, 1),
                                RoundList(raw, 2))
        self._keep = None
        return self._done


def preprocess_device(x, y, *, stream: int | None = None):
    """hull::preprocess (hull.hpp:61-64, hull.cpp:53-99) on device tensors:
    returns (kept_x, kept_y, discarded) -- the points outside the strict
    interior of the extremes' quadrilateral, in input order."""
    import torch
    x, y, _, px, py, dx, n = _prepare(x, y, None)
    if not dx:
        raise ValueError("preprocess_device needs CUDA tensors")
    L = _lib.load()
    device = int(x.device.index)
    if stream is None:
        stream = torch.cuda.current_stream(x.device).cuda_stream
    ox = torch.empty(max(n, 1), dtype=torch.float64, device=x.device)
    oy = torch.empty(max(n, 1), dtype=torch.float64, device=x.device)
    kept, disc = ctypes.c_uint64(0), ctypes.c_uint64(0)
    err = ctypes.create_string_buffer(256)
    rc = L.sh_b200_preprocess(px, py, n, device, _lib.stream_handle(stream), ox.data_ptr(),
                              oy.data_ptr(), n,
                              ctypes.byref(kept), ctypes.byref(disc), err, 256)
    if rc:
        _raise(rc, err.value.decode(errors="replace"))
    k = int(kept.value)
    return ox[:k], oy[:k], int(disc.value)


# --- multi-GPU (include/seghull_b200.h sh_b200_hull_multi / _shards / _gathered) ---

@dataclass(frozen=True)
class MultiTimings:
    """sh_multi_ms: host wall-clock milliseconds of a multi-GPU call."""
    shards_ms: float
    gather_ms: float
    merge_ms: float
    total_ms: float
    shards: int
    block_cap: int


def _multi_out(cap: int, out_device, device: int):
    if out_device:
        import torch
        dev = torch.device("cuda", device)
        return (torch.empty(cap, dtype=torch.float64, device=dev),
                torch.empty(cap, dtype=torch.float64, device=dev),
                torch.empty(cap, dtype=torch.int64, device=dev))
    return np.empty(cap, np.float64), np.empty(cap, np.float64), np.empty(cap, np.int64)


def _addr(a):
    return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data


def _finish_multi(rc, h, bufs, err, tm=None):
    if rc:
        _raise(rc, err.value.decode(errors="replace"))
    ox, oy, oi = bufs
    r = HullResult(ox[:h], oy[:h], oi[:h])
    if tm is not None:
        r.kernels = MultiTimings(tm.shards_ms, tm.gather_ms, tm.merge_ms, tm.total_ms,
                                 int(tm.shards), int(tm.block_cap))
    return r


def run_multi(x, y, devices, mode: int = Mode.WithPreprocess, *, cap: int | None = None,
              out_device: bool = False) -> HullResult:
    """Hull of host arrays x, y split contiguously over ``devices`` (one host
    thread + workspace per shard inside the library; the merge runs on
    devices[0]).  Same vertices and canonical global indices as :func:`run`
    on the whole input; ``stats`` stay empty (a sharded run has no
    whole-input rounds); ``kernels`` holds the MultiTimings."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = int(x.size)
    if y.shape != x.shape:
        raise ValueError("x and y differ in length")
    L = _lib.load()
    devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
    cap = max(int(cap if cap is not None else min(max(n, 2), 1 << 22)), 2)
    while True:
        bufs = _multi_out(cap, out_device, int(devices[0]))
        h = ctypes.c_uint64(0)
        tm = _lib.sh_multi_ms()
        err = ctypes.create_string_buffer(256)
        flags = _lib.SH_HOST_PTRS | (_lib.SH_OUT_DEVICE if out_device else 0)
        rc = L.sh_b200_hull_multi(x.ctypes.data, y.ctypes.data, n, int(mode), flags, devs,
                                  len(devices), _addr(bufs[2]), _addr(bufs[0]), _addr(bufs[1]),
                                  cap, ctypes.byref(h), ctypes.byref(tm), err, 256)
        if rc == 100 and int(h.value) > cap:  # SH_CAP_TOO_SMALL: retry with the size needed
            cap = int(h.value)
            continue
        return _finish_multi(rc, int(h.value), bufs, err, tm)


def run_shards(shards, mode: int = Mode.WithPreprocess, *, root_device: int | None = None,
               cap: int = 1 << 16, out_device: bool = False) -> HullResult:
    """Hull of pre-placed shards: a list of (x, y, first) with x, y CUDA float64
    tensors on their own devices (all device-resident) -- e.g. shards that each
    GPU generated itself.  The merge runs on ``root_device`` (default: the
    first shard's device)."""
    L = _lib.load()
    arr = (_lib.sh_shard * len(shards))()
    for g, (sx, sy, first) in enumerate(shards):
        if not (sx.is_cuda and sy.is_cuda) or sx.dtype != sy.dtype or sx.shape != sy.shape:
            raise ValueError("run_shards needs equal-length float64 CUDA tensors per shard")
        arr[g].device = int(sx.device.index)
        arr[g].x, arr[g].y = sx.data_ptr(), sy.data_ptr()
        arr[g].n, arr[g].first = int(sx.shape[0]), int(first)
    root = int(arr[0].device if root_device is None else root_device)
    # tensors created by torch's stream: make them complete before other streams read them
    import torch
    for g in range(len(shards)):
        torch.cuda.synchronize(int(arr[g].device))
    while True:
        bufs = _multi_out(cap, out_device, root)
        h = ctypes.c_uint64(0)
        tm = _lib.sh_multi_ms()
        err = ctypes.create_string_buffer(256)
        flags = _lib.SH_DEVICE_PTRS | (_lib.SH_OUT_DEVICE if out_device else 0)
        rc = L.sh_b200_hull_shards(arr, len(shards), int(mode), flags, root, _addr(bufs[2]),
                                   _addr(bufs[0]), _addr(bufs[1]), cap, ctypes.byref(h),
                                   ctypes.byref(tm), err, 256)
        if rc == 100 and int(h.value) > cap:
            cap = int(h.value)
            continue
        return _finish_multi(rc, int(h.value), bufs, err, tm)


def pack_device(x, y, block, *, first: int = 0, mode: int = Mode.WithPreprocess,
                stream: int | None = None) -> int:
    """Hull of x, y written as ONE fixed-size payload block in device memory
    (SH_OUT_PAD): ``block`` is a float64 CUDA tensor of 3*cap entries
    {x[cap] | y[cap] | global index as int64 bits[cap]}; indices are offset by
    ``first``.  x, y: CUDA float64 tensors on the block's device, or host
    arrays (copied inside the call).  Returns h; h > cap leaves the overflow
    marker in the block (the merge then reports the capacity needed)."""
    import torch
    x, y, _, px, py, dx, n = _prepare(x, y, None)
    if not block.is_cuda or block.dtype != torch.float64:
        raise ValueError("pack_device needs a CUDA float64 block")
    if dx and x.device != block.device:
        raise ValueError("x, y and the block must live on one device")
    cap = int(block.numel()) // 3
    if stream is None:
        stream = torch.cuda.current_stream(block.device).cuda_stream
    flags = ((_lib.SH_DEVICE_PTRS if dx else _lib.SH_HOST_PTRS) | _lib.SH_OUT_DEVICE
             | _lib.SH_OUT_PAD | _lib.SH_NO_STATS)
    try:
        res, *_ = _call(px, py, n, None, mode, flags, int(block.device.index), stream,
                        block.data_ptr(), None, None, cap, 0, id_base=first)
    except CapacityError:  # the block carries the overflow marker
        return int(_tls.io[1].h)
    return int(res.h)


def hull_gathered(payload, nblocks: int, n_total: int, mode: int = Mode.WithPreprocess, *,
                  stream: int | None = None, out_device: bool = True, out=None):
    """The merge step of a one-process-per-GPU run: ``payload`` is the
    all-gathered float64 CUDA tensor of ``nblocks`` pack_device blocks.
    Returns ((x, y, indices), h) -- device tensors when out_device, written
    into ``out`` = (x, y, idx) buffers of nblocks * block_cap entries when
    given -- or (None, needed_cap) when a block overflowed."""
    import torch
    L = _lib.load()
    device = int(payload.device.index)
    bcap = int(payload.numel()) // (3 * nblocks)
    cap = max(2, nblocks * bcap)
    bufs = out if out is not None else _multi_out(cap, out_device, device)
    cap = min(cap, int(bufs[0].shape[0]))
    if stream is None:
        stream = torch.cuda.current_stream(payload.device).cuda_stream
    h = ctypes.c_uint64(0)
    err = ctypes.create_string_buffer(256)
    rc = L.sh_b200_hull_gathered(payload.data_ptr(), nblocks, bcap, n_total, int(mode),
                                 _lib.SH_OUT_DEVICE if out_device else 0, device,
                                 _lib.stream_handle(stream), _addr(bufs[2]), _addr(bufs[0]),
                                 _addr(bufs[1]), cap, ctypes.byref(h), err, 256)
    if rc == 100:
        return None, int(h.value)
    if rc:
        _raise(rc, err.value.decode(errors="replace"))
    k = int(h.value)
    return (bufs[0][:k], bufs[1][:k], bufs[2][:k]), k


# --- per-phase device API (hull.hpp:61-91; include/seghull_b200.h) -----------

_STATE_COLS = ("x", "y", "dist", "head", "keys", "first_pts", "flag")


@dataclass(frozen=True)
class SegmentMax:
    """primitives::SegmentMax (primitives.hpp:24-30)."""
    key: int
    value: float
    index: int


class HullState:
    """hull::HullState (hull.hpp:19-33) in HBM: one CUDA tensor per column,
    ``cap`` rows each, the first ``n`` in use.  Driven by first_split,
    compute_distances, find_farthest, split_segments, mark_interior and
    compact below, each one C-ABI call into libseghull_b200.so."""

    def __init__(self, cap: int, device: int = 0):
        import torch
        dev = torch.device("cuda", device)
        cap = max(int(cap), 1)
        f8 = dict(dtype=torch.float64, device=dev)
        i4 = dict(dtype=torch.int32, device=dev)
        self.x, self.y, self.dist = (torch.empty(cap, **f8) for _ in range(3))
        self.head, self.keys, self.first_pts, self.flag = (torch.empty(cap, **i4) for _ in range(4))
        self.device = device
        self._s = _lib.sh_hull_state()
        for k in _STATE_COLS:
            setattr(self._s, k, getattr(self, k).data_ptr())
        self._s.n = 0
        self._s.cap = cap

    @classmethod
    def from_columns(cls, device: int = 0, **cols) -> "HullState":
        """A state built from host columns (the reference tests' hand-made states)."""
        import torch
        n = len(cols["x"])
        st = cls(n, device)
        for k in _STATE_COLS:
            dt = np.float64 if k in ("x", "y", "dist") else np.int32
            getattr(st, k)[:n].copy_(torch.from_numpy(np.ascontiguousarray(cols[k], dt)))
        st._s.n = n
        return st

    @property
    def n(self) -> int:
        return int(self._s.n)

    def size(self) -> int:
        return self.n

    def segments(self) -> int:
        return 0 if self.n == 0 else int(self.keys[self.n - 1].item()) + 1

    def point(self, i: int) -> Point:
        return Point(float(self.x[i].item()), float(self.y[i].item()))

    def columns(self) -> dict:
        """Host copies of the n rows of every column."""
        return {k: getattr(self, k)[:self.n].cpu().numpy() for k in _STATE_COLS}

    def _stream(self):
        import torch
        return _lib.stream_handle(torch.cuda.current_stream(self.device).cuda_stream)


def _phase_rc(rc: int, what: str, msg: str = ""):
    if rc:
        _raise(rc, msg or what)


def first_split(x, y, *, device: int | None = None) -> HullState:
    """hull::first_split (hull.cpp:101-158): float64 CUDA tensors, or host
    arrays (uploaded first)."""
    import torch
    if isinstance(x, np.ndarray) or not getattr(x, "is_cuda", False):
        dev = 0 if device is None else device
        x = torch.as_tensor(np.ascontiguousarray(x, np.float64)).to(f"cuda:{dev}")
        y = torch.as_tensor(np.ascontiguousarray(y, np.float64)).to(f"cuda:{dev}")
    x, y = x.contiguous(), y.contiguous()
    st = HullState(int(x.shape[0]), int(x.device.index))
    err = ctypes.create_string_buffer(256)
    rc = _lib.load().sh_b200_first_split(x.data_ptr(), y.data_ptr(), int(x.shape[0]),
                                         ctypes.byref(st._s), st.device, st._stream(), err, 256)
    _phase_rc(rc, "first_split", err.value.decode(errors="replace"))
    return st


def compute_distances(st: HullState) -> None:
    """hull::compute_distances (hull.cpp:160-180)."""
    _phase_rc(_lib.load().sh_b200_compute_distances(ctypes.byref(st._s), st.device, st._stream()),
              "compute_distances")


class FarthestList(collections.abc.Sequence):
    """find_farthest's result: the device array (passed on to split_segments
    as is) and, on first access, its host copy as SegmentMax items."""

    def __init__(self, buf, m: int):
        self.buf, self.m, self._items = buf, m, None

    def _get(self):
        if self._items is None:
            raw = self.buf[:24 * self.m].cpu().numpy().tobytes()
            a = (_lib.sh_segment_max * self.m).from_buffer_copy(raw) if self.m else []
            self._items = [SegmentMax(int(e.key), float(e.value), int(e.index)) for e in a]
        return self._items

    def __getitem__(self, i):
        return self._get()[i]

    def __len__(self):
        return self.m


def find_farthest(st: HullState) -> FarthestList:
    """hull::find_farthest (hull.cpp:182-184; primitives.cpp:108-136)."""
    import torch
    cap = max(st.n, 1)
    buf = torch.empty(24 * cap, dtype=torch.uint8, device=f"cuda:{st.device}")
    m = ctypes.c_uint64(0)
    rc = _lib.load().sh_b200_find_farthest(ctypes.byref(st._s), buf.data_ptr(), cap,
                                           ctypes.byref(m), st.device, st._stream())
    _phase_rc(rc, "find_farthest")
    return FarthestList(buf, int(m.value))


def split_segments(st: HullState, farthest) -> None:
    """hull::split_segments (hull.cpp:186-194): ``farthest`` is find_farthest's
    result or any sequence of SegmentMax."""
    import torch
    if isinstance(farthest, FarthestList):
        buf, m = farthest.buf, farthest.m
    else:
        m = len(farthest)
        arr = (_lib.sh_segment_max * max(m, 1))()
        for j, e in enumerate(farthest):
            arr[j].key, arr[j].value, arr[j].index = int(e.key), float(e.value), int(e.index)
        buf = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(f"cuda:{st.device}")
    rc = _lib.load().sh_b200_split_segments(ctypes.byref(st._s), buf.data_ptr(), m, st.device,
                                            st._stream())
    _phase_rc(rc, "split_segments")


def mark_interior(st: HullState) -> None:
    """hull::mark_interior (hull.cpp:196-201)."""
    _phase_rc(_lib.load().sh_b200_mark_interior(ctypes.byref(st._s), st.device, st._stream()),
              "mark_interior")


def compact(st: HullState) -> int:
    """hull::compact (hull.cpp:203-217): returns the rows removed."""
    removed = ctypes.c_uint64(0)
    rc = _lib.load().sh_b200_compact(ctypes.byref(st._s), ctypes.byref(removed), st.device,
                                     st._stream())
    _phase_rc(rc, "compact")
    return int(removed.value)


def run(points: PointSet, mode: Mode = Mode.WithPreprocess,
        backend: Backend = Backend.B200) -> HullResult:
    """seghull::hull::run (hull.hpp:95) on the B200 backend."""
    if backend != Backend.B200:
        raise ValueError("this package implements Backend.B200 only; the Sequential/Multicore "
                         "backends are the reference's own CPU code")
    return run_arrays(points.x, points.y, mode)

"""oracle -- TEST INFRASTRUCTURE ONLY: the CPU checker for the sm_100a hull.

Two checkers live here, both loaded through ctypes:

* ``liboracle.so`` -- a plain-C restatement of the reference's hot path
  (``seghull::hull::run``, /root/reference/proj/core/src/hull.cpp:219-290),
  its generators (dataio.cpp:291-312) and its monotone-chain oracle
  (oracle.cpp:33-58).  See seghull_oracle.c for per-function citations.
* ``_ref/libseghull_ref.so`` -- the UNMODIFIED reference core compiled from
  /root/reference sources by oracle/Makefile (plus ref_shim.cpp, our C-ABI).
  It travels to the GPU box prebuilt; /root/reference itself does not.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_1501_04706_b200) never does: it fails loudly when its CUDA library is
missing instead of falling back to anything here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libseghull_ref.so")
REF_SRC = "/root/reference/proj"

_u64 = ctypes.c_uint64
_dp = ctypes.POINTER(ctypes.c_double)


class SegmentStats(ctypes.Structure):
    """hull.hpp:35-40"""

    _fields_ = [("iteration", _u64), ("segments", _u64),
                ("points_remaining", _u64), ("points_removed", _u64)]

    def as_tuple(self):
        return (self.iteration, self.segments, self.points_remaining, self.points_removed)


class PhaseTimings(ctypes.Structure):
    _fields_ = [("pre_ms", ctypes.c_double), ("split_ms", ctypes.c_double),
                ("recurse_ms", ctypes.c_double)]


ERRC = {1: "EmptyInput", 2: "NonFiniteInput", 3: "DegenerateInput",
        4: "InputTooLarge", 5: "InternalError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{ERRC.get(code, code)}: {msg}")
        self.code = code
        self.errc = ERRC.get(code, str(code))


@dataclass
class OracleHull:
    x: np.ndarray
    y: np.ndarray
    src: np.ndarray | None = None
    stats: list = field(default_factory=list)
    kept: int | None = None
    phases: tuple | None = None

    @property
    def h(self) -> int:
        return int(self.x.size)


def build(with_ref: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when the reference tree exists)."""
    targets = ["oracle"]
    if with_ref and os.path.isdir(REF_SRC):
        targets.append("ref")
        # the reference's bench harness driving Backend::B200 (needs the product library)
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1501_04706_b200",
                                       "libseghull_b200.so")):
            targets.append("hullbench")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_lib = None
_ref = None


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(with_ref=False)
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        L.or_gen_uniform.argtypes = [_u64, _u64, vp, vp]
        L.or_gen_circle.argtypes = [_u64, _u64, vp, vp]
        L.or_gen_disk.argtypes = [_u64, _u64, vp, vp]
        L.or_gen_disk.restype = _u64
        L.or_find_extremes.argtypes = [vp, vp, _u64, vp]
        L.or_preprocess.argtypes = [vp, vp, _u64, vp, vp, vp, vp]
        L.or_preprocess.restype = _u64
        L.or_first_split.argtypes = [vp, vp, _u64, vp, vp, vp]
        L.or_hull_run.argtypes = [vp, vp, _u64, ctypes.c_int, vp, vp, vp, vp, vp, _u64,
                                  vp, vp, vp]
        L.or_monotone_chain.argtypes = [vp, vp, _u64, vp, vp, vp]
        L.or_canonical_index.argtypes = [vp, vp, _u64, vp, vp, _u64, vp]
        L.or_fnv1a_vertices.argtypes = [vp, vp, _u64]
        L.or_fnv1a_vertices.restype = _u64
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref():
    """The compiled reference (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB_PATH):
            raise FileNotFoundError(
                f"{REF_LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        L = ctypes.CDLL(REF_LIB_PATH)
        vp = ctypes.c_void_p
        L.ref_gen_uniform.argtypes = [_u64, _u64, vp, vp]
        L.ref_gen_circle.argtypes = [_u64, _u64, vp, vp]
        L.ref_hull_run.argtypes = [vp, vp, _u64, ctypes.c_int, ctypes.c_int, vp, vp, _u64,
                                   vp, vp, _u64, vp, vp, ctypes.c_char_p, ctypes.c_size_t]
        L.ref_pointset_new.argtypes = [vp, vp, _u64]
        L.ref_pointset_new.restype = vp
        L.ref_pointset_free.argtypes = [vp]
        L.ref_hull_run_set.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
        L.ref_preprocess_discards.argtypes = [vp, vp, _u64]
        L.ref_preprocess_discards.restype = _u64
        L.ref_monotone_chain.argtypes = [vp, vp, _u64, vp, vp, vp]
        L.ref_preprocess.argtypes = [vp, vp, _u64, vp, vp, vp, vp]
        L.ref_write_points_binary.argtypes = [ctypes.c_char_p, vp, vp, _u64, ctypes.c_char_p,
                                              ctypes.c_size_t]
        L.ref_read_points_binary.argtypes = [ctypes.c_char_p, vp, vp, _u64, vp, ctypes.c_char_p,
                                             ctypes.c_size_t]
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.ref_state_first_split.argtypes = [vp, vp, _u64, ctypes.POINTER(ctypes.c_int)]
        L.ref_state_first_split.restype = vp
        L.ref_state_new.argtypes = [_u64, vp, vp, vp, vp, vp, vp, vp]
        L.ref_state_new.restype = vp
        L.ref_state_free.argtypes = [vp]
        L.ref_state_size.argtypes = [vp]
        L.ref_state_size.restype = _u64
        L.ref_state_get.argtypes = [vp] * 8
        for f in ("ref_state_compute_distances", "ref_state_mark_interior"):
            getattr(L, f).argtypes = [vp]
        L.ref_state_find_farthest.argtypes = [vp, vp, vp, vp, _u64]
        L.ref_state_find_farthest.restype = _u64
        L.ref_state_split_segments.argtypes = [vp, vp, vp, vp, _u64]
        L.ref_state_compact.argtypes = [vp]
        L.ref_state_compact.restype = _u64
        del i32p
        _ref = L
    return _ref


STATE_COLUMNS = ("x", "y", "dist", "head", "keys", "first_pts", "flag")


class RefHullState:
    """The reference's own hull::HullState driven through hull.hpp:61-91
    (test infrastructure: pins the device per-phase API)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def first_split(cls, x, y):
        x, y = _xy(x, y)
        code = ctypes.c_int(0)
        h = ref().ref_state_first_split(_ptr(x), _ptr(y), x.size, ctypes.byref(code))
        if not h:
            raise OracleError(code.value, "first_split")
        return cls(h)

    @classmethod
    def from_columns(cls, **cols):
        c = _state_cols(cols)
        n = c["x"].size
        return cls(ref().ref_state_new(n, *[_ptr(c[k]) for k in STATE_COLUMNS]))

    def __del__(self):
        if getattr(self, "_h", None):
            ref().ref_state_free(self._h)
            self._h = None

    def size(self) -> int:
        return int(ref().ref_state_size(self._h))

    def columns(self) -> dict:
        n = self.size()
        c = {k: np.empty(n, np.float64 if k in ("x", "y", "dist") else np.int32)
             for k in STATE_COLUMNS}
        ref().ref_state_get(self._h, *[_ptr(c[k]) for k in STATE_COLUMNS])
        return c

    def compute_distances(self):
        ref().ref_state_compute_distances(self._h)

    def find_farthest(self):
        n = self.size()
        k = np.empty(max(n, 1), np.int32)
        v = np.empty(max(n, 1), np.float64)
        i = np.empty(max(n, 1), np.uint64)
        m = int(ref().ref_state_find_farthest(self._h, _ptr(k), _ptr(v), _ptr(i), max(n, 1)))
        return k[:m].copy(), v[:m].copy(), i[:m].copy()

    def split_segments(self, key, value, index):
        key = np.ascontiguousarray(key, np.int32)
        value = np.ascontiguousarray(value, np.float64)
        index = np.ascontiguousarray(index, np.uint64)
        ref().ref_state_split_segments(self._h, _ptr(key), _ptr(value), _ptr(index), key.size)

    def mark_interior(self):
        ref().ref_state_mark_interior(self._h)

    def compact(self) -> int:
        return int(ref().ref_state_compact(self._h))


def _state_cols(cols):
    out = {}
    for k in STATE_COLUMNS:
        out[k] = np.ascontiguousarray(cols[k], np.float64 if k in ("x", "y", "dist") else np.int32)
    return out


def _xy(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError("x and y differ in length")
    return x, y


# --- generators ----------------------------------------------------------

def gen_uniform(n: int, seed: int):
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    lib().or_gen_uniform(n, seed, _ptr(x), _ptr(y))
    return x, y


def gen_circle(n: int, seed: int):
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    lib().or_gen_circle(n, seed, _ptr(x), _ptr(y))
    return x, y


def gen_disk(n: int, seed: int):
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    lib().or_gen_disk(n, seed, _ptr(x), _ptr(y))
    return x, y


# --- hull path ------------------------------------------------------------

def find_extremes(x, y):
    x, y = _xy(x, y)
    out = np.zeros(4, np.uint64)
    lib().or_find_extremes(_ptr(x), _ptr(y), x.size, _ptr(out))
    return tuple(int(v) for v in out)  # left, bottom, right, top


def preprocess(x, y):
    """hull::preprocess -> (kept_x, kept_y, kept_idx, discarded)."""
    x, y = _xy(x, y)
    n = x.size
    ox = np.empty(n, np.float64)
    oy = np.empty(n, np.float64)
    oi = np.empty(n, np.uint64)
    kept = _u64(0)
    d = lib().or_preprocess(_ptr(x), _ptr(y), n, _ptr(ox), _ptr(oy), _ptr(oi),
                            ctypes.byref(kept))
    k = kept.value
    return ox[:k], oy[:k], oi[:k], int(d)


def first_split(x, y):
    x, y = _xy(x, y)
    n = x.size
    ox = np.empty(n, np.float64)
    oy = np.empty(n, np.float64)
    head = np.empty(n, np.uint8)
    rc = lib().or_first_split(_ptr(x), _ptr(y), n, _ptr(ox), _ptr(oy), _ptr(head))
    if rc:
        raise OracleError(rc)
    return ox, oy, head


def hull_run(x, y, mode: int = 1) -> OracleHull:
    """Restated seghull::hull::run (hull.cpp:219-290)."""
    x, y = _xy(x, y)
    n = x.size
    cap = max(n, 2)
    ox = np.empty(cap, np.float64)
    oy = np.empty(cap, np.float64)
    src = np.empty(cap, np.uint64)
    h = _u64(0)
    stats_cap = 4096
    stats = (SegmentStats * stats_cap)()
    rounds = _u64(0)
    kept = _u64(0)
    bad = _u64(0)
    rc = lib().or_hull_run(_ptr(x), _ptr(y), n, mode, _ptr(ox), _ptr(oy), _ptr(src),
                           ctypes.byref(h), stats, stats_cap, ctypes.byref(rounds),
                           ctypes.byref(kept), ctypes.byref(bad))
    if rc:
        msg = f"index {bad.value}" if rc == 2 else ""
        raise OracleError(rc, msg)
    hh = h.value
    st = [stats[i].as_tuple() for i in range(min(rounds.value, stats_cap))]
    return OracleHull(ox[:hh].copy(), oy[:hh].copy(), src[:hh].copy(), st, kept.value)


def monotone_chain(x, y):
    x, y = _xy(x, y)
    n = x.size
    cap = max(n, 2)
    ox = np.empty(cap, np.float64)
    oy = np.empty(cap, np.float64)
    h = _u64(0)
    rc = lib().or_monotone_chain(_ptr(x), _ptr(y), n, _ptr(ox), _ptr(oy), ctypes.byref(h))
    if rc:
        raise OracleError(rc)
    return ox[:h.value].copy(), oy[:h.value].copy()


def canonical_index(x, y, vx, vy):
    """Lowest input index whose coordinate bits equal each vertex's."""
    x, y = _xy(x, y)
    vx, vy = _xy(vx, vy)
    out = np.empty(vx.size, np.int64)
    lib().or_canonical_index(_ptr(x), _ptr(y), x.size, _ptr(vx), _ptr(vy), vx.size, _ptr(out))
    return out


def fnv1a(vx, vy) -> str:
    vx, vy = _xy(vx, vy)
    return "%016x" % lib().or_fnv1a_vertices(_ptr(vx), _ptr(vy), vx.size)


# --- the compiled reference (oracle/_ref) --------------------------------

def ref_gen_uniform(n: int, seed: int):
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    ref().ref_gen_uniform(n, seed, _ptr(x), _ptr(y))
    return x, y


def ref_gen_circle(n: int, seed: int):
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    ref().ref_gen_circle(n, seed, _ptr(x), _ptr(y))
    return x, y


def ref_hull_run(x, y, mode: int = 1, backend: int = 0) -> OracleHull:
    """seghull::hull::run from the compiled reference; backend 0=Sequential, 1=Multicore."""
    x, y = _xy(x, y)
    n = x.size
    cap = max(n, 2)
    ox = np.empty(cap, np.float64)
    oy = np.empty(cap, np.float64)
    h = _u64(0)
    stats_cap = 4096
    stats = (SegmentStats * stats_cap)()
    rounds = _u64(0)
    ph = PhaseTimings()
    err = ctypes.create_string_buffer(256)
    rc = ref().ref_hull_run(_ptr(x), _ptr(y), n, mode, backend, _ptr(ox), _ptr(oy), cap,
                            ctypes.byref(h), stats, stats_cap, ctypes.byref(rounds),
                            ctypes.byref(ph), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    hh = h.value
    st = [stats[i].as_tuple() for i in range(min(rounds.value, stats_cap))]
    return OracleHull(ox[:hh].copy(), oy[:hh].copy(), None, st, None,
                      (ph.pre_ms, ph.split_ms, ph.recurse_ms))


def ref_preprocess_discards(x, y) -> int:
    x, y = _xy(x, y)
    return int(ref().ref_preprocess_discards(_ptr(x), _ptr(y), x.size))


def ref_monotone_chain(x, y):
    x, y = _xy(x, y)
    n = x.size
    cap = max(n, 2)
    ox = np.empty(cap, np.float64)
    oy = np.empty(cap, np.float64)
    h = _u64(0)
    rc = ref().ref_monotone_chain(_ptr(x), _ptr(y), n, _ptr(ox), _ptr(oy), ctypes.byref(h))
    if rc:
        raise OracleError(rc)
    return ox[:h.value].copy(), oy[:h.value].copy()


def ref_write_points_binary(path, x, y):
    """The reference's PTS2 writer (dataio.cpp:319-345); returns (status, message)."""
    x, y = _xy(x, y)
    err = ctypes.create_string_buffer(512)
    rc = ref().ref_write_points_binary(str(path).encode(), _ptr(x), _ptr(y), x.size, err, 512)
    return rc, err.value.decode(errors="replace")


def ref_read_points_binary(path, cap=1 << 24):
    """The reference's PTS2 reader (dataio.cpp:114-153): (status, message, x, y)."""
    x = np.empty(cap, np.float64)
    y = np.empty(cap, np.float64)
    n = ctypes.c_uint64(0)
    err = ctypes.create_string_buffer(512)
    rc = ref().ref_read_points_binary(str(path).encode(), _ptr(x), _ptr(y), cap, ctypes.byref(n),
                                      err, 512)
    return rc, err.value.decode(errors="replace"), x[:n.value].copy(), y[:n.value].copy()


def ref_preprocess(x, y):
    """The reference's hull::preprocess: (kept_x, kept_y, discarded)."""
    x, y = _xy(x, y)
    ox = np.empty(max(x.size, 1), np.float64)
    oy = np.empty(max(x.size, 1), np.float64)
    k, d = ctypes.c_uint64(0), ctypes.c_uint64(0)
    rc = ref().ref_preprocess(_ptr(x), _ptr(y), x.size, _ptr(ox), _ptr(oy), ctypes.byref(k),
                              ctypes.byref(d))
    if rc:
        raise OracleError(rc)
    return ox[:k.value].copy(), oy[:k.value].copy(), int(d.value)

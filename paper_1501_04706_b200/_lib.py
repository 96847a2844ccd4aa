"""ctypes binding of libseghull_b200.so (include/seghull_b200.h).

The shared library is built in-tree by ``paper_1501_04706_b200.build`` (nvcc,
sm_100a).  There is deliberately no fallback: if the library is missing the
import of any compute entry point raises, so a GPU test can never pass on a
silent CPU path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SHB_LIB") or os.path.join(HERE, "libseghull_b200.so")

_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_vp = ctypes.c_void_p


class sh_round_stat(ctypes.Structure):
    _fields_ = [("iteration", _u64), ("segments", _u64),
                ("points_remaining", _u64), ("points_removed", _u64), ("end_ns", _u64),
                ("table_ns", _u64), ("points_ns", _u64)]


class sh_phase_ms(ctypes.Structure):
    _fields_ = [("pre_ms", ctypes.c_double), ("split_ms", ctypes.c_double),
                ("recurse_ms", ctypes.c_double), ("total_ms", ctypes.c_double)]


class sh_kernel_ms(ctypes.Structure):
    _fields_ = [("h2d_ms", ctypes.c_double), ("extremes_ms", ctypes.c_double),
                ("filter_ms", ctypes.c_double), ("first_round_ms", ctypes.c_double),
                ("rounds_ms", ctypes.c_double), ("d2h_ms", ctypes.c_double)]


class sh_hull_request(ctypes.Structure):
    _fields_ = [("x", _vp), ("y", _vp), ("n", _u64), ("ids", _vp), ("mode", ctypes.c_int),
                ("flags", _u32), ("device", ctypes.c_int), ("stream", _vp), ("id_base", _u64)]


class sh_hull_result(ctypes.Structure):
    _fields_ = [("idx", _vp), ("x", _vp), ("y", _vp), ("cap", _u64), ("h", _u64),
                ("stats", _vp), ("stats_cap", _u64), ("rounds", _u64), ("kept", _u64),
                ("bad_index", _u64), ("phases", sh_phase_ms), ("kernels", sh_kernel_ms),
                ("kernel_launches", _u32),
                ("err", ctypes.c_char * 256), ("ticket", _u64)]


class sh_shard(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("x", _vp), ("y", _vp), ("n", _u64), ("first", _u64)]


class sh_multi_ms(ctypes.Structure):
    _fields_ = [("shards_ms", ctypes.c_double), ("gather_ms", ctypes.c_double),
                ("merge_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("shards", _u32), ("block_cap", _u64)]


class sh_hull_state(ctypes.Structure):
    _fields_ = [("x", _vp), ("y", _vp), ("dist", _vp), ("head", _vp), ("keys", _vp),
                ("first_pts", _vp), ("flag", _vp), ("n", _u64), ("cap", _u64)]


class sh_segment_max(ctypes.Structure):
    _fields_ = [("key", ctypes.c_int32), ("pad", ctypes.c_int32), ("value", ctypes.c_double),
                ("index", _u64)]


# every symbol include/seghull_b200.h declares (checked by tests/test_abi.py)
EXPORTS = ("sh_b200_hull", "sh_b200_hull_ex", "sh_b200_gen_uniform", "sh_b200_gen_disk",
           "sh_b200_gen_circle_host", "sh_b200_device_info", "sh_b200_release_pool",
           "sh_b200_abi_version", "sh_b200_read_pts2",
           "sh_b200_preprocess", "sh_b200_hull_multi", "sh_b200_hull_shards",
           "sh_b200_hull_gathered", "sh_b200_first_split", "sh_b200_compute_distances",
           "sh_b200_find_farthest", "sh_b200_split_segments", "sh_b200_mark_interior",
           "sh_b200_compact", "sh_b200_hull_wait")

SH_HOST_PTRS = 0
SH_DEVICE_PTRS = 1
SH_PHASE_TIMINGS = 2
SH_NO_STATS = 4
SH_OUT_DEVICE = 8
SH_OUT_PAD = 16
SH_ASYNC = 32
ABI_VERSION = 4

_lib = None


def load() -> ctypes.CDLL:
    """Load the CUDA library; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    L.sh_b200_hull.argtypes = [_vp, _vp, _u64, ctypes.c_int, _u32, ctypes.c_int, _vp, _vp, _vp,
                               _u64, _vp, _vp, _u64, _vp, _vp, ctypes.c_char_p, ctypes.c_size_t]
    L.sh_b200_hull_ex.argtypes = [ctypes.POINTER(sh_hull_request), ctypes.POINTER(sh_hull_result)]
    L.sh_b200_hull_wait.argtypes = [_u64, ctypes.POINTER(sh_hull_result)]
    L.sh_b200_gen_uniform.argtypes = [_vp, _vp, _u64, _u64, _u64, ctypes.c_int, _vp]
    L.sh_b200_gen_disk.argtypes = [_vp, _vp, _u64, _u64, ctypes.c_int, _vp]
    L.sh_b200_gen_circle_host.argtypes = [_vp, _vp, _u64, _u64]
    L.sh_b200_device_info.argtypes = [ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_char_p,
                                      ctypes.c_size_t]
    if hasattr(L, "sh_b200_read_pts2"):  # (absent from older builds used in A/B runs)
        L.sh_b200_read_pts2.argtypes = [ctypes.c_char_p, ctypes.c_int, _vp, _vp, _vp, _u64, _vp,
                                        ctypes.c_char_p, ctypes.c_size_t]
        L.sh_b200_read_pts2.restype = ctypes.c_int
    if hasattr(L, "sh_b200_preprocess"):
        L.sh_b200_preprocess.argtypes = [_vp, _vp, _u64, ctypes.c_int, _vp, _vp, _vp, _u64, _vp,
                                         _vp, ctypes.c_char_p, ctypes.c_size_t]
        L.sh_b200_preprocess.restype = ctypes.c_int
    L.sh_b200_hull_multi.argtypes = [_vp, _vp, _u64, ctypes.c_int, _u32, _vp, ctypes.c_int, _vp,
                                     _vp, _vp, _u64, _vp, _vp, ctypes.c_char_p, ctypes.c_size_t]
    L.sh_b200_hull_shards.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _u32, ctypes.c_int, _vp, _vp,
                                      _vp, _u64, _vp, _vp, ctypes.c_char_p, ctypes.c_size_t]
    L.sh_b200_hull_gathered.argtypes = [_vp, _u32, _u64, _u64, ctypes.c_int, _u32, ctypes.c_int,
                                        _vp, _vp, _vp, _vp, _u64, _vp, ctypes.c_char_p,
                                        ctypes.c_size_t]
    sp = ctypes.POINTER(sh_hull_state)
    L.sh_b200_first_split.argtypes = [_vp, _vp, _u64, sp, ctypes.c_int, _vp, ctypes.c_char_p,
                                      ctypes.c_size_t]
    L.sh_b200_compute_distances.argtypes = [sp, ctypes.c_int, _vp]
    L.sh_b200_find_farthest.argtypes = [sp, _vp, _u64, _vp, ctypes.c_int, _vp]
    L.sh_b200_split_segments.argtypes = [sp, _vp, _u64, ctypes.c_int, _vp]
    L.sh_b200_mark_interior.argtypes = [sp, ctypes.c_int, _vp]
    L.sh_b200_compact.argtypes = [sp, _vp, ctypes.c_int, _vp]
    for f in ("sh_b200_hull_multi", "sh_b200_hull_shards", "sh_b200_hull_gathered",
              "sh_b200_first_split", "sh_b200_compute_distances", "sh_b200_find_farthest",
              "sh_b200_split_segments", "sh_b200_mark_interior", "sh_b200_compact"):
        getattr(L, f).restype = ctypes.c_int
    L.sh_b200_release_pool.argtypes = []
    L.sh_b200_release_pool.restype = None
    L.sh_b200_abi_version.restype = ctypes.c_int
    if L.sh_b200_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH} has ABI {L.sh_b200_abi_version()}, expected {ABI_VERSION}: "
                          "rebuild it")
    _lib = L
    return L


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the (synchronising) legacy default stream


def stream_handle(s):
    """A torch stream's cuda_stream as the C-ABI's stream argument.  torch's
    default stream reports 0, which the C-ABI reads as "use the library's own
    (non-blocking) stream" -- work queued by torch before the call would then
    not be ordered before the hull.  Map it to cudaStreamLegacy instead."""
    if s is None:
        return None
    return CUDA_STREAM_LEGACY if int(s) == 0 else int(s)

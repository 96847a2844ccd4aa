"""Input generators for the hull path (dataio.hpp:44-66, dataio.cpp:291-312).

* :func:`gen_uniform` -- host, vectorised SplitMix64.  SplitMix64 is
  counter-based (draw k = mix(seed + k*0x9E3779B97F4A7C15)), so point i is
  x = draw(2i+1), y = draw(2i+2): bit-identical to the reference's loop.
* :func:`gen_uniform_device` / :func:`gen_disk_device` -- the same streams
  generated straight into HBM by sm_100a kernels (no H2D for the big configs).
* :func:`gen_circle` -- host, libm cos/sin through the C-ABI (device cos/sin
  are not bit-identical to glibc).
* :func:`gen_disk` -- host version of the disk generator SURVEY.md section 8d
  defines for config 3 (not part of the reference).
"""
from __future__ import annotations

import numpy as np

from . import _lib

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _draws(seed: int, k: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k.astype(np.uint64) * GAMMA
    return (_mix(z) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def gen_uniform(n: int, seed: int, first: int = 0, chunk: int = 1 << 22):
    """Points [first, first+n) of gen_uniform(., seed) as (x, y) float64 arrays."""
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        i = np.arange(first + a, first + b, dtype=np.uint64)
        x[a:b] = _draws(seed, 2 * i + 1)
        y[a:b] = _draws(seed, 2 * i + 2)
    return x, y


def gen_disk(n: int, seed: int, chunk: int = 1 << 22):
    """First n accepted (2u-1, 2v-1) with x*x + y*y < 1 (numpy rounds each op)."""
    xs, ys, got, c0 = [], [], 0, 0
    while got < n:
        j = np.arange(c0, c0 + chunk, dtype=np.uint64)
        px = 2.0 * _draws(seed, 2 * j + 1) - 1.0
        py = 2.0 * _draws(seed, 2 * j + 2) - 1.0
        acc = (px * px + py * py) < 1.0
        xs.append(px[acc])
        ys.append(py[acc])
        got += int(acc.sum())
        c0 += chunk
    return np.concatenate(xs)[:n].copy(), np.concatenate(ys)[:n].copy()


def gen_circle(n: int, seed: int):
    L = _lib.load()
    x = np.empty(n, np.float64)
    y = np.empty(n, np.float64)
    L.sh_b200_gen_circle_host(x.ctypes.data, y.ctypes.data, n, seed)
    return x, y


def gen_uniform_device(n: int, seed: int, first: int = 0, device: int = 0, stream=None):
    """torch float64 CUDA tensors (x, y) holding points [first, first+n)."""
    import torch
    L = _lib.load()
    dev = torch.device("cuda", device)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.sh_b200_gen_uniform(x.data_ptr(), y.data_ptr(), first, n, seed, device,
                               _lib.stream_handle(stream))
    if rc:
        raise RuntimeError(f"sh_b200_gen_uniform failed ({rc})")
    return x, y


def gen_disk_device(n: int, seed: int, device: int = 0, stream=None):
    import torch
    L = _lib.load()
    dev = torch.device("cuda", device)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.sh_b200_gen_disk(x.data_ptr(), y.data_ptr(), n, seed, device, _lib.stream_handle(stream))
    if rc:
        raise RuntimeError(f"sh_b200_gen_disk failed ({rc})")
    return x, y


# ---------------------------------------------------------------------------
# PTS2 binary point files (dataio.cpp:114-153 read, 319-345 write):
# "PTS2", u64 LE count, then count x {f64 LE x, f64 LE y}.
# ---------------------------------------------------------------------------

_PTS2 = b"PTS2"
_PTS2_DTYPE = np.dtype([("x", "<f8"), ("y", "<f8")])


def write_points_binary(path, x, y) -> None:
    """seghull::write_points(..., PointFormat::Binary) (dataio.cpp:319-345)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError("x and y differ in length")
    rec = np.empty(x.size, _PTS2_DTYPE)
    rec["x"] = x
    rec["y"] = y
    try:
        with open(path, "wb") as f:
            f.write(_PTS2)
            f.write(int(x.size).to_bytes(8, "little"))
            rec.tofile(f)
    except OSError as e:
        from .hull import Errc, Error
        raise Error(Errc.IoError, f"cannot open for writing: {path}") from e


def read_points_binary_device(path, device: int = 0, stream=None):
    """PTS2 file -> (x, y) float64 CUDA tensors, read straight to HBM by the
    library (sh_b200_read_pts2: pinned double-buffered chunks, device split).
    Errors as seghull::read_points_binary: hull.Error with Errc.FileNotFound,
    IoError, ParseError or NonFiniteInput and the reference's messages."""
    import ctypes

    import torch

    from .hull import _raise
    L = _lib.load()
    n = ctypes.c_uint64(0)
    err = ctypes.create_string_buffer(512)
    p = str(path).encode()
    rc = L.sh_b200_read_pts2(p, device, None, None, None, 0, ctypes.byref(n), err, 512)
    if rc:
        _raise(rc, err.value.decode(errors="replace"))
    dev = torch.device("cuda", device)
    x = torch.empty(n.value, dtype=torch.float64, device=dev)
    y = torch.empty(n.value, dtype=torch.float64, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.sh_b200_read_pts2(p, device, _lib.stream_handle(stream), x.data_ptr(), y.data_ptr(), n.value,
                             ctypes.byref(n), err, 512)
    if rc:
        _raise(rc, err.value.decode(errors="replace"))
    return x, y

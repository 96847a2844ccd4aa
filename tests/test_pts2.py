"""PTS2 binary point files (dataio.cpp:114-153,
319-345).  CPU: the writer is byte-identical to the reference's writer and the
reference's reader reads it back bit-exactly.  GPU: the library's loader
(sh_b200_read_pts2, file -> pinned chunks -> HBM, split to SoA on the device)
returns the reference reader's points and the reference's errors."""
import os

import numpy as np
import pytest

import oracle
from paper_1501_04706_b200 import dataio, hull

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _points(n, seed):
    x, y = dataio.gen_uniform(n, seed)
    x = x * 2e3 - 1e3
    if n >= 4:  # edge bit patterns
        x[:4] = [-0.0, 5e-324, 1.7976931348623157e308, -2.5]
        y[:4] = [0.0, -5e-324, -1e-300, 3.0]
    return x, y


@needs_ref
@pytest.mark.parametrize("n", [0, 1, 7, 100_003])
def test_writer_matches_reference_writer(tmp_path, n):
    x, y = _points(n, 3)
    ours, theirs = tmp_path / "ours.pts2", tmp_path / "ref.pts2"
    dataio.write_points_binary(ours, x, y)
    assert oracle.ref_write_points_binary(theirs, x, y)[0] == 0
    assert ours.read_bytes() == theirs.read_bytes()
    rc, msg, rx, ry = oracle.ref_read_points_binary(ours)
    assert rc == 0, msg
    assert np.array_equal(rx.view(np.uint64), x.view(np.uint64))
    assert np.array_equal(ry.view(np.uint64), y.view(np.uint64))


def _bad_files(tmp_path):
    x, y = _points(1000, 5)
    good = tmp_path / "good.pts2"
    dataio.write_points_binary(good, x, y)
    data = good.read_bytes()
    cases = {}
    cases["missing"] = tmp_path / "missing.pts2"
    p = tmp_path / "short_header.pts2"; p.write_bytes(b"PT"); cases["short_header"] = p
    p = tmp_path / "bad_magic.pts2"; p.write_bytes(b"PTS1" + data[4:]); cases["bad_magic"] = p
    p = tmp_path / "short_count.pts2"; p.write_bytes(b"PTS2\x01\x02"); cases["short_count"] = p
    p = tmp_path / "size.pts2"; p.write_bytes(data[:-5]); cases["size"] = p
    xn = x.copy(); xn[613] = np.inf
    p = tmp_path / "inf.pts2"; dataio.write_points_binary(p, xn, y); cases["inf"] = p
    yn = y.copy(); yn[77] = np.nan; yn[900] = np.nan
    p = tmp_path / "nan.pts2"; dataio.write_points_binary(p, x, yn); cases["nan"] = p
    return cases


@needs_ref
def test_reference_reader_errors_pinned(tmp_path):
    """The error codes the GPU loader must reproduce (status = 1 + Errc)."""
    want = {"missing": hull.Errc.FileNotFound, "short_header": hull.Errc.ParseError,
            "bad_magic": hull.Errc.ParseError, "short_count": hull.Errc.ParseError,
            "size": hull.Errc.ParseError, "inf": hull.Errc.NonFiniteInput,
            "nan": hull.Errc.NonFiniteInput}
    for name, path in _bad_files(tmp_path).items():
        rc, msg, _, _ = oracle.ref_read_points_binary(path)
        assert rc == 1 + int(want[name]), (name, rc, msg)


@pytest.mark.gpu
@needs_ref
def test_device_loader_errors_match_reference(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    for name, path in _bad_files(tmp_path).items():
        rc, msg, _, _ = oracle.ref_read_points_binary(path)
        with pytest.raises(hull.Error) as ei:
            dataio.read_points_binary_device(path)
        assert 1 + int(ei.value.code()) == rc, name
        assert str(ei.value).endswith(msg) or msg in str(ei.value), (name, str(ei.value), msg)


@pytest.mark.gpu
def test_device_loader_bit_exact_and_hull(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = 5_000_003  # three chunks, the last one partial
    x, y = dataio.gen_uniform(n, 21)
    path = tmp_path / "u.pts2"
    dataio.write_points_binary(path, x, y)
    dx, dy = dataio.read_points_binary_device(path)
    assert np.array_equal(dx.cpu().numpy().view(np.uint64), x.view(np.uint64))
    assert np.array_equal(dy.cpu().numpy().view(np.uint64), y.view(np.uint64))
    r = hull.run_device(dx, dy, 1)
    ref = oracle.hull_run(x, y, 1)
    assert r.h == ref.h
    assert np.array_equal(r.x.cpu().numpy().view(np.uint64), ref.x.view(np.uint64))
    empty = tmp_path / "e.pts2"
    dataio.write_points_binary(empty, np.empty(0), np.empty(0))
    ex, ey = dataio.read_points_binary_device(empty)
    assert ex.numel() == 0 and ey.numel() == 0

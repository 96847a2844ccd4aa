"""hull::preprocess as a device API (hull.hpp:61-64,
hull.cpp:53-99): K1's extremes, then the points outside the quadrilateral's
strict interior, compacted stably on the device.  Checked against the
reference's own preprocess (oracle/_ref): identical survivors, bit for bit and
in input order, identical discard counts; degenerate quadrilaterals keep all."""
import numpy as np
import pytest

import oracle
from paper_1501_04706_b200 import dataio, hull

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


def _cases():
    rng = np.random.default_rng(8)
    x, y = dataio.gen_uniform(100_000, 42)
    yield "kat_47769", x, y
    x, y = dataio.gen_uniform(3_000_001, 3)
    yield "uniform3m", x, y
    x, y = dataio.gen_circle(200_000, 4)
    yield "circle", x, y
    g = rng.integers(0, 20, size=(500_000, 2)).astype(np.float64)
    yield "grid_dups", g[:, 0].copy(), g[:, 1].copy()
    t = rng.uniform(-1, 1, 50_000)
    yield "collinear", t, 2 * t + 1  # 2 distinct corners: nothing discarded
    yield "triangle", np.array([0.0, 4, 0, 1, 1, 0.5]), np.array([0.0, 0, 4, 1, 0.5, 2])
    yield "single", np.full(1000, 3.0), np.full(1000, -1.0)
    yield "tiny", np.array([1.0]), np.array([2.0])


@pytest.mark.parametrize("name,x,y", list(_cases()), ids=[c[0] for c in _cases()])
def test_preprocess_matches_reference(name, x, y):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rx, ry, rd = oracle.ref_preprocess(x, y)
    kx, ky, d = hull.preprocess_device(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    assert d == rd, name
    assert np.array_equal(kx.cpu().numpy().view(np.uint64), rx.view(np.uint64)), name
    assert np.array_equal(ky.cpu().numpy().view(np.uint64), ry.view(np.uint64)), name
    if name == "kat_47769":
        assert d == 47769  # tests/test_hull.cpp:79


def test_preprocess_errors():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with pytest.raises(hull.Error) as ei:
        hull.preprocess_device(torch.empty(0, dtype=torch.float64, device="cuda"),
                               torch.empty(0, dtype=torch.float64, device="cuda"))
    assert ei.value.code() == hull.Errc.EmptyInput

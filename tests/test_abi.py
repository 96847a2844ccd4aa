"""CPU: the C-ABI library loads and exports every symbol include/*.h declares.

No compute calls here (there is no GPU in the CPU test environment); the
GPU suite (test_hull_gpu.py) exercises the symbols.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1501_04706_b200 import _lib, dataio, hull

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            txt = open(os.path.join(inc, f)).read()
            syms |= set(re.findall(r"\b(sh_b200_\w+)\s*\(", txt))
    return syms


def test_library_loads_and_exports_header_symbols():
    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 8
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/ but not exported"
    assert set(_lib.EXPORTS) == syms
    assert L.sh_b200_abi_version() == _lib.ABI_VERSION == 4


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_fallback_without_device():
    # n == 0 is rejected before any device work (hull.cpp:221 EmptyInput) ...
    with pytest.raises(hull.Error) as ei:
        hull.run(hull.PointSet([], []))
    assert ei.value.code() == hull.Errc.EmptyInput
    # ... and with no usable GPU the call fails loudly instead of computing on the CPU
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        with pytest.raises(hull.CudaError):
            hull.run(hull.PointSet([0.0, 1.0, 0.0], [0.0, 0.0, 1.0]))


def test_host_generators_bit_identical_to_reference_stream():
    import oracle
    x, y = dataio.gen_uniform(5000, 3)
    ox, oy = oracle.gen_uniform(5000, 3)
    assert np.array_equal(x.view(np.uint64), ox.view(np.uint64))
    assert np.array_equal(y.view(np.uint64), oy.view(np.uint64))
    # counter-based: a window of the stream equals the slice of the whole stream
    wx, wy = dataio.gen_uniform(100, 3, first=1234)
    assert np.array_equal(wx.view(np.uint64), ox[1234:1334].view(np.uint64))
    cx, cy = dataio.gen_circle(3000, 8)
    ocx, ocy = oracle.gen_circle(3000, 8)
    assert np.array_equal(cx.view(np.uint64), ocx.view(np.uint64))
    assert np.array_equal(cy.view(np.uint64), ocy.view(np.uint64))
    dx, dy = dataio.gen_disk(20000, 1)
    odx, ody = oracle.gen_disk(20000, 1)
    assert np.array_equal(dx.view(np.uint64), odx.view(np.uint64))
    assert np.array_equal(dy.view(np.uint64), ody.view(np.uint64))


def test_struct_layouts_match_header(tmp_path):
    assert ctypes.sizeof(_lib.sh_round_stat) == 56
    assert ctypes.sizeof(_lib.sh_phase_ms) == 32
    assert ctypes.sizeof(_lib.sh_hull_request) == 64
    # every ctypes mirror against the C compiler's view of include/seghull_b200.h
    names = ["sh_round_stat", "sh_phase_ms", "sh_kernel_ms", "sh_hull_request", "sh_hull_result",
             "sh_shard", "sh_multi_ms", "sh_hull_state", "sh_segment_max"]
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "seghull_b200.h"\nint main(void){\n' +
                   "".join(f'printf("%zu\\n", sizeof({n}));\n' for n in names) + "return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    sizes = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                            check=True).stdout.split()]
    for n, c_size in zip(names, sizes):
        assert ctypes.sizeof(getattr(_lib, n)) == c_size, n


def test_bench_reads_measured_peaks_layouts(tmp_path, monkeypatch):
    """bench.py's roofline peak: the driver-written MEASURED_PEAKS.json in any of
    the plausible layouts (sustained HBM preferred), else the profiling guide's
    fallback -- never a silent wrong unit."""
    import importlib.util
    import json
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    spec.loader.exec_module(bench)
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench.peaks() == (6650.0, "fallback")
    for doc, want in [({"hbm_gbs": 6460.5}, 6460.5),
                      ({"hbm": {"burst_gbs": 7000.0, "sustained_gbs": 6460.5}, "bf16_tflops": 1800}, 6460.5),
                      ({"HBM_TBps": 6.46}, 6460.0)]:
        (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps(doc))
        v, kind = bench.peaks()
        assert v == pytest.approx(want) and kind.startswith("measured")

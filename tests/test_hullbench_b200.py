"""the reference's OWN benchmark harness
(seghull::bench::run_bench: warm-up, median of repeats, monotone-chain baseline
and verification, CSV writer; core/src/bench.cpp:39-114) driving Backend::B200
through the C-ABI -- oracle/hullbench_b200.cpp, linked against the unmodified
reference objects with hull::run wrapped at link time."""
import csv
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "hullbench_b200")

pytestmark = pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/hullbench_b200 not built")


def _run(args, tmp_path):
    out = tmp_path / "records.csv"
    p = subprocess.run([EXE, *args, "--csv", str(out)], capture_output=True, text=True, timeout=600)
    rows = list(csv.DictReader(open(out))) if out.exists() else []
    return p, rows


def test_reference_harness_sequential_backend(tmp_path):
    """The harness itself (CPU backend): the reference's CSV and verify path."""
    p, rows = _run(["--gen", "uniform:50000:1", "--backend", "seq", "--repeat", "1", "--verify"],
                   tmp_path)
    assert p.returncode == 0, p.stderr
    assert [r["verified"] for r in rows] == ["true", "true"]


@pytest.mark.gpu
def test_reference_harness_b200_backend_verifies(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_04706_b200 import dataio
    pts = tmp_path / "disk.pts2"
    x, y = dataio.gen_disk(300_000, 3)
    dataio.write_points_binary(pts, x, y)
    p, rows = _run(["--gen", "uniform:1000000:1", "--gen", "circle:200000:2", "--input", str(pts),
                    "--backend", "b200", "--repeat", "2", "--verify"], tmp_path)
    assert p.returncode == 0, p.stdout + p.stderr
    assert len(rows) == 6
    assert all(r["verified"] == "true" for r in rows), rows
    hs = {(r["dataset"], r["mode"]): int(r["hull_size"]) for r in rows}
    assert hs[("uniform:1000000:1", "1")] == 40  # SURVEY.md section 8 sizes
    assert hs[("uniform:1000000:1", "1")] == hs[("uniform:1000000:1", "2")]

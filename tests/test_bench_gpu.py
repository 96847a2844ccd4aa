"""bench.py contract on the GPU box, including the N-rank path.

The N-GPU bench (torchrun, one process per GPU, NCCL all-gather of the shard
hulls) cannot run on a one-GPU box, so the N-rank code path runs with
SHB_BENCH_SHARE_GPU=1: every rank on cuda:0, the gather over gloo.  Checked:
the JSON line's contract keys, and that the merged hull of the ranks' shards
equals the one-device hull of the whole stream.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(tmp_path, nproc, extra_env=None):
    out = tmp_path / f"bench{nproc}.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc), "bench.py",
           "--gpus", str(nproc), "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
           "--json-out", str(out)]
    env = dict(os.environ, **(extra_env or {}))
    subprocess.run(cmd, cwd=ROOT, env=env, check=True, timeout=600)
    return json.loads(out.read_text())


def test_bench_two_ranks_share_one_gpu(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1501_04706_b200 import dataio, hull
    line = _bench(tmp_path, 2, {"SHB_BENCH_SHARE_GPU": "1"})
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "roofline",
              "gpu_launches", "clocks", "config"):
        assert k in line, k
    assert line["n_gpus"] == 2 and line["config"]["points_total"] == 40_000_000
    x, y = dataio.gen_uniform_device(40_000_000, 1)
    whole = hull.run_device(x, y, 1, stats=False)
    assert line["hull"]["h"] == whole.h
    # coordinates AND canonical global indices of the merged hull (sha256 of
    # x bits | y bits | int64 indices) equal the one-device hull of the stream
    import hashlib
    import numpy as np
    wx, wy = whole.x.cpu().numpy(), whole.y.cpu().numpy()
    wi = whole.indices.cpu().numpy().astype(np.int64)
    assert line["hull"]["sha256_x_y_idx"] == hashlib.sha256(
        wx.tobytes() + wy.tobytes() + wi.tobytes()).hexdigest()


def test_bench_single_gpu_line(tmp_path):
    """N = 1 default workload: the line's hull equals the reference golden."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "b1.json"
    subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3",
                    "--no-cpu-baseline", "--workload", "uniform1m", "--json-out", str(out)],
                   cwd=ROOT, check=True, timeout=600)
    line = json.loads(out.read_text())
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))["uniform_1m_s1"]
    assert line["hull"]["h"] == g["mode1"]["h"]
    assert line["hull"]["first"] == g["mode1"]["first"]
    assert line["config"]["points_total"] == 1_000_000
    assert line["e2e"]["value"] > 0 and line["e2e"]["pinned"]["value"] > 0
    assert line["gpu_launches"] > 0

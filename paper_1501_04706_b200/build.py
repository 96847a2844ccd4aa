"""In-tree build of libseghull_b200.so for sm_100a (nvcc; no JIT cache).

    python -m paper_1501_04706_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libseghull_b200.so")
SOURCES = ["k_pre.cu", "k_rounds.cu", "k_gen.cu", "k_gather.cu", "seghull_b200.cu", "pts2_io.cu",
           "phases.cu"]
HEADERS = ["device_common.cuh", "hull_kernels.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                       # no FMA contraction on the device
    # ptxas register-usage heuristics one notch above the default 5: K2 78 -> 75 us,
    # 20M uniform -2 us, disk -3 us, circle -7 us (same-box A/B, levels 8-10 alike)
    "-Xptxas", "-regUsageLevel=8",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fopenmp",  # ... nor on the host; OpenMP packs pageable H2D
    "-lgomp",
    "-I", os.path.join(ROOT, "include"),
    "-shared",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise FileNotFoundError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "seghull_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT + ".tmp", *[os.path.join(CSRC, f) for f in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

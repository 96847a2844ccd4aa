"""Golden for the 1B-point config (BASELINE.json configs[4]) from the REAL reference.

    make -C oracle ref1b
    PYTHONPATH=. python tests/golden/make_golden_1b.py [whole.json] [shards.json]

`oracle/_ref/ref_1b` links the unmodified reference core and prints the hull of
gen_uniform(1e9, 1) (see oracle/ref_1b.cpp).  Two routes, SURVEY.md section 8d:

  whole         `ref_1b 1000000000 1 0`: one seghull::hull::run(Mode 1,
                Multicore) over the whole input -- needs ~63 GB of host RAM, so
                it was run on the GPU box's host (196 GB, 16 threads, 92 s:
                tools/gpu_call1.sh) and its JSON brought back.
  shards+merge  `ref_1b 1000000000 1 8`: 8 shard runs plus a merge run (fits in
                this container's 62 GB; 8 threads, 179 s).

Both routes must give the same vertices and canonical indices; the entry keeps
the whole run's per-round SegmentStats (the shard route has none) and the
shard route's per-shard hull sizes.  Without arguments both routes are run
here (the whole one only if RAM allows).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_1b")


def run(shards: int) -> dict:
    out = subprocess.run([BIN, "1000000000", "1", str(shards)], check=True,
                         capture_output=True, text=True).stdout
    return json.loads(out)


def main():
    whole = json.load(open(sys.argv[1])) if len(sys.argv) > 1 else run(0)
    shards = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else run(8)
    w, s = whole["mode1"], shards["mode1"]
    for k in ("h", "fnv1a", "vx", "vy", "idx"):
        assert w[k] == s[k], f"routes disagree on {k}"
    ent = {"generator": "uniform", "n": whole["n"], "seed": whole["seed"],
           "routes": {"whole": {"threads": whole["threads"], "seconds": whole["seconds"]},
                      "shards+merge": {"shards": shards["shards"], "threads": shards["threads"],
                                       "seconds": shards["seconds"]}},
           "mode1": {"h": w["h"], "rounds": w["rounds"], "stats": w["stats"], "fnv1a": w["fnv1a"],
                     "first": w["first"], "vx": w["vx"], "vy": w["vy"], "idx": w["idx"],
                     "shard_h_8": s["shard_h"]}}
    path = os.path.join(HERE, "configs.json")
    cfg = json.load(open(path))
    cfg["uniform_1b_s1"] = ent
    with open(path, "w") as f:
        json.dump(cfg, f, indent=1)
    print("uniform_1b_s1:", w["h"], "vertices,", w["rounds"], "rounds")


if __name__ == "__main__":
    main()

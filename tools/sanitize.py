"""compute-sanitizer driver: a few hulls that take every round-kernel path
(small / medium / large tables, solo tail, one-CTA inputs), checked against
the oracle.  Run under the sanitizer on the box:

    compute-sanitizer --tool memcheck python tools/sanitize.py
    SCALE=0.2 compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1501_04706_b200 import dataio, hull  # noqa: E402

k = float(os.environ.get("SCALE", "1"))  # racecheck is slow: SCALE=0.2
cases = [("uniform", dataio.gen_uniform(int(2e6 * k), 3)), ("disk", dataio.gen_disk(int(1e6 * k), 3)),
         ("circle", dataio.gen_circle(int(1e6 * k), 3)), ("small", dataio.gen_uniform(5_000, 3))]
# a 900-vertex hull over an interior disk: the solo tail with more than 512 segments
_t = np.arange(900) * (2 * np.pi / 900)
_ix, _iy = dataio.gen_disk(int(2e5 * k), 4)
cases.append(("ring900", (np.concatenate([np.cos(_t), 0.99 * _ix]), np.concatenate([np.sin(_t), 0.99 * _iy]))))
for name, (x, y) in cases:
    for mode in (1, 2):
        r = hull.run_arrays(x, y, mode)
        ref = oracle.hull_run(x, y, mode)
        ok = np.array_equal(np.asarray(r.x), np.asarray(ref.x)) and np.array_equal(np.asarray(r.y), np.asarray(ref.y))
        print(f"{name} m{mode}: h={len(r)} rounds={r.rounds} {'ok' if ok else 'MISMATCH'}", flush=True)

# the multi-GPU entry points (3 shards on this device: K5-pack into the gather
# buffer, k_count / k_unpack, the merge) and the per-phase device API
for name, (x, y) in [("multi uniform", dataio.gen_uniform(int(3e5 * k) + 3, 5)),
                     ("multi circle", dataio.gen_circle(int(1e5 * k) + 3, 5))]:
    m = hull.run_multi(x, y, [0, 0, 0], 1)
    ref = oracle.hull_run(x, y, 1)
    ok = np.array_equal(np.asarray(m.x), np.asarray(ref.x)) and np.array_equal(np.asarray(m.y), np.asarray(ref.y))
    print(f"{name}: h={len(m)} {'ok' if ok else 'MISMATCH'}", flush=True)
x, y = dataio.gen_uniform(5000, 9)
st = hull.first_split(x, y)
for _ in range(64):
    hull.compute_distances(st)
    far = hull.find_farthest(st)
    if not any(f.value > 0.0 for f in far) and st.size() == len(far):
        break
    hull.split_segments(st, far)
    hull.mark_interior(st)
    hull.compact(st)
ref = oracle.hull_run(x, y, 2)
c = st.columns()
ok = np.array_equal(c["x"], ref.x) and np.array_equal(c["y"], ref.y)
print(f"phases uniform 5000: h={st.size()} {'ok' if ok else 'MISMATCH'}", flush=True)

"""Hot SASS of one kernel from `ncu -i REP --page source --csv --print-source sass`:
stall reasons summed, dynamic instruction mix, top instructions by stall samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
seen = {}
for r in data:
    if len(r) > iE and r[iS].isdigit() and r[0] not in seen:
        seen[r[0]] = r
data = list(seen.values())
tot = sum(int(r[iS]) for r in data)
print("stall samples", tot, "warp instructions", sum(int(r[iE] or 0) for r in data if r[iE].isdigit()))
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.Counter()
for r in data:
    for c in stalls:
        v = r[h.index(c)]
        if v.isdigit():
            agg[c] += int(v)
for c, v in agg.most_common(8):
    print(f"  {c:28s} {100 * v / tot:5.1f}%")
for r in sorted(data, key=lambda r: -int(r[iS]))[:top]:
    j = max(stalls, key=lambda c: int(r[h.index(c)]) if r[h.index(c)].isdigit() else 0)
    print(f"{int(r[iS]):6d} {100 * int(r[iS]) / tot:5.1f}% {r[0][-5:]} {r[1][:70]:70s} {j}")

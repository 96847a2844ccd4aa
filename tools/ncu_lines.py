"""Top source lines of an ncu --page source --print-source cuda,sass CSV by warp-stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = None; out = []; hdr = None
for r in rows:
    if r and r[0] == "File Path": f = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if len(r) > 4 and r[0] and r[2] == "-":
        try: out.append((int(r[4]), f, int(r[0]), r[1][:90], r))
        except ValueError: pass
tot = sum(o[0] for o in out); print("total samples", tot)
for o in sorted(out, key=lambda o: -o[0])[:k]:
    r = o[4]
    vals = sorted([(int(v), hdr[j]) for j, v in enumerate(r) if j >= 34 and j < len(hdr) and v.isdigit() and 'Not Issued' not in hdr[j]], reverse=True)[:2]
    print(f"{o[0]:7d} {100*o[0]/tot:5.1f}% {o[1]}:{o[2]} {o[3]} {[(v, n.replace('stall_', '')) for v, n in vals]}")

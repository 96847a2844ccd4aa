"""Dynamic SASS instruction mix of one kernel in an ncu report: python tools/ncu_mix.py REP KERNEL_REGEX N_POINTS"""
import collections, csv, subprocess, sys
rep, kre, n = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
ie = hdr.index("Instructions Executed"); src = hdr.index("Source"); ad = hdr.index("Address")
cnt = collections.Counter(); tot = 0
seen = set()
for r in data:
    if len(r) <= ie or not r[ie].isdigit() or r[ad] in seen: continue  # the CSV repeats rows
    seen.add(r[ad])
    op = r[src].split()
    if not op: continue
    o = op[1] if op[0].startswith('@') else op[0]
    o = o.split('.')[0]
    cnt[o] += int(r[ie]); tot += int(r[ie])
print(rows[0][1], f"warp-instr {tot}  thread-instr/pt {tot * 32 / n:.1f}")
print("  ".join(f"{o}:{c * 32 / n:.1f}" for o, c in cnt.most_common(24)))

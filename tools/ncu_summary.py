"""Summarise an ncu --set full report: key metrics per kernel (run here, not on the box)."""
import csv, io, subprocess, sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "L2 Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, si, ni, ui, vi, ii = (h.index(k) for k in ("Kernel Name", "Section Name", "Metric Name",
                                                    "Metric Unit", "Metric Value", "ID"))
    seen = {}
    for r in rows[1:]:
        if len(r) <= vi or r[ni] not in KEYS:
            continue
        seen.setdefault((r[ii], r[ki][:60]), {})[r[ni]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    traffic = {}
    if rr:
        hh = rr[0]
        try:
            ii2, rdi, wri = hh.index("ID"), hh.index("dram__bytes_read.sum"), hh.index("dram__bytes_write.sum")
            for r in rr[2:]:
                traffic[r[ii2]] = (r[rdi], r[wri], rr[1][rdi], rr[1][wri])
        except ValueError:
            pass
    for (i, k), m in seen.items():
        print(f"== [{i}] {k}")
        for key in KEYS:
            if key in m:
                print(f"   {key:40s} {m[key]}")
        if i in traffic:
            t = traffic[i]
            print(f"   {'dram read / write':40s} {t[0]} {t[2]} / {t[1]} {t[3]}")


if __name__ == "__main__":
    main(sys.argv[1])

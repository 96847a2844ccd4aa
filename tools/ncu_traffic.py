"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of one
ncu --set full capture -> profiles/ncu_traffic.json, read by bench.py for the
`roofline.traffic` field.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep uniform20m
"""
import csv
import io
import json
import os
import subprocess
import sys

NAMES = {"k1_extremes": "k1_extremes", "k2_classify": "k2_filter", "k3_round1": "k3_route_round1",
         "k_rounds": "k_rounds"}


def main(rep, workload):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    res = {}
    for r in rows[2:]:
        name = next((v for k, v in NAMES.items() if k in r[ki]), None)
        if not name:
            continue
        def val(metric):
            i = h.index(metric)
            v = float(r[i].replace(",", ""))
            u = units[i]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1,
                        "usecond": 1e3, "msecond": 1e6}.get(u, 1)
        ti = h.index("gpu__time_duration.sum")
        res[name] = {"dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                     "ncu_duration": f"{r[ti]} {units[ti]}"}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_traffic.json")
    try:
        with open(path) as f:
            allres = json.load(f)
    except Exception:
        allres = {}
    allres[workload] = res
    with open(path, "w") as f:
        json.dump(allres, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

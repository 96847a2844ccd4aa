"""Profiling driver: R hulls of one device-resident workload (for ncu; never a bench number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1501_04706_b200 import dataio, hull  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "uniform"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 20_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if kind == "uniform":
    x, y = dataio.gen_uniform_device(n, 1)
elif kind == "disk":
    x, y = dataio.gen_disk_device(n, 1)
else:
    hx, hy = dataio.gen_circle(n, 1)
    x, y = torch.from_numpy(hx).cuda(), torch.from_numpy(hy).cuda()
torch.cuda.synchronize()
trace = int(os.environ.get("TRACE_ROUND", "0"))
if trace:
    import ctypes
    from paper_1501_04706_b200 import _lib
    L = _lib.load()
    L.sh_b200_debug_trace_round(trace)
for _ in range(reps):
    r = hull.run_device(x, y, 1, timings=True)
    print(kind, n, "h", r.h, "rounds", r.rounds, r.kernels, r.phase_timings, flush=True)
    print("   round end (ms since K1 start):", [round(t, 4) for t in r.round_end_ms], flush=True)
    prev = 0.0
    for i, (ta, tp, te) in enumerate(r.round_phases_ms):
        if ta:
            print(f"   round {i+1}: table {1e3*(ta-prev):7.1f} us  points {1e3*(tp-ta):7.1f} us  close {1e3*(te-tp):7.1f} us", flush=True)
        prev = te
    if trace:
        buf = (ctypes.c_ulonglong * 32)()
        k = L.sh_b200_debug_last_timeline(buf, 32)
        ts = [buf[i] / 1e3 for i in range(k)]
        if trace == 255:
            print("   kernel marks (us): K1 end %.1f | K2 start %.1f end %.1f | K3 start %.1f end %.1f | KR start %.1f end %.1f" % tuple(ts[0:7]))
        else:
            print(f"   trace round {trace} (us since K1 start: start, table, prefix, points, flush, barrier, [winner]):", [round(t, 2) for t in ts])
        cb = (ctypes.c_ulonglong * 2048)()
        L.sh_b200_debug_last_ctas(cb, 2048)
        if trace == 255:
            import statistics
            for name, off in (("K1", 0), ("K2", 256), ("K3", 512)):
                e = sorted(cb[off + i] / 1e3 for i in range(148) if cb[off + i])
                if e:
                    print(f"   {name} CTA stream ends: min {e[0]:.1f} median {statistics.median(e):.1f} "
                          f"p90 {e[int(len(e) * 0.9)]:.1f} max {e[-1]:.1f} us", flush=True)
            for name, off in (("K1 end", 1024), ("K2 end", 1200), ("K3 streams (all warps)", 1400)):
                e = sorted(cb[off + i] / 1e3 for i in range(148) if cb[off + i])
                if e:
                    print(f"   {name}: min {e[0]:.1f} median {statistics.median(e):.1f} "
                          f"p90 {e[int(len(e) * 0.9)]:.1f} max {e[-1]:.1f} us", flush=True)
            print("   CTA0 entry/past-wait (us): K2 %.1f/%.1f K3 %.1f/%.1f KR %.1f/%.1f"
                  % tuple(cb[1600 + k] / 1e3 for k in range(6)), flush=True)
            print("   K3 CTA0 partials loaded %.1f, lexmin done %.1f | K2 CTA0 K1-partials loaded %.1f, "
                  "extremes done %.1f, fin written %.1f | K3 close: ticket %.1f runs summed %.1f rows combined %.1f"
                  % tuple(cb[1606 + k] / 1e3 for k in range(8)),
                  flush=True)
            continue
        ends = sorted(cb[i] / 1e3 for i in range(1024) if cb[i])
        slow = sorted((cb[i] / 1e3, i) for i in range(1024) if cb[i])[-10:]
        print("   slowest CTAs (end us, cta):", [(round(t, 1), i) for t, i in slow])
        if ends:
            import statistics
            print(f"   CTA point-phase ends: n={len(ends)} min {ends[0]:.1f} median {statistics.median(ends):.1f} max {ends[-1]:.1f} us; deciles",
                  [round(ends[int(len(ends) * d / 10)], 1) for d in range(10)])

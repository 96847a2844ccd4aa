"""bench.py -- B200 benchmark of the segment-based QuickHull hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload uniform20m]
                    [--impl b200|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

A "step" is one convex hull of one batch of synthetic points (BASELINE.json
metric "Mpoints/s and ms per 20M-point 2D hull"):

* N = 1: the 20M-uniform hull of gen_uniform(20e6, seed 1) (BASELINE.json
  configs[1], the paper's headline size), inputs resident in HBM.
* N > 1 (one process per GPU, NCCL): weak scaling -- rank r owns points
  [r*20M, (r+1)*20M) of the counter-based stream gen_uniform(N*20M, 1),
  generated on its own GPU.  Each rank's GPU hulls its shard and writes it as
  one fixed-size payload block (SH_OUT_PAD), ONE all-gather moves the blocks
  over NVLink (NCCL), and every rank's library merges them
  (sh_b200_hull_gathered; hull(union) == hull(union of shard hulls), SURVEY.md
  section 8e).  `value` = all points of the job / max-over-ranks time.

Also reported (one JSON line, rank 0):
  e2e           the same step through the public API with HOST inputs (H2D of
                x, y and D2H of the hull inside the timed region): pageable
                numpy arrays (the reference's caller passes std::vectors), and
                pinned buffers as a second figure
  roofline      the dominant kernel's algorithmic bytes / its CUDA-event time vs
                the measured HBM copy peak (MEASURED_PEAKS.json)
  cpu_baseline  the reference's own CPU path (oracle/_ref: seghull::hull::run,
                Backend::Multicore, all host threads) on the same points, rank 0, N = 1
  clocks        pynvml samples of SM clocks + throttle reasons during the timed region

`--impl reference` times the reference's CPU implementation (oracle/_ref, the
unmodified reference core compiled from its sources) on the same workload and
prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (generator, points per rank (weak) or total (strong), scaling, seed)
    "uniform1m": ("uniform", 1_000_000, "weak", 1),      # BASELINE.json configs[0]
    "uniform20m": ("uniform", 20_000_000, "weak", 1),    # configs[1]: the headline
    "disk20m": ("disk", 20_000_000, "weak", 1),
    "circle4m": ("circle", 4_000_000, "weak", 1),
    "uniform1b": ("uniform", 1_000_000_000, "strong", 1),
}
BASELINE_MPTS = 20_000_000 / 206.0e-3 / 1e6  # 20M uniform, Mode 1, 206.0 ms (K20c)
METRIC = "Mpoints/s (2D convex hull, Mode 1 = with quadrilateral filter)"
L2_BYTES = 126 * 1024 * 1024


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--workload", default="uniform20m", choices=sorted(WORKLOADS))
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--mode", type=int, default=1, choices=[1, 2])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--l2-flush", action="store_true",
                   help="flush L2 between timed steps even when the input is over 2x the L2 "
                        "(inputs up to 2x L2 are always flushed)")
    p.add_argument("--json-out", default=None)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def shard_of(workload, world, rank):
    kind, n, scaling, seed = WORKLOADS[workload]
    if scaling == "weak":
        n_rank, n_total = n, n * world
    else:
        n_total = n
        n_rank = (n + world - 1) // world
    first = rank * n_rank
    n_rank = max(0, min(n_rank, n_total - first))
    return kind, seed, first, n_rank, n_total, scaling


def l2_policy(a, n_rank):
    """(flush between timed steps?, the config note saying which)."""
    in_bytes = 16 * n_rank
    do_flush = a.l2_flush or in_bytes <= 2 * L2_BYTES
    note = (f"flushed between timed steps ({2 * L2_BYTES >> 20} MB write); input "
            f"16 B/pt x {n_rank}" if do_flush else
            f"no flush: input 16 B/pt x {n_rank} = {in_bytes >> 20} MB > "
            f"2 x {L2_BYTES >> 20} MB L2")
    return do_flush, note


def config_of(a, world):
    """The workload description -- identical in both arms (b200 and reference)."""
    kind, seed, first, n_rank, n_total, scaling = shard_of(a.workload, world, 0)
    return {"workload": a.workload, "generator": kind, "seed": seed,
            "points_per_gpu": n_rank, "points_total": n_total, "mode": a.mode,
            "parallelism": f"shard{world}" + ("+allgather_merge" if world > 1 else ""),
            "l2": l2_policy(a, n_rank)[1]}


def peaks():
    """HBM GB/s from the driver-written MEASURED_PEAKS.json (its layout is not
    fixed here: the first numeric entry under a key naming HBM, preferring the
    sustained figure -- the dominant kernel is timed inside a long step -- over
    the burst one), else the B200_PROFILING.md fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except Exception:
        return 6650.0, "fallback"

    found = []

    def walk(node, path):
        if isinstance(node, dict):
            for k, v in node.items():
                walk(v, path + [str(k).lower()])
        elif isinstance(node, (int, float)) and not isinstance(node, bool):
            key = "/".join(path)
            if "hbm" in key or "copy" in key or "dram" in key:
                found.append((key, float(node)))

    walk(p, [])
    tb = [(k, v * 1000.0 if v < 100 else v) for k, v in found]  # TB/s -> GB/s
    for pref in ("sustain", "gbs", "gb/s", "bw", ""):
        for k, v in tb:
            if pref in k and 1000.0 < v < 20000.0:
                return v, "measured (MEASURED_PEAKS.json: " + k + ")"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks: pynvml samples during the timed region
# ---------------------------------------------------------------------------

REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x2: "applications_clocks_setting", 0x100: "display_clock_setting",
           0x10: "sync_boost"}


class ClockSampler:
    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for bit, name in REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.005)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference core, or the C port)
# ---------------------------------------------------------------------------

def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_timer(x_host, y_host, mode):
    """Returns (run_once() -> seconds, kind, cores, description)."""
    import ctypes
    import numpy as np
    import oracle  # test/bench infrastructure: the CPU reference leg only
    x_host = np.ascontiguousarray(x_host)
    y_host = np.ascontiguousarray(y_host)
    if oracle.ref_available():
        R = oracle.ref()
        ps = R.ref_pointset_new(x_host.ctypes.data, y_host.ctypes.data, x_host.size)
        h = ctypes.c_uint64(0)

        def once():
            t0 = time.perf_counter()
            rc = R.ref_hull_run_set(ps, mode, 1, ctypes.byref(h))
            dt = time.perf_counter() - t0
            if rc:
                raise RuntimeError(f"reference hull::run failed ({rc})")
            return dt
        return once, "reference", host_cores(), "seghull::hull::run(Mode 1, Backend::Multicore)"

    def once_port():
        t0 = time.perf_counter()
        oracle.hull_run(x_host, y_host, mode)
        return time.perf_counter() - t0
    return once_port, "port", 1, "oracle C restatement of hull::run (sequential)"


def cpu_sample_points(kind, seed, first, n):
    """Host copy of the same points the GPU hulls (bounded sample = first n of the shard)."""
    import oracle
    if kind == "uniform":
        from paper_1501_04706_b200 import dataio
        return dataio.gen_uniform(n, seed, first=first)
    if kind == "disk":
        x, y = oracle.gen_disk(first + n, seed)
        return x[first:], y[first:]
    x, y = oracle.gen_circle(first + n, seed)
    return x[first:], y[first:]


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0  # rank 0 alone runs the CPU reference; the others exit without work
    kind, seed, first, n_rank, n_total, scaling = shard_of(a.workload, world, 0)
    # bounded sample: the whole job when it fits ~3 minutes, else one shard-sized
    # sample (Mpoints/s is size-normalised), else fewer points
    budget_s = 150.0
    n = min(n_total, 20_000_000)
    x, y = cpu_sample_points(kind, seed, 0, n)
    once, kindref, cores, desc = cpu_reference_timer(x, y, a.mode)
    t_first = once()
    est = t_first * (a.steps + a.warmup)
    while est > budget_s and n > 1_000_000:
        n //= 2
        x, y = x[:n].copy(), y[:n].copy()
        once, kindref, cores, desc = cpu_reference_timer(x, y, a.mode)
        t_first = once()
        est = t_first * (a.steps + a.warmup)
    for _ in range(max(0, a.warmup - 1)):
        once()
    times = [once() for _ in range(a.steps)]
    t = sum(times) / len(times)
    value = n / t / 1e6
    sample = f"{desc} on the first {n} points of the {a.workload} stream (seed {seed}), " \
             f"{a.steps} timed runs after {a.warmup} warm-up"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mpoints/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": value / BASELINE_MPTS,
        "dtype": "f64", "data": "synthetic",
        "config": config_of(a, world),
        "cpu_baseline": {"value": value, "unit": "Mpoints/s", "cores": cores, "kind": kindref,
                         "sample": sample},
        "e2e": {"value": value, "unit": "Mpoints/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line, a)
    return 0


def emit(line, a):
    s = json.dumps(line)
    print(s, flush=True)
    if a.json_out:
        with open(a.json_out, "w") as f:
            f.write(s + "\n")


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1501_04706_b200 import _lib, dataio, hull

    world, rank, local = dist_env()
    # SHB_BENCH_SHARE_GPU=1 (test only): every rank on cuda:0 and the gather
    # over gloo through host tensors, to exercise the N-rank path on one GPU
    share = world > 1 and os.environ.get("SHB_BENCH_SHARE_GPU") == "1"
    if share:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    elif world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    devi = dev.index
    _lib.load()
    kind, seed, first, n_rank, n_total, scaling = shard_of(a.workload, world, rank)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    # --- inputs resident in HBM (generated on the device where bit-identical) ---
    if kind == "uniform":
        x, y = dataio.gen_uniform_device(n_rank, seed, first=first, device=devi, stream=sp)
    elif kind == "disk":
        gx, gy = dataio.gen_disk_device(first + n_rank, seed, device=devi, stream=sp)
        x, y = gx[first:].clone(), gy[first:].clone()
        del gx, gy
    else:
        hx, hy = dataio.gen_circle(first + n_rank, seed)
        x = torch.from_numpy(hx[first:].copy()).to(dev)
        y = torch.from_numpy(hy[first:].copy()).to(dev)
    torch.cuda.synchronize()

    cap = max(n_rank, 2)
    out = (torch.empty(cap, dtype=torch.float64, device=dev),
           torch.empty(cap, dtype=torch.float64, device=dev),
           torch.empty(cap, dtype=torch.int64, device=dev))
    launches = [0]

    from paper_1501_04706_b200 import shard as shardmod

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if share else dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_gather(out, inp):
        if not share:
            return dist.all_gather_into_tensor(out, inp)
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu())
        out.copy_(o)

    def merged(px, py, out_device=True):
        """N > 1: this rank's shard hull packed by the GPU into one payload block,
        ONE all-gather (NCCL over NVLink), the library's merge on every rank."""
        res, h = shardmod.merged_hull(px, py, first, n_total, world, all_gather, mode=a.mode,
                                      out_device=out_device, stream=sp)
        # shard: K1, K2, K3, KR, K5-pack; merge: unpack, one-CTA pre + KR, K5 (device out)
        launches[0] += 9 if out_device else 8
        return res, h

    class _Final:
        def __init__(self, res, h):
            self.h = h
            self.x, self.y, self.indices = res

    def step(timings=False):
        if world > 1 and not timings:
            res, h = merged(x, y)
            return _Final(res, h), None
        dh = hull.run_device(x, y, a.mode, stream=sp, timings=timings, out=out)
        launches[0] += dh.kernel_launches
        return dh, dh

    # L2 between timed steps: inputs over 2x the L2 (320 MB for 20M points vs the
    # 126 MB L2) rely on their size (the contract's option "inputs larger than
    # L2"; a flush would also leave ~126 MB of dirty lines for K1 to write back);
    # smaller inputs get a flush (a write of 2x L2) outside the events, and
    # --l2-flush forces it for any size
    do_flush, _ = l2_policy(a, n_rank)
    flush = torch.empty(2 * L2_BYTES // 4 if do_flush else 1, dtype=torch.int32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # N = 1: each hull is submitted asynchronously (SH_ASYNC) and completed
    # after the next one is submitted, so the host side of hull i+1 (Python,
    # launches) overlaps the device work of hull i; every hull still runs in
    # full, in stream order, after its own L2 flush.  Two output buffers
    # alternate between the two hulls in flight.
    outs = [out, tuple(torch.empty_like(t) for t in out)]

    def run_steps(k, timed):
        pend = None
        last = None
        for i in range(k):
            if do_flush:
                flush.fill_(i)
            if timed:
                ev[i][0].record(stream)
            if world > 1:
                last, _ = step()
            else:
                p = hull.run_device(x, y, a.mode, stream=sp, out=outs[i & 1], wait=False)
            if timed:
                ev[i][1].record(stream)
            if world == 1:
                if pend is not None:
                    last = pend.result()
                    launches[0] += last.kernel_launches
                pend = p
        if pend is not None:
            last = pend.result()
            launches[0] += last.kernel_launches
        return last

    # --- warm-up (also JIT-free: the library is prebuilt) ---
    clocks = ClockSampler(devi)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    run_steps(a.warmup, False)
    # --- timed region: K steps, per-step CUDA events on the launching stream,
    #     L2 flushed between steps outside the events ---
    barrier()
    clocks.start()
    launches[0] = 0
    final = run_steps(a.steps, True)
    barrier()
    # the final hull of the last timed step, summarised for parity checks (its
    # buffers are reused by the calls below)
    fx = final.x[:final.h].cpu().numpy() if hasattr(final.x, "cpu") else np.asarray(final.x)
    fy = final.y[:final.h].cpu().numpy() if hasattr(final.y, "cpu") else np.asarray(final.y)
    fi = (final.indices[:final.h].cpu().numpy() if hasattr(final.indices, "cpu")
          else np.asarray(final.indices)).astype(np.int64)
    import hashlib
    digest = hashlib.sha256(fx.tobytes() + fy.tobytes() + fi.tobytes()).hexdigest()
    clocks.stop()
    gpu_launches = launches[0]
    t_rank = sum(s.elapsed_time(e) for s, e in ev) / 1e3  # seconds over K steps
    t_max = max_over_ranks(t_rank)
    ms_per_step = t_max / a.steps * 1e3
    value = n_total / (t_max / a.steps) / 1e6

    # --- per-kernel times (library CUDA events on the same stream) for the roofline ---
    ks = []
    for i in range(max(3, min(a.steps, 10))):
        if do_flush:
            flush.fill_(i)
        _, sh = step(timings=True)
        ks.append(sh)
    torch.cuda.synchronize()
    shard = ks[-1]
    hbm, peak_kind = peaks()
    st0 = shard.stats
    m1 = st0[0].points_remaining if st0 else 0
    kept = shard.kept
    n = n_rank
    kern = {
        # name: (algorithmic bytes per launch as designed, mean ms, SURVEY 8d bytes)
        #   K1 reads x, y; K2 reads x, y and writes 2 class bits per point; K3
        #   re-reads x, y + class bits (instead of a survivor set written by K2)
        #   and writes the round-1 live set (24 B per survivor m1, heads excluded)
        "k1_extremes": (16 * n, statistics.mean(k.kernels.extremes_ms for k in ks), 16 * n),
        "k2_filter": (16 * n + n // 4, statistics.mean(k.kernels.filter_ms for k in ks),
                      16 * n + 20 * kept),
        "k3_route_round1": (16 * n + n // 4 + 24 * (m1 - (st0[0].segments if st0 else 0)),
                            statistics.mean(k.kernels.first_round_ms for k in ks),
                            24 * (kept + m1)),
    }
    dom = max(kern, key=lambda k: kern[k][1])
    bytes_dom, ms_dom, survey_dom = kern[dom]
    achieved = bytes_dom / (ms_dom * 1e-3) / 1e9
    traffic, traffic_src = None, None
    try:  # DRAM bytes of the same kernel from one ncu --set full capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        t = tr.get(a.workload, {}).get(dom)
        if t:
            traffic = t["dram_bytes"]
            traffic_src = "profiles/ncu_traffic.json: " + tr.get("_source", "ncu --set full")
    except Exception:
        pass
    per_kernel = {k: {"ms": round(v[1], 5), "alg_bytes": v[0], "survey_bytes": v[2],
                      "GB/s": round(v[0] / (v[1] * 1e-3) / 1e9, 1) if v[1] > 0 else None,
                      "frac_survey": round(v[2] / (v[1] * 1e-3) / 1e9 / hbm, 4)
                      if v[1] > 0 else None}
                  for k, v in kern.items()}
    per_kernel["rounds_ge2"] = {"ms": round(statistics.mean(k.kernels.rounds_ms for k in ks), 5)}
    # whole-pipeline algorithmic bytes: 32n + 20k + sum 24 (m_{r-1} + m_r)
    ms_list = [kept] + [s.points_remaining for s in st0]
    b_alg = 32 * n + 20 * kept + sum(24 * (ms_list[i] + ms_list[i + 1])
                                     for i in range(len(ms_list) - 1))

    # --- e2e: the public API with HOST inputs (H2D + D2H inside the timed region).
    #     Primary: pageable numpy arrays, as the reference's caller passes its
    #     std::vectors; second figure: pinned host buffers. ---
    e2e = None
    if not a.no_e2e:
        hx_pg = x.cpu().numpy().copy()
        hy_pg = y.cpu().numpy().copy()
        hx_pin = torch.empty(n_rank, dtype=torch.float64, pin_memory=True)
        hy_pin = torch.empty(n_rank, dtype=torch.float64, pin_memory=True)
        hx_pin.copy_(x)
        hy_pin.copy_(y)
        torch.cuda.synchronize()
        d2h = [0]

        def e2e_step(hx, hy):
            if world > 1:
                (mx, my, mi), h = merged(hx, hy, out_device=False)
                d2h[0] = 24 * h
                return h
            r = hull.run_arrays(hx, hy, a.mode, device=devi, stream=sp)
            launches[0] += r.kernel_launches
            d2h[0] = 24 * len(r) + 32 * len(r.stats)  # x, y, int64 index; stats rows
            return len(r)

        def e2e_time(hx, hy):
            # the host side (pageable staging by 8 threads) settles after ~10 calls
            for _ in range(max(a.warmup, 10)):
                e2e_step(hx, hy)
            ke = max(3, min(a.steps, 10))
            barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for _ in range(ke):
                e2e_step(hx, hy)
            t1.record(stream)
            barrier()
            return max_over_ranks(t0.elapsed_time(t1) / 1e3) / ke

        te = e2e_time(hx_pg, hy_pg)
        tp = e2e_time(hx_pin, hy_pin)
        e2e = {"value": n_total / te / 1e6, "unit": "Mpoints/s", "ms_per_step": te * 1e3,
               "h2d_bytes_per_step": 16 * n_total,
               "d2h_bytes_per_step": d2h[0] * (world if world > 1 else 1),
               "path": ("hull.run_arrays -> sh_b200_hull_ex(SH_HOST_PTRS), pageable numpy x/y"
                        if world == 1 else
                        "shard.merged_hull(host shard) -> pack (SH_HOST_PTRS|SH_OUT_PAD), "
                        "all-gather, sh_b200_hull_gathered -> host"),
               "pinned": {"value": n_total / tp / 1e6, "ms_per_step": tp * 1e3,
                          "path": "same call, pinned (page-locked) host x/y"}}

    # --- CPU baseline (rank 0, N = 1 only): the reference on the same points ---
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        ns = min(n_rank, 20_000_000)
        hxs = x[:ns].cpu().numpy()
        hys = y[:ns].cpu().numpy()
        once, kindref, cores, desc = cpu_reference_timer(hxs, hys, a.mode)
        once()  # warm-up
        times, t_spent = [], 0.0
        while len(times) < 3 and (t_spent < 20.0 or len(times) < 1):
            dt = once()
            times.append(dt)
            t_spent += dt
        tc = statistics.median(times)
        cpu = {"value": ns / tc / 1e6, "unit": "Mpoints/s", "cores": cores, "kind": kindref,
               "sample": f"{desc} on the same {ns} resident points copied to host, "
                         f"median of {len(times)} runs after 1 warm-up",
               "ms_per_hull": tc * 1e3}


    if rank == 0:
        cl = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "Mpoints/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling,
            "vs_baseline": value / BASELINE_MPTS, "dtype": "f64", "data": "synthetic",
            "config": config_of(a, world),
            "hull": {"h": final.h, "rounds": shard.rounds, "kept_after_filter": shard.kept,
                     "sha256_x_y_idx": digest,
                     "first": [float(fx[0]).hex(), float(fy[0]).hex()] if final.h else None},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                         "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "traffic_source": traffic_src,
                         "alg_bytes": bytes_dom, "ms": round(ms_dom, 5),
                         "survey_bytes": survey_dom,
                         "frac_survey": round(survey_dom / (ms_dom * 1e-3) / 1e9 / hbm, 4),
                         "per_kernel": per_kernel,
                         "pipeline": {"alg_bytes": b_alg,
                                      "floor_ms": round(b_alg / (hbm * 1e9) * 1e3, 4),
                                      "frac": round(b_alg / (hbm * 1e9) /
                                                    (ms_per_step * 1e-3), 4)}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": cl,
        }
        emit(line, a)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_b200(a)


if __name__ == "__main__":
    sys.exit(main())

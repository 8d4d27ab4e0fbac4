#!/usr/bin/env python
"""Benchmark of the evaluate+stamp hot path (BASELINE.json metric:
"MOSFET eval+stamp per sec (1 B200, FP64) and % of FP64/HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--variant V]
    python bench.py --impl reference ...        # the CPU oracle arm

Headline workload: BASELINE configs[4] (clock/bus hub netlist, 8M FETs), the
largest config that fits one GPU -- BASELINE's metric names no config, and
the small configs are bound by launch latency, not by the method.  The same
JSON line carries `per_config`: configs[0..3] measured the same way (plus a
warm-L2 median over >= 1,000 back-to-back calls and a CUDA-graph replay
latency for configs[0] and [1], SURVEY §8(d) timing protocol).

One step = one ees_eval_stamp call over the whole netlist (every §8(a) row:
evaluation + stamping + side reductions), inputs resident in HBM, L2 flushed
before every step (256 MiB write, then read back so L2 holds clean lines), A
and b cleared outside the timed region (the caller's clear).  Timing:
CUDA events on the launching stream around each call, summed over exactly K
steps, barrier + synchronize on both sides, max over ranks.  N>1 runs N
independent replicas ("replicas only"), weak scaling.  Rank 0
prints ONE JSON line.
"""
from __future__ import annotations

import os

# OpenMP placement for the CPU oracle baselines:
# set before any library that links libgomp is loaded, i.e. before torch.
os.environ.setdefault("OMP_PLACES", "cores")
os.environ.setdefault("OMP_PROC_BIND", "close")

import argparse  # noqa: E402
import hashlib  # noqa: E402
import json  # noqa: E402
import math  # noqa: E402
import statistics  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import netgen  # noqa: E402

METRIC = "MOSFET eval+stamp per sec (1 B200, FP64) and % of FP64/HBM roofline"
UNIT = "FET eval+stamp/s"
L2_FLUSH_BYTES = 256 << 20
DEFAULT_CONFIG = 4          # BASELINE.json configs[4] (hub netlist, 8,000,000 FETs): the headline
SMALL_CONFIGS = (0, 1)      # latency-bound: >= 1,000 calls, warm-L2 and CUDA-graph figures too
KERNEL_SOURCES = ("ees_kernels.cu", "ees_host.cpp", "ees_tile.cpp", "ees_internal.h")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# FP64 operations of one evaluation as written in eval_fet1 (ees_kernels.cu;
# SURVEY §8(c) steps 1-8, both region branches evaluated, FMA = 2): the
# source-level count, ~46 in SURVEY §8(d).
FLOPS_PER_EVAL = 47


def algorithmic_bytes(n_dev, n, nnz):
    """SURVEY §8(d) compulsory bytes per call: 48 B device data per FET
    (4 x int32 terminals, f64 beta, 3 x f64 v_prev) + x read once (8 B per
    unknown) + A_vals read-modify-write (16 B per nonzero) + b RMW (16 B per
    unknown).  Slot maps, scratch and sector amplification are overhead.
    Returns (read bytes, write bytes)."""
    reads = 48 * n_dev + 8 * n + 8 * nnz + 8 * n
    writes = 8 * nnz + 8 * n
    return reads, writes


def reduce_max(x, world, device=None):
    """Max over ranks (timing is reported as the slowest rank)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def throughput(n_dev, world, ms_per_step):
    """Whole-job FETs evaluated+stamped per second: every rank runs one
    replica of the workload per step (weak scaling)."""
    return world * n_dev / (ms_per_step * 1e-3)


def source_hash():
    """Hash of the kernel + layout sources: a traffic figure captured by ncu
    on other sources is stale and is not reported as this code's."""
    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        with open(os.path.join(ROOT, "paper_2604_03079_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def load_traffic(cfg, variant):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/traffic.json), only if it was taken on these sources."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if cfg is None or not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    v = d.get(f"cfg{cfg}", {}).get(variant)
    if v is None:
        return None, None
    if isinstance(v, dict):
        src = {"profile": v.get("profile"), "src_hash": v.get("src_hash")}
        if v.get("src_hash") != source_hash():
            src["stale"] = True
            return None, src
        return v.get("bytes"), src
    return None, {"stale": True, "profile": "untagged"}


class ClockSampler:
    """Samples SM clock and throttle reasons while the GPU works: an
    `nvidia-smi -lms` subprocess (no GIL contention with the enqueueing
    thread; B200_PROFILING.md clocks line), timestamps kept, so the samples
    inside the timed region can be told from those of the whole window."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index, period_ms=10):
        self.index, self.period_ms = index, period_ms
        self.proc = None
        self.marks = {}
        self.rows = []

    def start(self):
        import subprocess
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)                  # nvidia-smi start-up: its first samples precede the work
        return self

    def mark(self, name):
        self.marks[name] = time.time()

    def stop(self):
        if self.proc is None:
            return
        time.sleep(2.5 * self.period_ms / 1e3)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        import datetime
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                self.rows.append((ts, float(f[1]), float(f[2]), f[4:8]))
            except Exception:
                continue

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": "nvidia-smi unavailable"}
        t0, t1 = self.marks.get("timed_start"), self.marks.get("timed_end")
        w0, w1 = self.marks.get("window_start", 0), self.marks.get("window_end", 1e18)
        timed = [r for r in self.rows if t0 is not None and t0 <= r[0] <= t1]
        window = [r for r in self.rows if w0 <= r[0] <= w1] or self.rows
        use = timed if len(timed) >= 3 else window
        reasons = sorted({n for r in use for n, a in zip(self.NAMES, r[3]) if a.lower() == "active"})
        return {"sm_mhz": statistics.median(r[1] for r in use), "sm_max_mhz": max(r[2] for r in use),
                "reasons": reasons, "samples": len(use), "samples_timed_region": len(timed),
                "sm_mhz_min": min(r[1] for r in use),
                "source": (f"nvidia-smi -lms {self.period_ms}: " +
                           ("samples inside the timed region" if use is timed else
                            "samples from warm-up through the roofline pass (timed region too short "
                            "for 3 samples)"))}


# ---------------------------------------------------------------- CPU side
def host_cores():
    """Cores this process may actually use: the affinity mask, capped by a
    cgroup CPU quota (v2 cpu.max or v1 cfs_quota/period) -- os.cpu_count()
    reports the machine, not the lease."""
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count() or 1
    quota = None
    try:
        q, per = open("/sys/fs/cgroup/cpu.max").read().split()[:2]
        if q != "max":
            quota = float(q) / float(per)
    except Exception:
        try:
            q = int(open("/sys/fs/cgroup/cpu/cpu.cfs_quota_us").read())
            per = int(open("/sys/fs/cgroup/cpu/cpu.cfs_period_us").read())
            if q > 0:
                quota = q / per
        except Exception:
            pass
    cores = aff if quota is None else max(1, min(aff, int(math.ceil(quota))))
    return cores, {"affinity": aff, "cgroup_quota_cpus": quota, "os_cpu_count": os.cpu_count()}


# The granted cores, read before any OpenMP runtime starts: with OMP_PROC_BIND
# set, libgomp pins the main thread to its first place when it initialises
# (torch loads it), after which the thread's affinity mask shows one core.
_HOST_CORES = host_cores()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def lscpu_summary():
    import subprocess
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
    except Exception:
        return None
    keep = ("Model name", "CPU(s)", "Thread(s) per core", "Core(s) per socket", "Socket(s)",
            "NUMA node(s)", "On-line CPU(s) list")
    d = {}
    for line in out.splitlines():
        k, _, v = line.partition(":")
        if k.strip() in keep:
            d[k.strip()] = v.strip()
    return d


def time_oracle(bl, kind, threads, reps, A, b):
    """Median of `reps` calls after one discarded warm-up; A and b are
    cleared outside each timed call."""
    A[:] = 0
    b[:] = 0
    bl.run(kind, A, b, threads)
    ts = []
    for _ in range(reps):
        A[:] = 0
        b[:] = 0
        t0 = time.perf_counter()
        bl.run(kind, A, b, threads)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), ts


def cpu_baseline(nl, reps=5):
    """The oracle's Table I kernels as they stand, on this host's
    granted cores: loadsingle (1 thread), ColorFused at 1 and T threads,
    loadomp at T threads; each the median of `reps` calls.  `value` is
    the fastest multi-threaded kernel; the thread scaling is reported, and
    flagged when T threads give less than 2x of one."""
    import oracle
    cores, cinfo = _HOST_CORES
    t_build = time.perf_counter()
    bl = oracle.Baseline(nl)
    t_build = time.perf_counter() - t_build
    A = np.zeros(bl.nnz)
    b = np.zeros(nl.n)
    runs = {}
    t_all = time.perf_counter()
    for name, kind, th in (("loadsingle_1t", "loadsingle", 1), ("colorfused_1t", "colorfused", 1),
                           (f"colorfused_{cores}t", "colorfused", cores), (f"loadomp_{cores}t", "loadomp", cores)):
        med, ts = time_oracle(bl, kind, th, reps, A, b)
        runs[name] = {"kernel": kind, "threads": th, "median_s": med, "value": nl.n_dev / med, "calls": len(ts)}
    t_all = time.perf_counter() - t_all
    bl.close()
    best = max((r for r in runs.values() if r["threads"] == cores), key=lambda r: r["value"])
    cf1 = runs["colorfused_1t"]["value"]
    cft = runs[f"colorfused_{cores}t"]["value"]
    ls = runs["loadsingle_1t"]["value"]
    scaling = {"colorfused_T_over_1t": cft / cf1, "best_T_over_loadsingle": best["value"] / ls,
               "flag_poor_scaling": cft / cf1 < 2.0 and cores >= 4}
    return {"value": best["value"], "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": (f"{nl.name}: the whole netlist ({nl.n_dev} FETs) per call; median of {reps} calls "
                       f"per kernel after one warm-up; {t_all:.1f} s of CPU runs (+{t_build:.1f} s plan setup)"),
            "best_kernel": f"{best['kernel']} x {best['threads']} threads", "runs": runs,
            "thread_scaling": scaling, "cores_info": cinfo,
            "omp": {k: os.environ.get(k) for k in ("OMP_PLACES", "OMP_PROC_BIND", "OMP_WAIT_POLICY")},
            "cpu_model": cpu_model(), "lscpu": lscpu_summary(),
            "context": "paper: up to 45x over single-thread on a 64-core workstation (P:21, P:160)"}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (the faster of the
    paper's multi-threaded kernels, ColorFused or loadomp, on the granted host
    cores) on the same config, metric and unit; rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    nl = netgen.config(args.config)
    import oracle
    cores, cinfo = _HOST_CORES
    bl = oracle.Baseline(nl)
    A = np.zeros(bl.nnz)
    b = np.zeros(nl.n)
    probe = {k: time_oracle(bl, k, cores, 1, A, b)[0] for k in ("colorfused", "loadomp")}
    kind = min(probe, key=probe.get)
    for _ in range(max(0, args.warmup - 1)):
        bl.run(kind, A, b, cores)
    el = 0.0
    for _ in range(args.steps):
        A[:] = 0
        b[:] = 0
        t0 = time.perf_counter()
        bl.run(kind, A, b, cores)
        el += time.perf_counter() - t0
    bl.close()
    value = nl.n_dev * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": netgen.CONFIG_NAMES[args.config], "n_dev": nl.n_dev,
                       "device": "host CPU (the oracle; no GPU work)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} full {kind} calls of {nl.name} on {cores} threads "
                                       f"(A, b cleared outside the timed calls)",
                             "kernel": kind, "probe_s": probe, "cores_info": cinfo,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side
class L2Flush:
    """Evicts L2 before a step: writes a 256 MiB buffer (> the 126 MB L2),
    then (mode "clean", the default) reads it back, so the lines left in L2
    are clean and the timed kernel does not pay for writing back the flush's
    own dirty data.  Mode "write" is the write alone."""

    def __init__(self, dev, mode="clean"):
        import torch
        self.buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
        self.mode = mode
        self.sink = torch.empty(1, dtype=torch.float32, device=dev)

    def __call__(self, k):
        import torch
        self.buf.fill_(float(k & 0xFF))
        if self.mode == "clean":
            torch.sum(self.buf, dim=0, keepdim=True, out=self.sink)

    def describe(self):
        return ("flushed before every step: 256 MiB write" +
                (" then read back (L2 left clean)" if self.mode == "clean" else ""))


def time_calls(ctx, nl, x, A, b, stream, steps, warmup, flush):
    """Per-call device ms (CUDA events on `stream`), L2 flushed before each
    (flush=None: back to back, warm L2)."""
    import torch
    with torch.cuda.stream(stream):
        for k in range(warmup):
            if flush:
                flush(k)
            A.zero_()
            b.zero_()
            ctx.eval_stamp(x, nl.h, A, b, stream=stream)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        torch.cuda.synchronize()
        for k in range(steps):
            if flush:
                flush(k)
                A.zero_()
                b.zero_()
            evs[k][0].record(stream)
            ctx.eval_stamp(x, nl.h, A, b, stream=stream)
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    return [e0.elapsed_time(e1) for e0, e1 in evs]


def graph_latency(ctx, nl, x, A, b, stream, reps):
    """One ees_eval_stamp captured in a CUDA graph, replayed `reps` times back
    to back (warm L2): device ms per call without host enqueue cost."""
    import torch
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        ctx.eval_stamp(x, nl.h, A, b, stream=stream)
    with torch.cuda.stream(stream):
        for _ in range(10):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del g
    return ms


def stream_reference(read_bytes, write_bytes, dev, stream, pre, steps, achieved_gbs):
    """Size calibration of the HBM roofline: ees_stream_probe, ONE library
    kernel that reads and writes the call's algorithmic bytes (same read /
    write mix), timed the same way as the call (same flush before each step,
    CUDA events on the same stream).  `frac` is the call's achieved bandwidth
    over the probe's."""
    import torch
    from paper_2604_03079_b200 import stream_probe
    src = torch.ones(max(2, int(read_bytes) // 8 + 2), dtype=torch.float64, device=dev)
    dst = torch.zeros(max(2, int(write_bytes) // 8 + 2), dtype=torch.float64, device=dev)
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for k in range(3):
            pre(k)
            stream_probe(src, read_bytes, dst, write_bytes, sink, stream)
        for k in range(steps):
            pre(k)
            evs[k][0].record(stream)
            stream_probe(src, read_bytes, dst, write_bytes, sink, stream)
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in evs)
    gbs = (read_bytes + write_bytes) / (ms * 1e-3) / 1e9
    del src, dst
    return {"kernel": "ees_stream_probe (one launch, 16 B vectors, same read/write mix), flushed",
            "read_bytes": int(read_bytes), "write_bytes": int(write_bytes), "ms": ms, "gbs": gbs,
            "frac": achieved_gbs / gbs}


PHASES = {"atomic": ["k_atomic"],
          "color": ["k_color x C", "k_rail_final"],
          "color_hybrid": ["k_color_h x C", "k_side_chunks + k_side_apply"],
          "gather": ["k_gather_eval", "k_gather_reduce", "k_gather_heavy"],
          "tile": ["k_tile"],
          "color_buf": ["k_gather_eval (t_calc)", "k_color_stamp x C + side sum (t_stamp)"]}


def measure(ctx, nl, cfg, args, dev, stream, flush, world, steps, warmup, small=False, clk=None):
    """Times one context the headline way and returns its record: per-call
    event times (flushed), the dominant kernel group's roofline from the
    library's per-phase events over a second pass, and for the small configs
    the warm-L2 median of >= 1,000 calls and the CUDA-graph latency."""
    import torch
    import torch.distributed as dist
    x = torch.from_numpy(nl.x).to(dev)
    A = torch.zeros(ctx.nnz, dtype=torch.float64, device=dev)
    b = torch.zeros(ctx.n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def step_pre(k):
        with torch.cuda.stream(stream):
            flush(k)                       # evict A, b, x, device data from L2
            A.zero_()
            b.zero_()

    if clk is not None:
        clk.mark("window_start")
    with torch.cuda.stream(stream):
        for k in range(warmup):
            step_pre(k)
            ctx.eval_stamp(x, nl.h, A, b, stream=stream)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clk is not None:
        clk.mark("timed_start")
    with torch.cuda.stream(stream):
        for k in range(steps):
            step_pre(k)
            evs[k][0].record(stream)
            ctx.eval_stamp(x, nl.h, A, b, stream=stream)
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    if clk is not None:
        clk.mark("timed_end")
    if world > 1:
        dist.barrier()
    per = [e0.elapsed_time(e1) for e0, e1 in evs]
    # second pass, same steps and flushes: the library's per-phase CUDA events
    # (on the launching stream) time each kernel group for the roofline
    ctx.phase_times()
    ctx.set_timing(True)
    with torch.cuda.stream(stream):
        for k in range(steps):
            step_pre(k)
            ctx.eval_stamp(x, nl.h, A, b, stream=stream)
    torch.cuda.synchronize()
    phase_ms, n_timed = ctx.phase_times()
    ctx.set_timing(False)
    if clk is not None:
        clk.mark("window_end")
    st = ctx.stats()
    variant = st["variant_chosen"]
    hbm, peak_src = peaks()
    rd, wr = algorithmic_bytes(nl.n_dev, ctx.n, ctx.nnz)
    alg = rd + wr
    key = "color_hybrid" if (variant == "color" and args.rule == "hybrid") else variant
    names = PHASES[key]
    phase_avg = {name: phase_ms[i] / max(1, n_timed) for i, name in enumerate(names)}
    kern_ms = sum(phase_avg.values())
    achieved = alg / (kern_ms * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(cfg, variant) if args.rule == "exclude_rails" else (None, None)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
            "kernel": " + ".join(names), "kernel_ms": kern_ms, "phase_ms": phase_avg,
            "algorithmic_bytes_per_launch": alg, "peak_source": peak_src,
            "per_unit": "48 B/FET + 8 B/unknown (x) + 16 B/nonzero (A RMW) + 16 B/unknown (b RMW)"}
    roof["stream_ref"] = stream_reference(rd, wr, dev, stream, step_pre, min(steps, 30), achieved)
    if args.work > 1:
        # S:229 work multiplier: evaluation arithmetic x k puts the path on the
        # FP64 pipe; peak = this device's FMA throughput measured now
        from paper_2604_03079_b200 import fp64_peak
        fpk = fp64_peak()
        flops = FLOPS_PER_EVAL * args.work * nl.n_dev
        ach = flops / (kern_ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": ach, "peak": fpk, "unit": "TFLOP/s", "frac": ach / fpk,
                "traffic": None, "kernel": roof["kernel"], "kernel_ms": kern_ms, "phase_ms": phase_avg,
                "algorithmic_flops_per_launch": flops,
                "peak_source": "measured now (ees_fp64_peak: independent DFMA chains, one wave)",
                "per_unit": f"{FLOPS_PER_EVAL} FP64 flops per evaluation x work {args.work}",
                "hbm_frac": achieved / hbm}
    ps = sorted(per)
    rec = {"per": per, "variant": variant, "colors": st["n_colors"], "n": ctx.n, "nnz": ctx.nnz,
           "tune_ms": st["tune_ms"], "setup_s": st["setup_s"], "launches_per_call": st["launches_per_call"],
           "p10_ms": ps[len(ps) // 10], "p50_ms": ps[len(ps) // 2], "p90_ms": ps[(9 * len(ps)) // 10],
           "roofline": roof, "x": x, "A": A, "b": b}
    if small:
        warm = time_calls(ctx, nl, x, A, b, stream, args.small_calls, 10, None)
        ws = sorted(warm)
        rec["warm_l2"] = {"calls": len(warm), "p10_ms": ws[len(ws) // 10], "p50_ms": ws[len(ws) // 2],
                          "p90_ms": ws[(9 * len(ws)) // 10],
                          "what": "back-to-back calls, no flush (L2 warm), CUDA events per call"}
        rec["graph_ms_per_call"] = graph_latency(ctx, nl, x, A, b, stream, args.small_calls)
    return rec


def per_config_records(Context, args, dev, stream, flush, world):
    out = {}
    for c in args.per_config:
        if c == args.config:
            continue
        nl = netgen.config(c)
        ctx = Context.from_netlist(nl, variant=args.variant)
        small = c in SMALL_CONFIGS
        steps = max(args.small_calls, args.steps) if small else max(20, min(args.steps, 50))
        r = measure(ctx, nl, c, args, dev, stream, flush, world, steps, 5, small=small)
        ms = reduce_max(sum(r["per"]), world, dev) / steps
        rec = {"workload": netgen.CONFIG_NAMES[c], "n_dev": nl.n_dev, "n": r["n"], "nnz": r["nnz"],
               "colors": r["colors"], "variant": r["variant"], "steps": steps,
               "value": throughput(nl.n_dev, world, ms), "ms_per_step": ms,
               "p10_ms": r["p10_ms"], "p50_ms": r["p50_ms"], "p90_ms": r["p90_ms"],
               "roofline": {k: r["roofline"][k] for k in ("frac", "achieved", "kernel", "kernel_ms",
                                                          "traffic", "traffic_source")},
               "stream_ref_frac": r["roofline"]["stream_ref"]["frac"],
               "tune_ms": r["tune_ms"], "setup_s": r["setup_s"]}
        for k in ("warm_l2", "graph_ms_per_call"):
            if k in r:
                rec[k] = r[k]
        out[f"cfg{c}"] = rec
        ctx.close()
        del r
    return out


def run_sweep(args):
    """B5: gen_synth N FETs as N/C cliques, C = 1..4096; every
    variant timed per C -> the stamping-variant crossover against the colour
    count (the GPU analogue of the paper's Fig. 5(c-d))."""
    import torch
    from paper_2604_03079_b200 import Context
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    flush = L2Flush(dev, args.flush)
    out = open(args.sweep_out, "w") if args.sweep_out else None
    for C in [int(c) for c in args.sweep_c.split(",")]:
        nl = netgen.gen_synth(args.sweep_n, C)
        ctx = Context.from_netlist(nl, variant="auto")
        st = ctx.stats()
        x = torch.from_numpy(nl.x).to(dev)
        A = torch.zeros(ctx.nnz, dtype=torch.float64, device=dev)
        b = torch.zeros(ctx.n, dtype=torch.float64, device=dev)
        rec = {"C": st["n_colors"], "n_dev": nl.n_dev, "nnz": ctx.nnz, "auto": st["variant_chosen"],
               "ms": {}}
        for v in ("color", "atomic", "gather", "tile", "color_buf"):
            ctx.set_variant(v)
            steps = args.steps if (v not in ("color", "color_buf") or C <= 512) else max(3, args.steps // 10)
            per = sorted(time_calls(ctx, nl, x, A, b, stream, steps, 3, flush))
            rec["ms"][v] = per[len(per) // 2]
        # NEXT-1: COLOR under the degree-threshold hybrid rule (hub nodes leave
        # the conflict relation; their entries take the side sum)
        ctx_h = Context.from_netlist(nl, variant="color", rule="hybrid", heavy_degree=args.heavy_degree)
        rec["C_hybrid"] = ctx_h.stats()["n_colors"]
        per = sorted(time_calls(ctx_h, nl, x, A, b, stream, args.steps, 3, flush))
        rec["ms"]["color_hybrid"] = per[len(per) // 2]
        ctx_h.close()
        rec["fet_per_s"] = {v: nl.n_dev / (ms * 1e-3) for v, ms in rec["ms"].items()}
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()
        ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--netlist", default=None,
                    help="another workload by name instead of --config (netgen.named: adder64, "
                         "adder64_r14, adder64_r89, cfgN@scale)")
    ap.add_argument("--variant", default="auto", choices=["auto", "color", "atomic", "gather", "tile", "color_buf"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rule", default="exclude_rails", choices=["exclude_rails", "paper", "hybrid"],
                    help="conflict relation of the colouring (COLOR variant)")
    ap.add_argument("--heavy-degree", type=int, default=64, help="hybrid rule threshold")
    ap.add_argument("--work", type=int, default=1, help="S:229 work multiplier (FP64-bound probe)")
    ap.add_argument("--flush", default="clean", choices=["clean", "write"],
                    help="L2 flush before each step: write 256 MiB (+ read it back: clean)")
    ap.add_argument("--tile-form", type=int, default=None, choices=[0, 1],
                    help="force the TILE layout form (A/B experiments; default: chosen at setup)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--per-config", default="0,1,2,3",
                    help="configs measured into the line's per_config record ('' = none)")
    ap.add_argument("--small-calls", type=int, default=1000,
                    help="calls for the small configs' flushed, warm-L2 and CUDA-graph figures")
    ap.add_argument("--sweep", action="store_true", help="B5 colour-count crossover sweep")
    ap.add_argument("--sweep-n", type=int, default=4_000_000)
    ap.add_argument("--sweep-c", default="1,2,4,8,16,32,64,128,256,512,1024,2048,4096")
    ap.add_argument("--sweep-out", default=None)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.per_config = [int(c) for c in args.per_config.replace("none", "").split(",") if c.strip() not in ("", "''")]
    if args.netlist or args.rule != "exclude_rails" or args.work > 1:
        args.per_config = []
    if args.impl == "reference":
        return run_reference(args)
    if args.sweep:
        return run_sweep(args)

    import torch
    import torch.distributed as dist
    from paper_2604_03079_b200 import Context

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream()
    flush = L2Flush(dev, args.flush)

    nl = netgen.named(args.netlist) if args.netlist else netgen.config(args.config)
    cfg = None if args.netlist else args.config
    ctx = Context.from_netlist(nl, variant=args.variant, rule=args.rule, heavy_degree=args.heavy_degree,
                               tile_form=args.tile_form)
    if args.work > 1:
        ctx.set_work(args.work)
    clk = ClockSampler(torch.cuda.current_device()).start()
    try:
        r = measure(ctx, nl, cfg, args, dev, stream, flush, world, args.steps, args.warmup,
                    small=cfg in SMALL_CONFIGS, clk=clk)
    finally:
        clk.stop()
    per = r["per"]
    max_ms = reduce_max(sum(per), world, dev)
    ms_per_step = max_ms / args.steps
    value = throughput(nl.n_dev, world, ms_per_step)

    # end to end through the host-buffer ABI call (pinned buffers): H2D x,
    # evaluate+stamp, D2H A and b, every step
    e2e = None
    if not args.no_e2e:
        hx = torch.from_numpy(nl.x).pin_memory()
        hA = torch.zeros(ctx.nnz, dtype=torch.float64).pin_memory()
        hb = torch.zeros(ctx.n, dtype=torch.float64).pin_memory()
        for _ in range(3):
            ctx.eval_stamp_host(hx, nl.h, hA, hb, stream=stream, assign=True)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            ev[k][0].record(stream)
            ctx.eval_stamp_host(hx, nl.h, hA, hb, stream=stream, assign=True)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        e_ms = reduce_max(sum(a.elapsed_time(bq) for a, bq in ev), world, dev) / args.steps
        e2e = {"value": throughput(nl.n_dev, world, e_ms), "unit": UNIT,
               "h2d_bytes_per_step": 8 * ctx.n,
               "d2h_bytes_per_step": 8 * (ctx.n + ctx.nnz), "ms_per_step": e_ms,
               "api": "ees_eval_stamp_host(..., EES_HOST_ASSIGN): pinned host x in, A and b out",
               "pcie_gbs": 8 * (2 * ctx.n + ctx.nnz) / (e_ms * 1e-3) / 1e9}
        del hx, hA, hb
    launches = r["launches_per_call"]
    for k in ("x", "A", "b"):
        r.pop(k)
    ctx.close()

    per_config = per_config_records(Context, args, dev, stream, flush, world) if args.per_config else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(nl, args.cpu_reps)

    if rank == 0:
        config = {"workload": (f"{nl.name} ({nl.n_dev} FETs)" if args.netlist
                               else netgen.CONFIG_NAMES[args.config]),
                  "config_index": cfg, "n_dev": nl.n_dev, "n": r["n"], "nnz": r["nnz"],
                  "colors": r["colors"], "variant": r["variant"], "tune_ms": r["tune_ms"],
                  "rule": args.rule, "work": args.work, "l2": flush.describe(),
                  "parallelism": "replicas" if world > 1 else "single",
                  "p10_ms": r["p10_ms"], "p50_ms": r["p50_ms"], "p90_ms": r["p90_ms"],
                  "setup_s": r["setup_s"]}
        for k in ("warm_l2", "graph_ms_per_call"):
            if k in r:
                config[k] = r[k]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config,
            "roofline": r["roofline"],
            "per_config": per_config,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

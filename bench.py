#!/usr/bin/env python
"""Benchmark of the evaluate+stamp hot path (BASELINE.json metric:
"MOSFET eval+stamp per sec (1 B200, FP64) and % of FP64/HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--variant V]
    python bench.py --impl reference ...        # the CPU oracle arm

One step = one ees_eval_stamp call over the whole netlist (every §8(a) row:
evaluation + stamping + rail side-reduction), inputs resident in HBM, L2
flushed before every step (256 MiB write, then read back so L2 holds clean
lines), A and b cleared outside the timed
region (the caller's clear).  Timing: CUDA events on the launching
stream around each call, summed over exactly K steps, barrier + synchronize
on both sides, max over ranks.  N>1 runs N independent replicas (DESIGN.md
§6: "replicas only"), weak scaling.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import netgen  # noqa: E402

METRIC = "MOSFET eval+stamp per sec (1 B200, FP64) and % of FP64/HBM roofline"
UNIT = "FET eval+stamp/s"
L2_FLUSH_BYTES = 256 << 20
DEFAULT_CONFIG = 1          # BASELINE.json configs[1] (ring oscillators, 202,000 FETs)


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
    unknown).  Slot maps, scratch and sector amplification are overhead."""
    return 48 * n_dev + 8 * n + 16 * nnz + 16 * n


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


def load_traffic(cfg, variant):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = d.get(f"cfg{cfg}", {}).get(variant)
    return v


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while running."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index, period=0.001):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_baseline(nl, budget_s=10.0):
    """The oracle's Table I kernels as they stand, on this host's
    cores: ColorFused and loadomp with all cores, loadsingle with 1 thread.
    Bounded sample: repeat full calls on the same netlist until budget_s."""
    import oracle
    cores = os.cpu_count() or 1
    bl = oracle.Baseline(nl)
    nnz = bl.nnz
    A = np.zeros(nnz)
    b = np.zeros(nl.n)
    out = {}
    for kind, threads, budget in (("colorfused", cores, budget_s), ("loadomp", cores, budget_s / 3),
                                  ("loadsingle", 1, budget_s / 3)):
        bl.run(kind, A, b, threads)      # warm-up
        reps, t0 = 0, time.perf_counter()
        while True:
            bl.run(kind, A, b, threads)
            reps += 1
            el = time.perf_counter() - t0
            if el >= budget:
                break
        out[kind] = dict(value=nl.n_dev * reps / el, threads=threads, calls=reps, seconds=el)
    bl.close()
    best = out["colorfused"]
    return {"value": best["value"], "unit": UNIT, "cores": best["threads"], "kind": "oracle",
            "sample": f"{nl.name}: {best['calls']} full ColorFused calls ({nl.n_dev} FETs each) "
                      f"in {best['seconds']:.1f} s on {best['threads']} threads",
            "loadsingle_1t": out["loadsingle"]["value"], "loadomp": out["loadomp"]["value"],
            "colorfused": out["colorfused"]["value"], "cpu_model": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    """--impl reference: the CPU oracle (ColorFused, all host cores) on the same
    config, metric and unit; rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    nl = netgen.config(args.config)
    import oracle
    cores = os.cpu_count() or 1
    bl = oracle.Baseline(nl)
    A = np.zeros(bl.nnz)
    b = np.zeros(nl.n)
    for _ in range(args.warmup):
        bl.run("colorfused", A, b, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        A[:] = 0
        b[:] = 0
        bl.run("colorfused", A, b, cores)
    el = time.perf_counter() - t0
    bl.close()
    value = nl.n_dev * args.steps / el
    # n_gpus: the launch's N (the oracle itself runs on rank 0's host cores only)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": netgen.CONFIG_NAMES[args.config], "n_dev": nl.n_dev,
                       "device": "host CPU (the oracle; no GPU work)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} full ColorFused calls of {nl.name}",
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
    """Per-call device ms (CUDA events on `stream`), L2 flushed before each."""
    import torch
    for k in range(warmup):
        with torch.cuda.stream(stream):
            flush(k)
            A.zero_(); b.zero_()
        ctx.eval_stamp(x, nl.h, A, b, stream=stream)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush(k)
            A.zero_(); b.zero_()
        evs[k][0].record(stream)
        ctx.eval_stamp(x, nl.h, A, b, stream=stream)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    return sorted(e0.elapsed_time(e1) for e0, e1 in evs)


def stream_reference(nbytes, dev, stream, pre, steps, achieved_gbs):
    """Size calibration of the HBM roofline: a plain streaming read (torch.sum
    over an FP64 tensor of the call's algorithmic bytes) timed the same way as
    the call (same flush before each step, CUDA events on the same stream).
    At small byte counts the flushed-L2 ramp, not the copy peak, bounds any
    kernel (profiles/r01_l_ab.md); `frac` is the call's achieved bandwidth
    over this one's."""
    import torch
    src = torch.ones(max(1, int(nbytes) // 8), dtype=torch.float64, device=dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for k in range(3):
            pre(k)
            torch.sum(src, 0, out=out[0])
        for k in range(steps):
            pre(k)
            evs[k][0].record(stream)
            torch.sum(src, 0, out=out[0])
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)[steps // 2]
    gbs = nbytes / (ms * 1e-3) / 1e9
    del src
    return {"kernel": "torch.sum over the algorithmic bytes (read-only stream), flushed",
            "bytes": int(nbytes), "ms": ms, "gbs": gbs, "frac": achieved_gbs / gbs}


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
            per = time_calls(ctx, nl, x, A, b, stream, steps, 3, flush)
            rec["ms"][v] = per[len(per) // 2]
        # NEXT-1: COLOR under the degree-threshold hybrid rule (hub nodes leave
        # the conflict relation; their entries take the side sum)
        ctx_h = Context.from_netlist(nl, variant="color", rule="hybrid", heavy_degree=args.heavy_degree)
        rec["C_hybrid"] = ctx_h.stats()["n_colors"]
        per = time_calls(ctx_h, nl, x, A, b, stream, args.steps, 3, flush)
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="B5 colour-count crossover sweep")
    ap.add_argument("--sweep-n", type=int, default=4_000_000)
    ap.add_argument("--sweep-c", default="1,2,4,8,16,32,64,128,256,512,1024,2048,4096")
    ap.add_argument("--sweep-out", default=None)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
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

    nl = netgen.named(args.netlist) if args.netlist else netgen.config(args.config)
    ctx = Context.from_netlist(nl, variant=args.variant, rule=args.rule, heavy_degree=args.heavy_degree)
    if args.work > 1:
        ctx.set_work(args.work)
    st = ctx.stats()
    stream = torch.cuda.Stream()
    x = torch.from_numpy(nl.x).to(dev)
    A = torch.zeros(ctx.nnz, dtype=torch.float64, device=dev)
    b = torch.zeros(ctx.n, dtype=torch.float64, device=dev)
    flush = L2Flush(dev, args.flush)
    torch.cuda.synchronize()

    def step_pre(k):
        with torch.cuda.stream(stream):
            flush(k)                       # evict A, b, x, device data from L2
            A.zero_()
            b.zero_()

    with torch.cuda.stream(stream):
        for k in range(args.warmup):
            step_pre(k)
            ctx.eval_stamp(x, nl.h, A, b, stream=stream)
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                step_pre(k)
                evs[k][0].record(stream)
                ctx.eval_stamp(x, nl.h, A, b, stream=stream)
                evs[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per = [e0.elapsed_time(e1) for e0, e1 in evs]
    # second pass, same K steps and flushes: the library's per-phase CUDA events
    # (on the launching stream) time each kernel group for the roofline
    ctx.phase_times()
    ctx.set_timing(True)
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            step_pre(k)
            ctx.eval_stamp(x, nl.h, A, b, stream=stream)
    torch.cuda.synchronize()
    phase_ms, n_timed = ctx.phase_times()
    ctx.set_timing(False)
    total_ms = sum(per)
    max_ms = reduce_max(total_ms, world, dev)
    ms_per_step = max_ms / args.steps
    value = throughput(nl.n_dev, world, ms_per_step)
    st = ctx.stats()
    variant = st["variant_chosen"]

    # roofline of the dominant kernel group, timed by the library's per-phase
    # CUDA events on the launching stream over the timed region
    hbm, peak_src = peaks()
    alg = algorithmic_bytes(nl.n_dev, ctx.n, ctx.nnz)
    phases = {"atomic": ["k_atomic"],
              "color": (["k_color_h x C", "k_side_chunks + k_side_apply"] if args.rule == "hybrid"
                        else ["k_color x C", "k_rail_final"]),
              "gather": ["k_gather_eval", "k_gather_reduce", "k_gather_heavy"],
              "tile": ["k_tile"],
              "color_buf": ["k_gather_eval (t_calc)", "k_color_stamp x C + side sum (t_stamp)"]}[variant]
    phase_avg = {name: phase_ms[i] / max(1, n_timed) for i, name in enumerate(phases)}
    kern_ms = sum(phase_avg.values())
    achieved = alg / (kern_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None if args.netlist else load_traffic(args.config, variant),
            "kernel": " + ".join(phases), "kernel_ms": kern_ms, "phase_ms": phase_avg,
            "algorithmic_bytes_per_launch": alg, "peak_source": peak_src,
            "per_unit": "48 B/FET + 8 B/unknown (x) + 16 B/nonzero (A RMW) + 16 B/unknown (b RMW)"}
    roof["stream_ref"] = stream_reference(alg, dev, stream, step_pre, min(args.steps, 30), achieved)
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

    # end to end through the host-buffer ABI call (pinned buffers)
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
               "api": "ees_eval_stamp_host(..., EES_HOST_ASSIGN): pinned host x in, A and b out"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(nl, args.cpu_budget)

    if rank == 0:
        per_sorted = sorted(per)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": (f"{nl.name} ({nl.n_dev} FETs)" if args.netlist
                                    else netgen.CONFIG_NAMES[args.config]),
                       "config_index": None if args.netlist else args.config,
                       "n_dev": nl.n_dev, "n": ctx.n, "nnz": ctx.nnz, "colors": st["n_colors"],
                       "variant": variant, "tune_ms": st["tune_ms"], "rule": args.rule,
                       "work": args.work,
                       "l2": flush.describe(),
                       "parallelism": "replicas" if world > 1 else "single",
                       "p10_ms": per_sorted[len(per) // 10], "p50_ms": per_sorted[len(per) // 2],
                       "p90_ms": per_sorted[(9 * len(per)) // 10], "setup_s": st["setup_s"]},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": st["launches_per_call"] * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Timing floor of bench.py's methodology (debug): event time of a trivial
kernel after the same L2 flush, vs the library's smallest call (cfg0, a
1-FET netlist), flushed and warm."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import netgen  # noqa: E402
from paper_2604_03079_b200 import Context  # noqa: E402


def timed(fn, pre, steps=50):
    st = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(5):
        pre(k); fn()
    torch.cuda.synchronize()
    for k in range(steps):
        pre(k)
        evs[k][0].record(st); fn(); evs[k][1].record(st)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
    return t[len(t) // 2]


def main():
    dev = torch.device("cuda", 0)
    fl = bench.L2Flush(dev, "clean")
    one = torch.zeros(1, device=dev)
    print("trivial torch kernel, flushed: %.2f us" % timed(lambda: one.add_(1.0), fl))
    print("trivial torch kernel, warm:    %.2f us" % timed(lambda: one.add_(1.0), lambda k: None))
    # streaming calibration: what a plain torch kernel achieves on cfg1's
    # compulsory bytes (20.2 MB) after the same flush
    for mb in (4, 20.2, 80, 400):
        src = torch.ones(int(mb * 1e6 / 8), dtype=torch.float64, device=dev)
        out = torch.zeros(1, dtype=torch.float64, device=dev)
        t = timed(lambda: torch.sum(src, 0, out=out[0]), fl)
        print("stream read %6.1f MB (torch sum), flushed: %8.2f us = %7.1f GB/s" % (mb, t, mb * 1e3 / t))
        dst = torch.empty_like(src)
        t = timed(lambda: dst.copy_(src), fl)
        print("stream copy %6.1f MB (read+write), flushed: %8.2f us = %7.1f GB/s" % (mb, t, 2 * mb * 1e3 / t))
        del src, dst
    for name, nl in (("1 FET", netgen.custom("one", 3, [(0, 1, 2, -1)], 0, netgen.bench_models())),
                     ("cfg0", netgen.config(0)), ("cfg1", netgen.config(1))):
        ctx = Context.from_netlist(nl)
        x = torch.from_numpy(nl.x).to(dev)
        A = torch.zeros(ctx.nnz, dtype=torch.float64, device=dev)
        b = torch.zeros(ctx.n, dtype=torch.float64, device=dev)
        for v in ("atomic", "tile"):
            ctx.set_variant(v)
            f = lambda: ctx.eval_stamp(x, nl.h, A, b)
            print("%-6s %-6s flushed %.2f us   warm %.2f us" % (name, v, timed(f, fl), timed(f, lambda k: None)))
        ctx.close()


if __name__ == "__main__":
    main()

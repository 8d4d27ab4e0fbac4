#!/usr/bin/env python
"""Per-CTA timeline of one EES_TILE call (debug): python tools/tile_trace.py [config]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import netgen  # noqa: E402
from paper_2604_03079_b200 import Context  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    nl = netgen.config(cfg)
    ctx = Context.from_netlist(nl, variant="tile")
    x = torch.from_numpy(nl.x).cuda()
    A = torch.zeros(ctx.nnz, dtype=torch.float64, device="cuda")
    b = torch.zeros(ctx.n, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for k in range(3):
        ctx.eval_stamp(x, nl.h, A, b)
    torch.cuda.synchronize()
    flush.fill_(1)
    torch.cuda.synchronize()
    tr = ctx.tile_trace(x, nl.h, A, b).astype(np.int64)
    st = ctx.stats()
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = np.where(tr > 0, tr - t0, -1)
    print(f"cfg{cfg}: tiles={st['n_tiles']} ctas={tr.shape[0]} span={(tr.max() - t0) / 1e3:.2f} us")
    def q(a):
        a = a[a >= 0]
        if not len(a):
            return "-"
        return "p10 %.2f p50 %.2f p90 %.2f max %.2f us" % tuple(np.percentile(a, [10, 50, 90, 100]) / 1e3)
    print(" start     ", q(rel[:, 0]))
    print(" staged    ", q(rel[:, 1]))
    for i in range(6):
        s = 2 + 2 * i                      # slots: 2+2i evaluated (+ next gathers), 3+2i reduced
        prev = tr[:, 1] if i == 0 else tr[:, s - 1]
        ok = (tr[:, s] > 0) & (prev > 0) & (tr[:, s + 1] > 0)
        if not ok.any():
            break
        print(f" tile{i}: (B0+) eval+gather {q(np.where(ok, tr[:, s] - prev, -1))}")
        print(f"        B1+reduce+RED {q(np.where(ok, tr[:, s + 1] - tr[:, s], -1))}")
    print(" grid sync ", q(rel[:, 62]), "(then the side targets, summed by the whole grid)" if (tr[:, 62] > 0).any()
          else "(none: no side targets)")
    print(" end       ", q(rel[:, 63]))


if __name__ == "__main__":
    main()

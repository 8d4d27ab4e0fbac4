#!/usr/bin/env python
"""B5 sweep records (bench.py --sweep-out JSONL) -> markdown table.

    python tools/sweep_md.py profiles/r01_o_sweep_b5.jsonl r01_o > profiles/r01_o_sweep_b5.md
"""
import json
import sys

V = ["color", "color_buf", "atomic", "gather", "tile", "color_hybrid"]
recs = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
tag = sys.argv[2] if len(sys.argv) > 2 else ""
n = recs[0]["n_dev"] if recs else 0
print(f"# B5 crossover sweep ({tag}): gen_synth, N = {n:,} FETs, C = 1..4096; us per call (median, clean L2 flush)")
print()
print("C_hybrid = colours under the degree-threshold hybrid rule (K = 64). Fastest per row in bold.")
print()
print("| C | C_hybrid | " + " | ".join(V) + " | AUTO picks |")
print("|---|---|" + "---|" * len(V) + "---|")
for r in recs:
    ms = r["ms"]
    best = min(ms, key=ms.get)
    cells = [(f"**{ms[v] * 1e3:.0f}**" if v == best else f"{ms[v] * 1e3:.0f}") for v in V]
    print(f"| {r['C']} | {r.get('C_hybrid', '')} | " + " | ".join(cells) + f" | {r['auto']} |")

#!/usr/bin/env python
"""B5 sweep records (bench.py --sweep-out JSONL) -> markdown table, with the
five BASELINE configs' colour counts (profiles/config_colors.json, both
conflict rules) marked at the sweep row they fall on (
the GPU analogue of the paper's Fig. 5(c-d)).

    python tools/sweep_md.py profiles/r02_sweep_b5.jsonl r02 > profiles/r02_sweep_b5.md
"""
import json
import math
import os
import sys

V = ["color", "color_buf", "atomic", "gather", "tile", "color_hybrid"]
recs = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
tag = sys.argv[2] if len(sys.argv) > 2 else ""
cc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "config_colors.json")
marks = {}
if os.path.exists(cc):
    for name, r in json.load(open(cc)).items():
        for rule, short in (("exclude_rails", "rails excl."), ("paper", "paper rule")):
            C = r[f"C_{rule}"]
            # nearest sweep row on a log scale (the sweep doubles C)
            row = min(recs, key=lambda q: abs(math.log(max(1, q["C"])) - math.log(max(1, C))))["C"]
            marks.setdefault(row, []).append(f"{name} {short} C={C:,}")
n = recs[0]["n_dev"] if recs else 0
print(f"# B5 crossover sweep ({tag}): gen_synth, N = {n:,} FETs, C = 1..4096; us per call (median, clean L2 flush)")
print()
print("C_hybrid = colours under the degree-threshold hybrid rule (K = 64). Fastest per row in bold. "
      "'configs here' marks the BASELINE configs whose colour count (either conflict rule, "
      "profiles/config_colors.json) is nearest this row; counts above 4,096 are marked on the last row.")
print()
print("| C | C_hybrid | " + " | ".join(V) + " | AUTO picks | configs here |")
print("|---|---|" + "---|" * len(V) + "---|---|")
for r in recs:
    ms = r["ms"]
    best = min(ms, key=ms.get)
    cells = [(f"**{ms[v] * 1e3:.0f}**" if v == best else f"{ms[v] * 1e3:.0f}") for v in V]
    print(f"| {r['C']} | {r.get('C_hybrid', '')} | " + " | ".join(cells) + f" | {r['auto']} | "
          + "; ".join(marks.get(r["C"], [])) + " |")

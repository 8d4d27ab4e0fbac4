#!/usr/bin/env python
"""Colour count C of the five BASELINE configs under both conflict rules
(rails excluded / paper-literal), from the library's host-only setup
(no GPU): the marks of the B5 crossover table.

    python tools/config_colors.py > profiles/config_colors.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import netgen  # noqa: E402
from paper_2604_03079_b200 import Context  # noqa: E402


def main():
    out = {}
    for c in range(5):
        nl = netgen.config(c)
        rec = {"workload": netgen.CONFIG_NAMES[c], "n_dev": nl.n_dev}
        for rule in ("exclude_rails", "paper"):
            ctx = Context.from_netlist(nl, variant="atomic", rule=rule, host_only=True)
            st = ctx.stats()
            rec[f"C_{rule}"] = st["n_colors"]
            rec[f"max_conflict_node_degree_{rule}"] = st["max_conflict_node_degree"]
            ctx.close()
        out[f"cfg{c}"] = rec
        print(c, rec, file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

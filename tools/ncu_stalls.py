#!/usr/bin/env python
"""Warp-stall and shared-memory-wavefront attribution of one kernel from an
`ncu --set full --import-source on` report (its source page, per SASS line).

    python tools/ncu_stalls.py gpurun_out/r02_e/prof_c4_tile.ncu-rep [top_n] >> profiles/r02_e_tile_stalls.md
"""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def main(rep, top_n=14):
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kernel = rows[0][1] if rows and len(rows[0]) > 1 else "?"
    h, R = rows[1], rows[2:]
    ix = {k: i for i, k in enumerate(h)}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError, IndexError):
            return 0.0

    tot = sum(f(r, "# Samples") for r in R)
    st = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    print(f"## {rep.split('/')[-1]}: `{kernel[:60]}`\n")
    print(f"- warp instructions executed: {int(sum(f(r, 'Instructions Executed') for r in R)):,}")
    print(f"- shared-memory wavefronts: {int(sum(f(r, 'L1 Wavefronts Shared') for r in R)):,} "
          f"(ideal {int(sum(f(r, 'L1 Wavefronts Shared Ideal') for r in R)):,})")
    shares = sorted(((sum(f(r, k) for r in R), k[6:]) for k in st), reverse=True)[:8]
    print(f"- stall samples ({int(tot):,}): " + ", ".join(f"{k} {100 * v / tot:.1f}%" for v, k in shares))
    print("\n| SASS | samples | executed | top stall |\n|---|---|---|---|")
    for r in sorted(R, key=lambda r: -f(r, "# Samples"))[:top_n]:
        s = max(((f(r, k), k[6:]) for k in st))
        print(f"| `{r[ix['Source']].strip()[:60]}` | {int(f(r, '# Samples'))} | "
              f"{int(f(r, 'Instructions Executed')):,} | {s[1]} {int(s[0])} |")
    print()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 14)

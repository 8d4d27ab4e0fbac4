#!/usr/bin/env python
"""Summarise a gpurun_out/ directory (bench JSON lines + ncu reports) into
markdown / JSON under profiles/.

    python tools/summarize.py gpurun_out profiles/r01
"""
import csv
import glob
import io
import json
import os
import re
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
RAW_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__bytes.sum.per_second",
            "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
            "lts__t_requests_srcunit_tex_op_red.sum",
            "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
            "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
            "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_sector_hit_rate.pct"]


def bench_lines(d):
    out = []
    for f in sorted(glob.glob(os.path.join(d, "bench*.log"))):
        for line in open(f):
            line = line.strip()
            if line.startswith("{"):
                try:
                    j = json.loads(line)
                except Exception:
                    continue
                j["_file"] = os.path.basename(f)
                out.append(j)
    return out


def ncu_raw(rep):
    r = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k in RAW_KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = row[i] + (" " + units[i] if units[i] else "")
        res.append(d)
    return res


def main(src, dst):
    os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
    lines = bench_lines(src)
    md = ["# bench + ncu summary", "", f"source: `{src}`", ""]
    md.append("| file | config | variant | FET/s | ms/step | kernel ms | roofline frac | frac of stream probe | e2e FET/s |")
    md.append("|---|---|---|---|---|---|---|---|---|")
    for j in lines:
        r = j.get("roofline", {})
        e = j.get("e2e") or {}
        md.append(f"| {j['_file']} | {j['config'].get('config_index')} | {j['config'].get('variant')} | "
                  f"{j['value']:.3e} | {j['ms_per_step']:.4f} | {r.get('kernel_ms', 0):.4f} | "
                  f"{r.get('frac', 0):.3f} | {(r.get('stream_ref') or {}).get('frac', float('nan')):.3f} | "
                  f"{e.get('value', 0):.3e} |")
        for name, pc in (j.get("per_config") or {}).items():
            pr = pc.get("roofline", {})
            md.append(f"| {j['_file']} per_config | {name} | {pc.get('variant')} | {pc['value']:.3e} | "
                      f"{pc['ms_per_step']:.4f} | {pr.get('kernel_ms', 0):.4f} | {pr.get('frac', 0):.3f} | "
                      f"{pc.get('stream_ref_frac', float('nan')):.3f} | |")
    md.append("")
    reps = sorted(glob.glob(os.path.join(src, "*.ncu-rep")))
    ncu = {}
    for rep in reps:
        rows = ncu_raw(rep)
        ncu[os.path.basename(rep)] = rows
        md.append(f"## {os.path.basename(rep)}")
        for d in rows:
            md.append(f"- `{d['kernel'][:70]}`")
            for k in RAW_KEYS:
                if k in d:
                    md.append(f"  - {k}: {d[k]}")
        md.append("")
    open(dst + ".md", "w").write("\n".join(md) + "\n")
    update_traffic(ncu, src, os.path.basename(dst))
    json.dump({"bench": lines, "ncu": ncu}, open(dst + ".json", "w"), indent=1)
    print(dst + ".md")


_UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def _bytes(v):
    num, unit = v.split()
    return float(num) * _UNIT[unit]


def update_traffic(ncu, src, profile):
    """profiles/traffic.json: DRAM read+write bytes per launch of the dominant
    kernel, from `ncu --set full` captures named prof_c<cfg>_<variant>.ncu-rep
    (bench.py reports it as roofline.traffic), tagged with the profile name
    and the hash of the kernel sources the capture ran on (src_hash.txt
    written by the GPU script; bench.py drops a figure whose hash differs)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    hf = os.path.join(src, "src_hash.txt")
    if not os.path.exists(hf):
        print("no src_hash.txt in", src, "- traffic.json not updated")
        return
    h = open(hf).read().strip()
    for rep, rows in ncu.items():
        m = re.match(r"prof_c(\d)_(\w+?)\.ncu-rep", rep)
        if not m or not rows:
            continue
        r = rows[0]
        if "dram__bytes_read.sum" not in r:
            continue
        d.setdefault(f"cfg{m.group(1)}", {})[m.group(2)] = {
            "bytes": _bytes(r["dram__bytes_read.sum"]) + _bytes(r["dram__bytes_write.sum"]),
            "profile": f"{profile} ({rep})", "src_hash": h}
    json.dump(d, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

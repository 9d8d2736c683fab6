#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

  python tools/ncu_summary.py launches <launches.csv> [--bench bench.json]
  python tools/ncu_summary.py full <prof.ncu-rep>

The launch list (gpu__time_duration + dram bytes per launch, cold-cache and
serialised under ncu) is reduced to one row per kernel kind: launches, mean
duration, DRAM bytes per launch, achieved DRAM GB/s and the share of the
step's kernel time.  The full capture is reduced to the speed-of-light,
occupancy and stall lines that matter for an HBM-bound kernel.
"""
import csv
import json
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(anonymous namespace\)::|nsm::|unnamed>::|void ", "", name)
    name = re.sub(r"\(long, .*", "", name)
    return name.strip()


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) <= max(ki, mi, vi):
            continue
        per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[idi]] = short(r[ki])
    agg = OrderedDict()
    for lid, m in per.items():
        a = agg.setdefault(names[lid], {"n": 0, "t": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["t"] += m.get("gpu__time_duration.sum", 0.0)
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["t"] for a in agg.values()) or 1.0
    out = ["| kernel | launches | mean µs | DRAM MB/launch (rd+wr) | DRAM GB/s | share of kernel time |",
           "|---|---|---|---|---|---|"]
    for k, a in agg.items():
        t = a["t"] / a["n"]
        b = (a["rd"] + a["wr"]) / a["n"]
        out.append(f"| `{k}` | {a['n']} | {t / 1e3:.1f} | {b / 1e6:.1f} | {b / t:.0f} | {a['t'] / tot:.1%} |")
    return "\n".join(out)


KEYS = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Waves Per SM", "Issued Warp Per Scheduler", "No Eligible", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction"]


def full(path: str) -> str:
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    ni, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    out = []
    seen = set()
    kern = None
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if kern is None:
            kern = short(r[ni])
            out += [f"kernel `{kern}`", "", "| metric | value |", "|---|---|"]
        key = (r[mi], r[ui])
        if r[mi] in KEYS and key not in seen:
            seen.add(key)
            out.append(f"| {r[mi]} ({r[ui]}) | {r[vi]} |")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        h, u, v = rr[0], rr[1], rr[2]
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "lts__t_bytes.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"):
            if k in h:
                j = h.index(k)
                out.append(f"| {k} ({u[j]}) | {v[j]} |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))

#!/usr/bin/env python
"""Write profiles/<name>.md from a tools/gpu_final.sh run brought back in gpurun_out/
(bench lines C2..C5, the reference arm, ncu launch lists and the full capture of the C2
residual) and refresh profiles/ncu_traffic.json and the committed launch lists.

  python tools/round_md.py r01_v9_round "title" "intro paragraph"
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")


def sh(*a):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), *a],
                          capture_output=True, text=True, check=True).stdout


def main(name, title, intro):
    b = {c: json.load(open(os.path.join(G, f"bench_{c}.json"))) for c in ["C2", "C3", "C4", "C5"]}
    ref = json.loads(open(os.path.join(G, "bench_ref.json")).readline())
    l2 = sh("launches", os.path.join(G, "launches_C2.csv"), "--bench", os.path.join(G, "bench_C2.json"))
    l5 = sh("launches", os.path.join(G, "launches_C5.csv"))
    full = sh("full", os.path.join(G, "prof_residual_C2.ncu-rep"))
    rd = wr = None
    for line in full.splitlines():
        if line.startswith("| dram__bytes_read.sum (Mbyte)"):
            rd = float(line.split("|")[2])
        if line.startswith("| dram__bytes_write.sum (Mbyte)"):
            wr = float(line.split("|")[2])
    traffic = int(round((rd + wr) * 1e6)) if rd is not None and wr is not None else None
    if traffic:
        json.dump({"_source": "ncu --set full (cold cache, serialised): dram__bytes_read.sum + dram__bytes_write.sum "
                              f"of one launch; profiles/{name}.md", "C2": {"residual": traffic}},
                  open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    for c in ["C2", "C5"]:
        shutil.copy(os.path.join(G, f"launches_{c}.csv"), os.path.join(ROOT, "profiles", f"r01_launches_{c}.csv"))
    rows = []
    for c, d in b.items():
        r = d["roofline"]
        parts = ", ".join(d["config"].get("offset_aligned_parts") or []) or "-"
        rows.append(f"| {c} | {d['ms_per_step']} | {d['value']} | {d['config']['frac_of_hbm_peak']} | "
                    f"{d['config']['floor_gbs']} | {r['frac']} | {r['alone_frac']} | {r['sweeps_frac']} | {parts} | "
                    f"{d['e2e']['value']} |")
    clk = b["C2"]["clocks"]
    md = f"""# {title}

`bash tools/gpu_final.sh` on one B200 (SM clock {clk['sm_mhz']} MHz under load, throttle reasons {clk['reasons']}).
{intro}

| config | ms / apply | GB/s | of measured peak | floor GB/s | residual in-step | residual alone | sweeps | aligned parts | e2e GB/s |
|---|---|---|---|---|---|---|---|---|---|
""" + "\n".join(rows) + f"""

`value` = algorithmic bytes of the path that ran / device time, L2 flushed before each step; `floor GB/s` = the
implementation-independent floor (each stored entry at 12 B, each n-vector once) / the same time; `e2e` = the same
bytes / the time of `nsm_smooth_host` on pinned host vectors (PCIe copies included).

Reference arm (`bench.py --impl reference`: the single-threaded C oracle, C2): {ref['ms_per_step']} ms per
application, {ref['value']} GB/s.

Full bench line (C2, the default workload):

```json
{json.dumps(b['C2'])}
```

## ncu launch list, C2 default command (cold cache, serialised; `profiles/r01_launches_C2.csv`)

{l2}
(The `at::` kernels are the bench's own L2-flush fill/read, outside the timed smoother calls.)

## ncu launch list, C5 (`profiles/r01_launches_C5.csv`)

{l5}
## ncu --set full, C2 residual kernel

{full}
DRAM traffic per launch {traffic / 1e6 if traffic else float('nan'):.1f} MB vs the algorithmic
{b['C2']['roofline']['bytes_per_launch'] / 1e6:.1f} MB (the r write stays in L2 at kernel end).
"""
    open(os.path.join(ROOT, "profiles", f"{name}.md"), "w").write(md)
    print(f"profiles/{name}.md written; traffic {traffic}")


if __name__ == "__main__":
    main(*sys.argv[1:4])

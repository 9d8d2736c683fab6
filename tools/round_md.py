#!/usr/bin/env python
"""Write profiles/<name>.md from a tools/gpu_final.sh run brought back in gpurun_out/
(bench lines C2..C5 with C3 the default workload, the reference arm, ncu launch lists of
C3 and C4 and the full captures of their residual kernels and the C3 sweep) and refresh
profiles/ncu_traffic.json and the committed launch lists.

  python tools/round_md.py r02_round "title" "intro paragraph"
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


def dram_of(full: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of a full-capture summary
    (ncu prints them in byte / Kbyte / Mbyte / Gbyte)."""
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    got = {}
    for line in full.splitlines():
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if line.startswith(f"| {k} ("):
                unit = line.split("(")[1].split(")")[0]
                got[k] = float(line.split("|")[2]) * scale.get(unit, float("nan"))
    if len(got) != 2:
        return None
    return int(round(got["dram__bytes_read.sum"] + got["dram__bytes_write.sum"]))


def main(name, title, intro):
    b = {c: json.load(open(os.path.join(G, f"bench_{c}.json"))) for c in ["C3", "C2", "C4", "C5"]}
    ref = json.loads(open(os.path.join(G, "bench_ref.json")).readline())
    l3 = sh("launches", os.path.join(G, "launches_C3.csv"))
    l4 = sh("launches", os.path.join(G, "launches_C4.csv"))
    fulls = {k: sh("full", os.path.join(G, f"prof_{k}.ncu-rep")) for k in ("residual_C3", "sweep_C3", "residual_C4")}
    traffic = {k: dram_of(v) for k, v in fulls.items()}
    json.dump({"_source": "ncu --set full (cold cache, serialised): dram__bytes_read.sum + dram__bytes_write.sum "
                          f"of one launch; profiles/{name}.md",
               "C3": {"residual": traffic["residual_C3"], "sweep": traffic["sweep_C3"]},
               "C4": {"residual": traffic["residual_C4"]}},
              open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    for c in ["C3", "C4"]:
        shutil.copy(os.path.join(G, f"launches_{c}.csv"), os.path.join(ROOT, "profiles", f"{name}_launches_{c}.csv"))
    coupled_md = ""
    cp = os.path.join(G, "prof_coupled_C3.ncu-rep")
    cl = os.path.join(G, "bench_C3_coupled.json")
    if os.path.exists(cp) and os.path.exists(cl):
        dc = json.loads(open(cl).readline())
        coupled_md = (f"## Coupled sweeps (opt-in, `--coupled on`): C3 {dc['ms_per_step']} ms per application, "
                      f"sweeps kernel at {dc['roofline'].get('sweeps_frac')} of peak on its algorithmic bytes\n\n"
                      + sh("full", cp) + "\n")
    rows = []
    for c, d in b.items():
        r = d["roofline"]
        det = d.get("detail", {})
        parts = ", ".join(det.get("offset_aligned_parts") or []) or "-"
        rows.append(f"| {c} | {d['ms_per_step']} | {d['value']} | {det.get('frac_of_hbm_peak')} | "
                    f"{det.get('floor_gbs')} | {r['frac']} | {r.get('alone_frac')} | {r.get('sweeps_frac')} | {parts} | "
                    f"{d['e2e']['value']} |")
    clk = b["C3"]["clocks"]
    cpu = b["C3"].get("cpu_baseline") or {}
    md = f"""# {title}

`bash tools/gpu_final.sh` on one B200 (SM clock {clk['sm_mhz']} MHz under load, throttle reasons {clk['reasons']}).
{intro}

| config | ms / apply | GB/s | of measured peak | floor GB/s | residual in-step | residual alone | sweeps | aligned parts | e2e GB/s |
|---|---|---|---|---|---|---|---|---|---|
""" + "\n".join(rows) + f"""

`value` = algorithmic bytes of the path that ran / device time, L2 flushed before each step; `floor GB/s` = the
implementation-independent floor (each stored entry at 12 B, each n-vector once) / the same time; `e2e` = the same
bytes / the time of `nsm_smooth_host` on pinned host vectors (PCIe copies included).

CPU oracle on the box's host (C3, the default line's `cpu_baseline`): all cores {cpu.get('cores')} threads
{cpu.get('ms_per_apply')} ms per application ({cpu.get('value')} GB/s); one thread
{(cpu.get('single_core') or {}).get('ms_per_apply')} ms ({(cpu.get('single_core') or {}).get('value')} GB/s).
Reference arm (`bench.py --impl reference`, the all-cores oracle, C3): {ref.get('ms_per_step')} ms per
application, {ref.get('value')} GB/s.

Full bench line (C3, the default workload):

```json
{json.dumps(b['C3'])}
```

## ncu launch list, default command (C3; cold cache, serialised; `profiles/{name}_launches_C3.csv`)

{l3}
(The `at::` kernels are the bench's own L2-flush reads, outside the timed smoother calls.)

## ncu launch list, C4 (`profiles/{name}_launches_C4.csv`)

{l4}
## ncu --set full, C3 residual kernel

{fulls['residual_C3']}
## ncu --set full, C3 sweep kernel

{fulls['sweep_C3']}
## ncu --set full, C4 residual kernel

{fulls['residual_C4']}
{coupled_md}DRAM traffic per launch (ncu, cold): C3 residual {(traffic['residual_C3'] or 0) / 1e6:.1f} MB vs the algorithmic
{b['C3']['roofline']['bytes_per_launch'] / 1e6:.1f} MB; C4 residual {(traffic['residual_C4'] or 0) / 1e6:.1f} MB vs
{b['C4']['roofline']['bytes_per_launch'] / 1e6:.1f} MB.
"""
    open(os.path.join(ROOT, "profiles", f"{name}.md"), "w").write(md)
    return md
    print(f"profiles/{name}.md written; traffic {traffic}")


if __name__ == "__main__":
    main(*sys.argv[1:4])

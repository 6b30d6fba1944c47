"""Summarise ncu reports into profiles/ (run in the build container, reads gpurun_out/*.ncu-rep).

    python tools/ncu_summary.py --round r01 [--launches gpurun_out/launches_bench.csv]

Writes profiles/<round>_ncu_summary.md (one row per profiled kernel: duration, DRAM bytes and
throughput, L2/L1 hit, SM/issue utilisation, occupancy, registers) and profiles/ncu_traffic.json
(DRAM bytes per launch per bench config, read by bench.py for roofline.traffic).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
]
# report name -> bench config key
REPORTS = {
    "hotspot2d": "hotspot2d",
    "hotspot3d_512": "hotspot3d",
    "hotspot3d_large": "hotspot3d_large",
    "fdtd": "fdtd",
    "fdtd_fused": "fdtd_fused",
    "skeleton": "skeleton",
}
UNIT = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw(rep: str) -> list[dict]:
    if rep.endswith(".csv"):  # `ncu --page raw --csv` already exported on the GPU box
        with open(rep) as fh:
            out = fh.read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                             capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = None
                d[m] = (v, units[i])
        res.append(d)
    return res


def scaled(entry, m, to):
    v, u = entry[m]
    return None if v is None else v * UNIT.get(u, 1.0) / to


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--dir", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    lines = [f"# ncu summary ({a.round})", "",
             "`ncu --set full --clock-control none --import-source on` of `tools/profile_run.py` "
             "(stream mode, binary64 and binary32, the BASELINE configs), via `tools/profile_all.sh`. Times are "
             "cold-cache, serialised replays (compare shares, not absolutes); DRAM bytes are per launch.",
             "",
             "| config | dtype | kernel | grid x block | regs | time (us) | DRAM read (MB) | DRAM write (MB) | "
             "DRAM % peak | L2 hit % | L1 hit % | SM % | warps active % | inst (M) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for (rep, key), dtype in [(kv, dt) for dt in ("f64", "f32") for kv in REPORTS.items()]:
        path = os.path.join(a.dir, f"ncu_{rep}_{dtype}_raw.csv")
        if not os.path.exists(path):
            path = os.path.join(a.dir, f"ncu_{rep}_{dtype}.ncu-rep")
        if not os.path.exists(path):
            continue
        per_kernel = {}
        for e in raw(path):
            name = e["kernel"].split("(")[0].replace("void ", "").strip()
            t_us = scaled(e, "gpu__time_duration.sum", 1e-6)
            rd = scaled(e, "dram__bytes_read.sum", 1e6)
            wr = scaled(e, "dram__bytes_write.sum", 1e6)
            lines.append(
                f"| {key} | {dtype} | `{name}` | {int(e['launch__grid_size'][0])} x {int(e['launch__block_size'][0])} | "
                f"{int(e['launch__registers_per_thread'][0])} | {t_us:.2f} | {rd:.2f} | {wr:.2f} | "
                f"{e['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]:.1f} | "
                f"{e['lts__t_sector_hit_rate.pct'][0]:.1f} | {e['l1tex__t_sector_hit_rate.pct'][0]:.1f} | "
                f"{e['sm__throughput.avg.pct_of_peak_sustained_elapsed'][0]:.1f} | "
                f"{e['sm__warps_active.avg.pct_of_peak_sustained_active'][0]:.1f} | "
                f"{e['smsp__inst_executed.sum'][0] / 1e6:.2f} |")
            per_kernel.setdefault(name, []).append((rd + wr) * 1e6)
        # bytes per iteration = sum over the iteration's kernels of their mean per-launch traffic
        traffic[f"{key}:{dtype}"] = int(sum(sum(v) / len(v) for v in per_kernel.values()))
    if a.launches and os.path.exists(a.launches):
        lines += ["", "## Launch list of a short bench run (`ncu --metrics gpu__time_duration.sum`)", ""]
        shares = {}
        with open(a.launches) as fh:
            rows = [r for r in csv.reader(fh) if len(r) > 10]
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        for r in rows[1:]:
            try:
                v = float(r[vi].replace(",", ""))
            except ValueError:
                continue
            n = r[ki].split("(")[0].replace("void ", "").strip()
            c, t = shares.get(n, (0, 0.0))
            shares[n] = (c + 1, t + v)
        tot = sum(t for _, t in shares.values())
        lines += ["| kernel | launches | total time (ms) | share |", "|---|---|---|---|"]
        for n, (c, t) in sorted(shares.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{n}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.round}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("\n".join(lines))
    print(json.dumps(traffic))


if __name__ == "__main__":
    sys.exit(main())

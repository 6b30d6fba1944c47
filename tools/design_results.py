"""Regenerate the results table and the e2e bullet of DESIGN.md §10 from the committed bench lines
(profiles/r02_bench_1gpu.json, profiles/r02_bench_reference.json), so the document quotes the
measured numbers verbatim. Docs tooling.
    python tools/design_results.py"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_1gpu.json")))
ref = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_reference.json")))
c, f = d["configs"], d["f32"]


def pair(name, key, fmt):
    return " / ".join(fmt.format(c[name][dt][key]) for dt in ("f32", "f64"))


def frac(name):
    return " / ".join(f"{c[name][dt]['roofline']['frac']:.3f}" for dt in ("f32", "f64"))


rows = [
    "| Config (BASELINE.json) | dtype | K | graph µs/iter | stream µs/iter | graph vs stream (± err) | HBM fraction |",
    "|---|---|---|---|---|---|---|",
    f"| **Hotspot2D 1024², N = 10⁴ (headline)** | **f64** | {d['impl_detail']['batch_size']} | **{d['value']:.2f}** | "
    f"{d['stream_us_per_iter']:.2f} | **{d['speedup_vs_stream']:.2f}× ± {d['speedup_vs_stream_err']:.3f}** | "
    "L2-resident: launch/pattern floor |",
    f"| Hotspot2D 1024², N = 10⁴ | f32 | {f['batch_size']} | {f['us_per_iter']:.2f} | {f['stream_us_per_iter']:.2f} | "
    f"{f['speedup_vs_stream']:.2f}× ± {f['speedup_vs_stream_err']:.3f} | L2-resident |",
]
for name, label, nd, hbm in (("skeleton", "Skeleton 2¹⁴, N = 10⁴", 2, None),
                             ("hotspot3d", "Hotspot3D 512²×8, N = 10³", 2, None),
                             ("fdtd", "FDTD 256³, two half-steps, N = 2000", 1, ""),
                             ("fdtd_fused", "FDTD 256³, fused leapfrog, N = 2000", 1, " (of 48 / 96 B/cell)"),
                             ("hotspot3d_large", "Hotspot3D 2048²×256, N = 100", 0, "")):
    num = "{:.%df}" % nd
    last = ("launch-bound" if name == "skeleton" else "L2-resident") if hbm is None else (
        f"**{frac(name)}**{hbm}" if not hbm else f"{frac(name)}{hbm}")
    rows.append(f"| {label} | f32 / f64 | {pair(name, 'batch_size', '{}')} | {pair(name, 'us_per_iter', num)} | "
                f"{pair(name, 'stream_us_per_iter', num)} | {pair(name, 'speedup_vs_stream', '{:.2f}×')} | {last} |")
e, cb = d["e2e"], d["cpu_baseline"]
k = d["impl_detail"]["batch_size"]
e2e = (f"* **Headline e2e** (the drop-in call `workloads.run_batched(hotspot_program(), HotspotWorkload(binary64),\n"
       f"  {k}, {10000 // k})`, host wall clock incl. conversion, pageable H2D, build, launches, D2H and the result\n"
       f"  dataclass): {e['value']:.2f} µs/iter; the pinned `DeviceSolver` path {e['pinned']['value']:.2f}. The **unmodified "
       f"reference** on\n  the same box's {cb['host_cores']} host cores (`iterbatch.workloads.time_workload`, LOOP, "
       f"workers={cb['cores']}; serial\n  {cb['workers_none_us_per_iter']:,.0f}): {cb['value']:,.0f} µs/iter (`cpu_baseline`), "
       f"and the reference arm {ref['value']:,.0f} µs/iter\n  (`profiles/r02_bench_reference.json`) — both binary64, the "
       f"same config object.\n")
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
a = s.index("| Config (BASELINE.json) | dtype | K |")
b = s.index("* **Headline e2e**")
s = s[:a] + "\n".join(rows) + "\n\n" + s[b:]
a = s.index("* **Headline e2e**")
b = s.index("* Every launch-bound config meets")
s = s[:a] + e2e + s[b:]
open(p, "w").write(s)
print("\n".join(rows))
print(e2e)

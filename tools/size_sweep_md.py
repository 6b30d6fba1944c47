"""Render gpurun_out/size_sweep.json (tools/size_sweep.py) as profiles/<round>_size_sweep.md."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for dt in ("f64", "f32"):
    path = os.path.join(ROOT, "gpurun_out", f"size_sweep_{dt}.json")
    if os.path.exists(path):
        rows += json.load(open(path))
out = [f"# Problem-size sweep on one B200 ({rnd})", "",
       "`python tools/size_sweep.py` under gpurun (DTYPE=f64 and f32): device time per iteration (CUDA events, L2 "
       "flushed before every run, median of 3), graph = best of K ∈ {10, 50, 100} × programmatic edges "
       "on/off, stream = Listing 1; HBM = algorithmic bytes per iteration / graph time against the "
       "measured copy bandwidth. The paper's picture: graph batching pays most where the per-iteration "
       "kernel is short (launch-bound), and never loses at large sizes.", "",
       "| dtype | workload | size | iterations | graph µs/iter | stream µs/iter | graph vs stream | HBM fraction | K | PDL |",
       "|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    out.append(f"| {r.get('dtype', 'f32')} | {r['workload']} | {'x'.join(map(str, r['size']))} | {r['iterations']} | "
               f"{r['graph_us_per_iter']:.3f} | {r['stream_us_per_iter']:.3f} | {r['speedup']:.2f}× | "
               f"{r['hbm_frac']:.2f} | {r['K']} | {r['pdl']} |")
open(os.path.join(ROOT, "profiles", f"{rnd}_size_sweep.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:12]))

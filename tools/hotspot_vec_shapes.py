"""Hotspot (default: binary64 Hotspot2D 1024^2, the headline config) per k_hotspot_vec shape: rows
per thread R, CTA size, CTA width, warp shuffles; graph with PDL edges at K = 100, device us/iter,
median of 5, interleaved (every shape once per round, 3 rounds). Diagnostic.
    python tools/hotspot_vec_shapes.py            # DTYPE=f32, SIZE=512,8 (Hotspot3D) ..."""
import itertools
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

KEYS = ("IB_HOTSPOT_VEC_ROWS", "IB_HOTSPOT_BLOCK", "IB_HOTSPOT_BX", "IB_HOTSPOT_SHUFFLE", "IB_HOTSPOT_KERNEL")
dtype = os.environ.get("DTYPE", "f64")
size = [int(x) for x in os.environ.get("SIZE", "1024").split(",")]
workload = "hotspot2d" if len(size) == 1 else "hotspot3d"
st = cli.build_workload(workload, size)
RS = (1, 2) if workload == "hotspot2d" else (1, 2, 4)
shapes = [("auto", {})]
BXS = tuple(int(x) for x in os.environ.get("BXS", "64,128,256").split(","))
SHS = tuple(int(x) for x in os.environ.get("SHS", "0,1").split(","))
if os.environ.get("RS"):
    RS = tuple(int(x) for x in os.environ["RS"].split(","))
for r, bs, bx, sh in itertools.product(RS, (128, 256, 512, 1024), BXS, SHS):
    if bx > bs:
        continue
    shapes.append((f"R={r} block={bs} bx={bx} sh={sh}", {"IB_HOTSPOT_KERNEL": "vec", "IB_HOTSPOT_VEC_ROWS": r,
                                                          "IB_HOTSPOT_BLOCK": bs, "IB_HOTSPOT_BX": bx,
                                                          "IB_HOTSPOT_SHUFFLE": sh}))
res = {name: [] for name, _ in shapes}
n, k = (2000, 100) if workload == "hotspot2d" else (1000, 50)
for _ in range(3):
    for name, env in shapes:
        for key in KEYS:
            os.environ.pop(key, None)
        os.environ.update({key: str(v) for key, v in env.items()})
        s = wl.DeviceSolver(st, dtype)
        s.run_batched(k, n // k, pdl=True)
        g = []
        for _ in range(5):
            s.flush_l2()
            g.append(s.run_batched(k, n // k, pdl=True).gpu_s / n)
        d = s.describe()[0]
        s.close()
        res[name].append((1e6 * statistics.median(g), d["grid"], d["block"]))
for name, v in sorted(res.items(), key=lambda kv: statistics.median(x[0] for x in kv[1])):
    print(f"{dtype} {workload} {name:34s} {statistics.median(x[0] for x in v):7.3f} us/iter  grid {v[0][1]} block {v[0][2]}", flush=True)

"""k_hotspot_tma shape sweep on Hotspot3D 2048x2048x256 (diagnostic): groups per thread G
(IB_TMA_GROUPS), ring depth (IB_TMA_STAGES), rows per CTA (IB_HOTSPOT_RPC); device-timed graph
execution (K = 5, 20 iterations, L2 flushed), median of 3, and the HBM fraction of 12 (24) B/cell.

    DTYPE=f64 python tools/tma_tune.py
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

dtype = os.environ.get("DTYPE", "f64")
size = [int(x) for x in os.environ.get("SIZE", "2048,2048,256").split(",")]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
st = cli.build_workload("hotspot3d", size)
groups = (2, 4) if dtype == "f64" else (1, 2, 4)
variants = [("auto", {})]
for g in groups:
    for ns in (3, 4, 6):
        for rpc in (0, 8, 32):
            variants.append((f"G={g} ns={ns} rpc={rpc or 'auto'}",
                             {"IB_TMA_GROUPS": g, "IB_TMA_STAGES": ns, **({"IB_HOTSPOT_RPC": rpc} if rpc else {})}))
if os.environ.get("AUTO_ONLY"):
    variants = variants[:1]
KEYS = ("IB_TMA_GROUPS", "IB_TMA_STAGES", "IB_HOTSPOT_RPC")
s = wl.DeviceSolver(st, dtype)
cells = size[0] * size[1] * size[2]
B = cells * 3 * (8 if dtype == "f64" else 4)
try:
    for name, env in variants:
        for k in KEYS:
            os.environ.pop(k, None)
        for k, v in env.items():
            os.environ[k] = str(v)
        s.build_graph(5)  # the launch list is computed at build time from the environment
        s.run_graph(1)
        t = []
        for _ in range(3):
            s.flush_l2()
            t.append(s.run_graph(4).gpu_s / 20)
        s.destroy_graph()
        d = s.describe()[0]
        us = 1e6 * statistics.median(t)
        print(f"{os.environ.get('IB_LIB_PATH', 'in-tree'):22s} {dtype} {name:28s} {us:9.1f} us/iter  {B / (us * 1e-6) / 1e9:7.0f} GB/s  "
              f"frac {B / (us * 1e-6) / 1e9 / peak:.3f}  grid {d['grid']} smem {d['smem']}", flush=True)
finally:
    s.close()

"""Hotspot2D vectorised-kernel shapes past one wave (diagnostic): rows per thread x CTA size at
2048^2 / 1536^2 (argv sizes), binary32, graph us/iter (one row per thread past one
wave).
    python tools/hotspot2d_shapes.py [N ...]"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl
for size in ([int(a)] for a in (sys.argv[1:] or ["2048", "1536"])):
    st = cli.build_workload("hotspot2d", size)
    for name, env in (("default", {}), ("old 256x2 R2", {"IB_HOTSPOT_VEC_ROWS": "2", "IB_HOTSPOT_BLOCK": "512"}), ("R2 256x4", {"IB_HOTSPOT_VEC_ROWS": "2", "IB_HOTSPOT_BLOCK": "1024"}),
                      ("R4 256x2", {"IB_HOTSPOT_VEC_ROWS": "4", "IB_HOTSPOT_BLOCK": "512"}),
                      ("R4 256x4", {"IB_HOTSPOT_VEC_ROWS": "4", "IB_HOTSPOT_BLOCK": "1024"}),
                      ("R1 256x2", {"IB_HOTSPOT_VEC_ROWS": "1", "IB_HOTSPOT_BLOCK": "512"}),
                      ("R2 256x1", {"IB_HOTSPOT_VEC_ROWS": "2", "IB_HOTSPOT_BLOCK": "256"})):
        for k in ("IB_HOTSPOT_VEC_ROWS", "IB_HOTSPOT_BLOCK"): os.environ.pop(k, None)
        os.environ.update(env)
        s = wl.DeviceSolver(st, "f32")
        s.run_batched(50, 4, pdl=True)
        g = []
        for _ in range(5):
            s.flush_l2(); s.upload(st)
            g.append(s.run_batched(50, 4, pdl=True).gpu_s / 200)
        d = s.describe()[0]
        s.close()
        print(size, f"{name:9s} {1e6*statistics.median(g):7.3f}  grid {d['grid'][:2]} block {d['block'][:2]}", flush=True)

"""A/B of two runtime builds on the launch-bound hotspot configs (diagnostic): run once per
library (IB_LIB_PATH), graph + PDL at K=50 and per-kernel stream, median of 7, device us/iter.
  python tools/ab_hotspot.py            # the in-tree library
  IB_LIB_PATH=ab/lib_old.so python tools/ab_hotspot.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

tag = os.environ.get("IB_LIB_PATH", "in-tree")
for w, size, n in (("hotspot2d", [1024], 2000), ("hotspot3d", [512, 8], 1000)):
    st = cli.build_workload(w, size)
    s = wl.DeviceSolver(st, "f32")
    s.run_batched(50, n // 50, pdl=True)
    g, sp = [], []
    for _ in range(7):
        s.flush_l2(); s.upload(st)
        g.append(s.run_batched(50, n // 50, pdl=True).gpu_s / n)
        s.flush_l2(); s.upload(st)
        sp.append(s.run_stream(n).gpu_s / n)
    print(f"{tag:16s} {w:9s} graph+pdl {1e6*statistics.median(g):6.3f}  stream {1e6*statistics.median(sp):6.3f}", flush=True)
    s.close()

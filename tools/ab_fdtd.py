"""A/B of two runtime builds on FDTD 256^3 binary32 (diagnostic): run once per library
(IB_LIB_PATH), two half-steps and fused, graph at K=20, device us/iter, median of 5.
  python tools/ab_fdtd.py ; IB_LIB_PATH=ab/lib_old.so python tools/ab_fdtd.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

tag = os.environ.get("IB_LIB_PATH", "in-tree")
n = int(os.environ.get("N", "200"))
st = cli.build_workload("fdtd", [int(os.environ.get("SIZE", "256"))])
for fuse in (False, True):
    s = wl.DeviceSolver(st, os.environ.get("DTYPE", "f32"), fuse=fuse)
    s.run_batched(20, n // 20)
    g = []
    for _ in range(5):
        s.flush_l2()
        g.append(s.run_batched(20, n // 20).gpu_s / n)
    print(f"{tag:28s} {'fused' if fuse else 'H+E  '} {1e6 * statistics.median(g):8.2f} us/iter", flush=True)
    s.close()

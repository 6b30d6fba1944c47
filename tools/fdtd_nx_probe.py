"""Fused / two-half-step FDTD time vs nx at ny = nz = 256 (diagnostic for slab shapes)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import workloads as wl

for nx in [int(a) for a in (sys.argv[1:] or ["64", "66", "96", "128", "130", "132", "160", "192", "256"])]:
    st = wl.te101_cavity(nx, 256, 256)
    for fuse in (False, True):
        s = wl.DeviceSolver(st, "f32", fuse=fuse)
        s.run_batched(20, 5)
        g = []
        for _ in range(3):
            s.flush_l2()
            g.append(s.run_batched(20, 5).gpu_s / 100)
        d = s.describe()
        s.close()
        print(f"nx={nx:4d} {'fused' if fuse else 'H+E  '} {1e6*statistics.median(g):8.2f} us/iter  "
              + "; ".join(f"{x['kernel'][:40]} grid {x['grid'][0]} block {x['block'][0]} smem {x['smem']}" for x in d), flush=True)

"""FDTD config sweep on short slabs (diagnostic): nx planes at ny = nz = 256, two half-steps and
fused, per (IB_FDTD_TJ, IB_FDTD_CHUNKS, IB_FDTD_STAGES)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import workloads as wl

nxs = [int(a) for a in (sys.argv[1:] or ["34", "66"])]
cfgs = [("auto", {})] + [(f"tj={tj} ch={ch} ns={ns}", {"IB_FDTD_TJ": tj, "IB_FDTD_CHUNKS": ch, "IB_FDTD_STAGES": ns})
                         for tj in (2, 3, 4) for ch in (1, 2, 3) for ns in (0, 3, 4)]
if os.environ.get("CFGS"):  # e.g. CFGS="3:3:4,3:2:4" (tj:chunks:stages)
    cfgs = [("auto", {})] + [(f"tj={a} ch={b} ns={c}", {"IB_FDTD_TJ": int(a), "IB_FDTD_CHUNKS": int(b),
                                                       "IB_FDTD_STAGES": int(c)})
                             for a, b, c in (x.split(":") for x in os.environ["CFGS"].split(","))]
for nx in nxs:
    st = wl.te101_cavity(nx, 256, 256)
    for name, env in cfgs:
        for k in ("IB_FDTD_TJ", "IB_FDTD_CHUNKS", "IB_FDTD_STAGES"):
            os.environ.pop(k, None)
        os.environ.update({k: str(v) for k, v in env.items() if v})
        row = []
        for fuse in (False, True):
            try:
                s = wl.DeviceSolver(st, "f32", fuse=fuse)
                s.run_batched(20, 5)
                g = []
                for _ in range(3):
                    s.flush_l2()
                    g.append(s.run_batched(20, 5).gpu_s / 100)
                d = s.describe()[0]
                s.close()
                row.append(f"{1e6 * statistics.median(g):7.2f} (grid {d['grid'][0]})")
            except Exception as e:
                row.append(f"err {str(e)[:40]}")
        print(f"nx={nx:3d} {name:18s} H+E {row[0]:22s} fused {row[1]}", flush=True)

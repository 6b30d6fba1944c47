"""k_hotspot_vec CTA shape sweep (diagnostic): CTA width cap IB_HOTSPOT_BX x row-blocks, rows per
thread, on the launch-bound hotspot configs; graph + PDL at K = 50, median of 5."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

for w, size, n in (("hotspot2d", [1024], 2000), ("hotspot3d", [512, 8], 1000)):
    st = cli.build_workload(w, size)
    for r in (1, 2, 4):
        for bx in (32, 64, 128, 256):
            for bs in (256, 512, 1024):
                if bs < bx:
                    continue
                os.environ.update({"IB_HOTSPOT_KERNEL": "vec", "IB_HOTSPOT_VEC_ROWS": str(r),
                                   "IB_HOTSPOT_BX": str(bx), "IB_HOTSPOT_BLOCK": str(bs)})
                s = wl.DeviceSolver(st, "f32")
                s.run_batched(50, n // 50, pdl=True)
                g = []
                for _ in range(5):
                    s.flush_l2(); s.upload(st)
                    g.append(s.run_batched(50, n // 50, pdl=True).gpu_s / n)
                print(f"{w:9s} R={r} bx={bx:3d} by={bs // bx:2d}  {1e6 * statistics.median(g):6.3f} us/iter", flush=True)
                s.close()

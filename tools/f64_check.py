"""binary64 (the reference's precision) per-iteration device time of every BASELINE config."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

CFGS = [("vector", [16384], 10000, 100, False), ("hotspot2d", [1024], 10000, 80, False),
        ("hotspot3d", [512, 8], 1000, 40, False), ("fdtd", [256], 200, 20, False),
        ("fdtd", [256], 200, 20, True), ("hotspot3d", [2048, 2048, 256], 20, 5, False)]
for w, size, n, k, fuse in CFGS:
    st = cli.build_workload(w, size)
    for dtype in ("f32", "f64"):
        s = wl.DeviceSolver(st, dtype, fuse=fuse)
        s.run_batched(k, n // k, pdl=True)
        best = None
        for pdl in (False, True):
            xs = []
            for _ in range(3):
                s.flush_l2()
                xs.append(s.run_batched(k, n // k, pdl=pdl).gpu_s / n)
            t = statistics.median(xs)
            best = t if best is None else min(best, t)
        print(f"{w:9s} {str(size):16s} fuse={int(fuse)} {dtype}: {1e6*best:9.3f} us/iter  "
              f"{s.iteration_bytes / best / 1e9:7.0f} GB/s", flush=True)
        s.close()

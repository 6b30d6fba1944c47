"""Where the vectorised lean FDTD kernels stop beating the staged k_fdtd_lf (two half-steps):
IB_FDTD_KERNEL=lean vs staged over cube sizes, both precisions; graph K = 20, best of plain / PDL
edges, median of 3. Diagnostic for the L2-size threshold in fdtd_launches.
    python tools/lean_vs_staged.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

for dtype in ("f32", "f64"):
    for n in (96, 112, 128, 144, 160, 192, 224, 256):
        st = cli.build_workload("fdtd", [n])
        it = 40 if n >= 192 else 100
        res = {}
        for kernel in ("lean", "staged", "lean", "staged"):
            os.environ["IB_FDTD_KERNEL"] = kernel
            s = wl.DeviceSolver(st, dtype)
            s.run_batched(20, it // 20)
            best = None
            for pdl in (False, True):
                xs = []
                for _ in range(3):
                    s.flush_l2()
                    xs.append(s.run_batched(20, it // 20, pdl=pdl).gpu_s / it)
                best = min(best or 1e9, statistics.median(xs))
            mb = s.iteration_bytes / 1e6
            s.close()
            res[kernel] = min(res.get(kernel, 1e9), 1e6 * best)
        print(f"{dtype} {n:4d}^3  lean {res['lean']:9.2f}  staged {res['staged']:9.2f} us/iter  "
              f"({mb:.0f} MB/iter)", flush=True)

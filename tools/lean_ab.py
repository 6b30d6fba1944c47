"""Scalar vs vectorised lean FDTD kernels (IB_FDTD_KERNEL=lean, IB_FDTD_LEANV=0/1): graph K = 20,
plain and PDL edges (the better), device us/iter, median of 3, interleaved. Diagnostic.
    python tools/lean_ab.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

CASES = [("f32", [32]), ("f32", [64]), ("f32", [128]), ("f32", [256]), ("f32", [96, 256, 720]),
         ("f64", [64]), ("f64", [128]), ("f64", [256]), ("f64", [96, 256, 384]), ("f64", [384])]
os.environ["IB_FDTD_KERNEL"] = "lean"
for dtype, dims in CASES:
    st = cli.build_workload("fdtd", dims)
    n = 200 if max(dims) <= 128 else 40
    row = {}
    for _ in range(2):
        for v in ("0", "1"):
            os.environ["IB_FDTD_LEANV"] = v
            s = wl.DeviceSolver(st, dtype)
            s.run_batched(20, n // 20)
            best = None
            for pdl in (False, True):
                xs = []
                for _ in range(3):
                    s.flush_l2()
                    xs.append(s.run_batched(20, n // 20, pdl=pdl).gpu_s / n)
                best = min(best or 1e9, statistics.median(xs))
            gbs = s.iteration_bytes / best / 1e9
            s.close()
            row.setdefault(v, []).append((1e6 * best, gbs))
    out = "  ".join(f"{'vector' if v == '1' else 'scalar'} {min(x[0] for x in r):9.2f} us/iter "
                    f"({max(x[1] for x in r):6.0f} GB/s)" for v, r in row.items())
    print(f"{dtype} {'x'.join(map(str, dims)):12s} {out}", flush=True)

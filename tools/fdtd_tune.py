"""FDTD 256^3: two-half-step vs fused variants per tile height / ring depth, device-timed (CUDA
events, programmatic edges off and on, the better of the two). DTYPE=f32|f64, N=cells per axis."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

n = int(os.environ.get("N", "256"))
dtype = os.environ.get("DTYPE", "f32")
dims = [int(x) for x in os.environ["DIMS"].split(",")] if os.environ.get("DIMS") else [n]
st = cli.build_workload("fdtd", dims)
variants = [("two-kernel staged (default)", False, {}), ("two-kernel lean", False, {"IB_FDTD_KERNEL": "lean"}),
            ("fused default", True, {})]
shapes = ((4, 3), (4, 4), (4, 5), (4, 6), (3, 4), (3, 7), (3, 8), (2, 8), (2, 10)) if dtype == "f32" else ((4, 3), (3, 4), (2, 3), (2, 4), (2, 5), (2, 6), (1, 6))
for fuse in (True, False):
    for tj, ns in shapes:
        variants.append((f"{'fused' if fuse else 'two-kernel'} tj={tj} ns={ns}", fuse,
                         {"IB_FDTD_TJ": tj, "IB_FDTD_STAGES": ns}))
KEYS = ("IB_FDTD_TJ", "IB_FDTD_STAGES", "IB_FDTD_CTAS", "IB_FDTD_CHUNKS", "IB_FDTD_TILES", "IB_FDTD_KERNEL")
for name, fuse, env in variants:
    for k in KEYS:
        os.environ.pop(k, None)
    for k, v in env.items():
        os.environ[k] = str(v)
    try:
        s = wl.DeviceSolver(st, dtype, fuse=fuse)
    except Exception as e:
        print(f"{name}: {e}", flush=True)
        continue
    s.run_batched(20, 5, pdl=True)
    best = None
    for pdl in (False, True):
        xs = []
        for _ in range(3):
            s.flush_l2()
            xs.append(s.run_batched(20, 10, pdl=pdl).gpu_s / 200)
        t = statistics.median(xs)
        best = t if best is None else min(best, t)
    print(f"{dtype} {name:36s} {1e6*best:8.1f} us/iter  {s.iteration_bytes/best/1e9:7.0f} GB/s", flush=True)
    s.close()

"""FDTD 256^3 binary32: two-kernel vs fused leapfrog variants, device-timed (CUDA events)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

n = int(os.environ.get("N", "256"))
st = cli.build_workload("fdtd", [n])
variants = [("two-kernel staged (default)", False, {}), ("two-kernel lean", False, {"IB_FDTD_KERNEL": "lean"}),
            ("fused default", True, {})]
for fuse in (True, False):
    for tj, ns in ((4, 6), (6, 4), (6, 3), (8, 3), (3, 4)):
        variants.append((f"{'fused' if fuse else 'two-kernel'} tj={tj} ns={ns}", fuse,
                         {"IB_FDTD_TJ": tj, "IB_FDTD_STAGES": ns}))
for name, fuse, env in variants:
    for k in ("IB_FDTD_TJ", "IB_FDTD_STAGES", "IB_FDTD_CTAS", "IB_FDTD_CHUNKS", "IB_FDTD_TILES", "IB_FDTD_KERNEL"):
        os.environ.pop(k, None)
    for k, v in env.items():
        os.environ[k] = str(v)
    try:
        s = wl.DeviceSolver(st, "f32", fuse=fuse)
    except Exception as e:
        print(f"{name}: {e}", flush=True)
        continue
    s.run_batched(20, 5, pdl=True)
    xs = []
    for _ in range(3):
        s.flush_l2()
        xs.append(s.run_batched(20, 10, pdl=True).gpu_s / 200)
    t = statistics.median(xs)
    print(f"{name:36s} {1e6*t:8.1f} us/iter  {s.iteration_bytes/t/1e9:7.0f} GB/s", flush=True)
    s.close()

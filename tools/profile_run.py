"""Run a few stream-mode iterations of one config (a short command for ncu to wrap).

    python tools/profile_run.py --workload fdtd --size 256 --iters 3 [--dtype f32]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_09398_b200 import cli  # noqa: E402
from paper_2501_09398_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", required=True)
ap.add_argument("--size", required=True)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--fuse", action="store_true", help="FDTD: the fused one-kernel leapfrog")
ap.add_argument("--graph", type=int, default=0, help="also run a graph of this batch size")
ap.add_argument("--slabs", type=int, default=1, help="axis-0 slabs on device 0 (hotspot, FDTD)")
ap.add_argument("--halo", default="store", help="slab halo exchange: store | copy")
a = ap.parse_args()
state = cli.build_workload(a.workload, [int(x) for x in a.size.split(",")])
s = wl.DeviceSolver(state, a.dtype, fuse=a.fuse, devices=[0] * a.slabs if a.slabs > 1 else None,
                    halo=a.halo)
t = s.run_stream(a.iters)
print(f"{a.workload} {a.size} {a.dtype}: {1e6 * t.gpu_s / a.iters:.2f} us/iter (stream, incl. profiler)")
if a.graph:
    s.run_batched(a.graph, 1, build="capture" if a.slabs > 1 else "manual")
s.close()

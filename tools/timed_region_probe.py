"""Why is a bench step sometimes slower than the same run in the K sweep? (diagnostic)

Replicates bench.py's timed loop for the headline (Hotspot2D 1024^2 binary64, K = 100, PDL): per
step re-upload the inputs, flush L2, run_batched, device time; in rounds with and without the NVML
clock sampler running, with and without the per-step upload. Prints every step's us/iter.
    python tools/timed_region_probe.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

dtype = os.environ.get("DTYPE", "f64")
st = cli.build_workload("hotspot2d", [1024])
n, k = 10000, 100
s = wl.DeviceSolver(st, dtype, devices=[0])
for _ in range(3):
    s.flush_l2()
    s.run_batched(k, n // k, pdl=True)
for rnd in range(3):
    for sampler in (True, False):
        for upload in (True, False):
            xs = []
            ctx = bench.Clocks(0) if sampler else None
            if ctx:
                ctx.__enter__()
            try:
                for _ in range(10):
                    if upload:
                        s.upload(st)
                    s.flush_l2()
                    xs.append(1e6 * s.run_batched(k, n // k, pdl=True).gpu_s / n)
            finally:
                if ctx:
                    ctx.__exit__(None, None, None)
            print(f"round {rnd} sampler={int(sampler)} upload={int(upload)}: mean {statistics.fmean(xs):.3f} "
                  f"median {statistics.median(xs):.3f} max {max(xs):.3f}  "
                  + " ".join(f"{x:.2f}" for x in xs), flush=True)
s.close()

"""Compute side of Hotspot3D 2048x2048x256 strong scaling, measured on ONE B200: the graph
iteration time of one rank's slab at P = 1, 2, 4, 8 (2048/P owned rows + the two halo rows a
rank also reads), run as a single-GPU grid of that shape. Efficiency = T(1) / (P * T(P)) is what
the kernel alone can deliver; the exchange (halo stores fused into the kernel over NVLink) and
the two one-thread ordering kernels per iteration come on top."""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import workloads as wl  # noqa: E402

N, K = 40, 10
rng = np.random.default_rng(7)
print("| P | slab rows (+halo) | graph µs/iter | µs/iter × P | efficiency vs P = 1 |")
print("|---|---|---|---|---|")
t1 = None
for P in (1, 2, 4, 8):
    rows = 2048 // P + (0 if P == 1 else 2)
    shape = (rows, 2048, 256)
    t = rng.random(shape, dtype=np.float32).astype(np.float64)
    st = wl.HotspotWorkload(t, t * 1e-3, 0.1)
    s = wl.DeviceSolver(st, "f32")
    del t, st
    s.run_batched(K, N // K)
    g = []
    for _ in range(3):
        s.flush_l2()
        g.append(s.run_batched(K, N // K).gpu_s / N)
    s.close()
    us = 1e6 * statistics.median(g)
    t1 = t1 or us
    print(f"| {P} | {rows} | {us:.1f} | {us * P:.1f} | {t1 / (us * P):.3f} |", flush=True)

"""Compute side of strong scaling, measured on ONE B200: the graph iteration time of one rank's
slab at P = 1, 2, 4, 8, run as a single-GPU grid of that shape (the slab's owned planes plus the
halo planes a rank also reads). Efficiency = T(1) / (P * T(P)) is what the kernels alone can
deliver; the exchange (halo stores fused into the kernels over NVLink, one system-scope fence per
boundary warp) and the one-thread ordering kernels come on top.
Configs: Hotspot3D 2048x2048x256 (the BASELINE multi-GPU config) and FDTD 256^3 (two half-steps
and the fused leapfrog)."""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import workloads as wl  # noqa: E402


def timed(st, n, k, fuse=False):
    s = wl.DeviceSolver(st, "f32", fuse=fuse)
    s.run_batched(k, n // k)
    g = []
    for _ in range(3):
        s.flush_l2()
        g.append(s.run_batched(k, n // k).gpu_s / n)
    s.close()
    return 1e6 * statistics.median(g)


def table(title, rows_fn, n, k, fuse=False):
    print(f"\n**{title}**\n")
    print("| P | slab planes (+halo) | graph µs/iter | µs/iter × P | efficiency vs P = 1 |")
    print("|---|---|---|---|---|")
    t1 = None
    for P in (1, 2, 4, 8):
        st, planes = rows_fn(P)
        us = timed(st, n, k, fuse)
        del st
        t1 = t1 or us
        print(f"| {P} | {planes} | {us:.1f} | {us * P:.1f} | {t1 / (us * P):.3f} |", flush=True)


rng = np.random.default_rng(7)


def hotspot(P):
    rows = 2048 // P + (0 if P == 1 else 2)
    t = rng.random((rows, 2048, 256), dtype=np.float32).astype(np.float64)
    return wl.HotspotWorkload(t, t * 1e-3, 0.1), rows


def fdtd(P):
    # the lattice has nx + 1 = 257 planes; a rank owns ~257/P of them plus a halo plane each side
    nx = 256 // P + (0 if P == 1 else 2)
    return wl.te101_cavity(nx, 256, 256), nx + 1


what = sys.argv[1:] or ["hotspot3d", "fdtd", "fdtd_fused"]
if "hotspot3d" in what:
    table("Hotspot3D 2048²×256 (binary32, K = 10, N = 40)", hotspot, 40, 10)
if "fdtd" in what:
    table("FDTD 256³, two half-steps (binary32, K = 20, N = 100)", fdtd, 100, 20)
if "fdtd_fused" in what:
    table("FDTD 256³, fused leapfrog (binary32, K = 20, N = 100)", fdtd, 100, 20, fuse=True)

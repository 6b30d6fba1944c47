"""Halo-exchange variants of the single-process slab path on ONE device (all slabs share its SMs,
so this measures the exchange's own cost — extra graph nodes, cross-stream edges, copies — not
scaling): 1 slab vs P slabs with the kernel's fused halo stores (v2) vs peer-copy
faces (v1, IB_HALO_COPY). Device us/iteration, captured graphs, median of 5."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

CASES = [("hotspot3d", [512, 8], 1000, 20), ("hotspot3d", [1024, 1024, 64], 100, 10),
         ("hotspot3d", [2048, 2048, 64], 40, 10), ("fdtd", [256], 100, 20)]
print("| grid | slabs | exchange | graph us/iter | stream us/iter |")
print("|---|---|---|---|---|")
for w, size, n, k in CASES:
    st = cli.build_workload(w, size)
    shape = "x".join(map(str, st.temperature.shape)) if w != "fdtd" else "fdtd " + "x".join(map(str, st.dims))
    for slabs, halo in ((1, "store"), (2, "store"), (2, "copy"), (4, "store"), (4, "copy")):
        s = wl.DeviceSolver(st, "f32", devices=[0] * slabs if slabs > 1 else None, halo=halo)
        try:
            s.run_batched(k, n // k, build="capture")
            g, r = [], []
            for _ in range(5):
                s.flush_l2()
                g.append(s.run_batched(k, n // k, build="capture").gpu_s / n)
                s.flush_l2()
                r.append(s.run_stream(n).gpu_s / n)
            print(f"| {shape} | {slabs} | {'-' if slabs == 1 else halo} | "
                  f"{1e6 * statistics.median(g):.2f} | {1e6 * statistics.median(r):.2f} |", flush=True)
        finally:
            s.close()

"""Problem-size sweep (the paper's speed-up-vs-workload-size view): for each solver and a range of
sizes, graph-mode (best of K in {10, 50, 100}, programmatic edges on/off) vs stream-mode device
time per iteration, and the graph's HBM fraction. Writes gpurun_out/size_sweep_<dtype>.json (DTYPE=f32|f64).
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6527.5
DTYPE = os.environ.get("DTYPE", "f32")
CASES = [("vector", [[2 ** e] for e in (10, 14, 18, 22, 24, 26)], 1000),
         ("hotspot2d", [[n] for n in (128, 256, 512, 1024, 2048, 4096, 8192)], 1000),
         ("hotspot3d", [[n, 8] for n in (64, 128, 256, 512, 1024, 2048)] + [[1024, 1024, 64], [2048, 2048, 64]], 200),
         ("fdtd", [[n] for n in (16, 32, 64, 128, 256, 384)], 100)]


def med(f, reps=3):
    return statistics.median(f() for _ in range(reps))


rows = []
for w, sizes, n in CASES:
    for size in sizes:
        st = cli.build_workload(w, size)
        s = wl.DeviceSolver(st, DTYPE)
        s.run_batched(10, n // 10)

        def stream():
            s.flush_l2()
            return s.run_stream(n).gpu_s

        best = None
        for k in (10, 50, 100):
            for pdl in (False, True):
                def g(k=k, pdl=pdl):
                    s.flush_l2()
                    return s.run_batched(k, n // k, pdl=pdl).gpu_s
                t = med(g)
                if best is None or t < best[0]:
                    best = (t, k, pdl)
        ts = med(stream)
        it = s.iteration_bytes
        row = {"dtype": DTYPE, "workload": w, "size": size, "iterations": n, "graph_us_per_iter": 1e6 * best[0] / n,
               "K": best[1], "pdl": best[2], "stream_us_per_iter": 1e6 * ts / n,
               "speedup": ts / best[0], "hbm_frac": it / (best[0] / n) / 1e9 / PEAK}
        rows.append(row)
        print(f"{w:9s} {str(size):18s} graph {row['graph_us_per_iter']:9.3f}  stream {row['stream_us_per_iter']:9.3f}  "
              f"x{row['speedup']:.2f}  HBM {row['hbm_frac']:.2f}  (K={best[1]}, pdl={best[2]})", flush=True)
        s.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open(f"gpurun_out/size_sweep_{DTYPE}.json", "w"), indent=1)

"""Graph-mode variants on B200: build cost and execution per iteration for every way the runtime
can batch iterations (run under gpurun; writes gpurun_out/graph_modes_<dtype>.json, DTYPE=f32|f64 and prints a table).

  stream            Listing 1: one cudaLaunchKernel per kernel from the C++ loop
  stream+pdl        the same with the programmatic-stream-serialization launch attribute
  manual            Listing 3: cudaGraphCreate + K cudaGraphAddKernelNode, N/K cudaGraphLaunch
  capture           stream capture of the stream-mode sequence instead of explicit nodes
  manual+pdl        programmatic edges between consecutive kernel nodes
  device-launch     instantiated with cudaGraphInstantiateFlagDeviceLaunch (as the paper)
  while             the K-chain inside a conditional WHILE node: ONE cudaGraphLaunch for all batches
  while+pdl         both
  peeled N+7        loop peeling: floor(N/K) replays + one remainder graph (N not divisible by K)
  odd K=25 baked    odd batch on a ping-pong solver: two executables, parity baked into each
  odd K=25 patched  one executable re-pointed with cudaGraphExecKernelNodeSetParams between launches

Device time (CUDA events) per iteration, L2 flushed before each run, median of 5; T_C is the host
build time (create + instantiate + upload).
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

DTYPE = os.environ.get("DTYPE", "f32")
CFGS = [("skeleton 2^14", "vector", [16384], 10000, 100), ("hotspot2d 1024^2", "hotspot2d", [1024], 10000, 80),
        ("hotspot3d 512^2x8", "hotspot3d", [512, 8], 1000, 40), ("fdtd 256^3", "fdtd", [256], 200, 20)]


def main():
    rows = []
    for label, w, size, n, k in CFGS:
        st = cli.build_workload(w, size)
        s = wl.DeviceSolver(st, DTYPE)

        def timed(fn):
            xs, tcs = [], []
            for _ in range(5):
                s.flush_l2()
                t = fn()
                xs.append(t.gpu_s)
                tcs.append(t.build_s)
            return 1e6 * statistics.median(xs), 1e6 * statistics.median(tcs)

        def graph(**kw):
            def f():
                b = s.build_graph(k, **kw)
                r = s.run_graph(n // k)
                s.destroy_graph()
                r.build_s = b.build_s
                return r
            return f

        def graph25(**kw):  # odd K on a ping-pong solver: two executables vs one re-pointed one
            def f():
                b = s.build_graph(25, pdl=True, **kw)
                r = s.run_graph(n // 25)
                s.destroy_graph()
                r.build_s = b.build_s
                return r
            return f

        modes = [
            ("stream", lambda: s.run_stream(n)),
            ("stream+pdl", lambda: s.run_stream(n, pdl=True)),
            ("manual", graph()),
            ("capture", graph(build="capture")),
            ("manual+pdl", graph(pdl=True)),
            ("device-launch", graph(device_launch=True)),
            ("while", graph(while_loop=True)),
            ("while+pdl", graph(while_loop=True, pdl=True)),
            ("peeled N+7", lambda: s.run_peeled(n + 7, k)),
            ("odd K=25 baked", graph25()),
            ("odd K=25 patched", graph25(patch=True)),
        ]
        timed(modes[2][1])  # warm-up
        for name, fn in modes:
            t, tc = timed(fn)
            iters = n + 7 if name.startswith("peeled") else n
            row = {"config": label, "K": k, "N": iters, "mode": name, "us_per_iter": t / iters,
                   "T_C_us": tc if not name.startswith("stream") else 0.0}
            rows.append(row)
            print(f"{label:18s} K={k:<4d} {name:14s} {row['us_per_iter']:8.3f} us/iter  T_C {row['T_C_us']:9.1f} us",
                  flush=True)
        s.close()
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", f"graph_modes_{DTYPE}.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()

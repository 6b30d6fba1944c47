"""Per-kernel launch gaps from Nsight Systems (the paper's own evidence).

  --run CONFIG MODE   run one workload under `nsys profile --cuda-graph-trace=node`:
                      MODE stream | graph | graph_pdl (K from the bench's sweep)
  --analyze DIR       read DIR/<config>_<mode>_cuda_gpu_trace.csv (nsys stats -r cuda_gpu_trace)
                      and print the gap table (markdown)

Gap = start of kernel k+1 minus end of kernel k on the device, for the solver's kernels only,
after dropping the first 10% (warm-up). Stream mode: every gap is t_b. Graph mode: gaps inside
a K-node graph are t_i, the gap between the last node of one graph and the first of the next is
t_a (model.py:48-74). With programmatic edges t_i is negative: kernel k+1 starts
before kernel k ends. tools/nsys_run.sh drives the whole capture on the GPU box.
"""
import csv
import glob
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CONFIGS = {  # name: (workload, size, iterations, K)
    "skeleton": ("vector", [16384], 2000, 20),
    "hotspot2d": ("hotspot2d", [1024], 2000, 80),
    "hotspot3d": ("hotspot3d", [512, 8], 1000, 20),
    "fdtd": ("fdtd", [256], 200, 20),
}


def run(name: str, mode: str) -> None:
    from paper_2501_09398_b200 import cli, workloads as wl

    w, size, n, k = CONFIGS[name]
    st = cli.build_workload(w, size)
    s = wl.DeviceSolver(st, "f32")
    if mode == "stream":
        s.run_stream(n)
    else:
        s.run_batched(k, n // k, pdl=(mode == "graph_pdl"))
    s.sync()
    s.close()


def _rows(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.strip()]
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"Start') or ln.startswith("Start"))
    return list(csv.DictReader(lines[start:]))


def analyze(d: str) -> None:
    print("| config | mode | kernels | K | median gap in graph t_i / stream t_b (µs) | p10–p90 | "
          "median gap between graphs t_a (µs) | median kernel t_k (µs) | mean start-to-start per "
          "iteration (µs) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for name, (_, _, n, k) in CONFIGS.items():
        for mode in ("stream", "graph", "graph_pdl"):
            paths = glob.glob(os.path.join(d, f"{name}_{mode}_cuda_gpu_trace.csv"))
            if not paths:
                continue
            rows = _rows(paths[0])
            key_s = next(c for c in rows[0] if c.startswith("Start"))
            key_d = next(c for c in rows[0] if c.startswith("Duration"))
            key_n = "Name"
            unit = 1e-3 if "(ns)" in key_s else 1.0  # -> us
            ks = [(float(r[key_s]) * unit, float(r[key_d]) * unit) for r in rows
                  if r.get(key_n, "").find("ib::k_") >= 0 and "k_flush" not in r[key_n]]
            ks.sort()
            per_it = 2 if name == "fdtd" else 1
            nodes = k * per_it
            skip = len(ks) // 10
            skip -= skip % nodes  # start at a graph boundary
            gaps_i, gaps_a = [], []
            for j in range(skip, len(ks) - 1):
                gap = ks[j + 1][0] - (ks[j][0] + ks[j][1])
                if mode != "stream" and (j + 1) % nodes == 0:
                    gaps_a.append(gap)
                else:
                    gaps_i.append(gap)
            if not gaps_i:
                continue
            q = statistics.quantiles(gaps_i, n=10)
            ta = f"{statistics.median(gaps_a):.2f}" if gaps_a else "—"
            tk = statistics.median(dur for _, dur in ks[skip:])
            period = (ks[-1][0] - ks[skip][0]) / (len(ks) - 1 - skip) * per_it
            print(f"| {name} | {mode} | {len(ks)} | {k if mode != 'stream' else '—'} | "
                  f"{statistics.median(gaps_i):.2f} | {q[0]:.2f} – {q[-1]:.2f} | {ta} | {tk:.2f} | "
                  f"{period:.2f} |")


if __name__ == "__main__":
    if sys.argv[1] == "--run":
        run(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "--analyze":
        analyze(sys.argv[2])
    else:
        raise SystemExit(__doc__)

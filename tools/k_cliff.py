"""Is the Hotspot2D K = 200-250 slowdown real, and where does it come from?

    python tools/k_cliff.py [--dtype f32] [--reps 12] [--procs 3] > gpurun_out/k_cliff.json

Runs P fresh processes; each builds ONE DeviceSolver for Hotspot2D 1024^2 (N = 10^4) and measures,
in interleaved round-robin order (so a slow phase of the box hits every K alike), for each
K in KS x {plain, PDL}:
  * full run T_C + T_E (device events, L2 flushed before) - what bench.py's pick_k ranks;
  * T_E of a prebuilt executable (run_graph), so build cost and execution can be told apart;
  * the graph's device-memory footprint (IB_FLAG_MEMINFO build, outside the timed runs);
  * the SM clock (NVML) sampled right after each run.
Prints one JSON object per process and a summary (median / min / max / bimodality) per K.
Diagnostic tooling, not product.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KS = [50, 80, 100, 125, 200, 250, 400, 500]
N = 10000


def child(dtype: str, reps: int) -> dict:
    import numpy as np  # noqa: F401

    from paper_2501_09398_b200 import cli
    from paper_2501_09398_b200 import workloads as wl

    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        clk = lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)  # noqa: E731
    except Exception:  # noqa: BLE001
        clk = lambda: None  # noqa: E731
    state = cli.build_workload("hotspot2d", [1024])
    s = wl.DeviceSolver(state, dtype, devices=[0])
    out = {"pid": os.getpid(), "dtype": dtype, "full": {}, "exec": {}, "mem": {}, "clk": {}}
    try:
        for pdl in (False, True):  # first-instantiate growth paid up front (as bench.py does)
            s.build_graph(max(KS), pdl=pdl)
            s.destroy_graph()
        for k in KS:
            for pdl in (False, True):
                t = s.build_graph(k, pdl=pdl, meminfo=True)
                out["mem"][f"{k}{'p' if pdl else ''}"] = t.graph_bytes
                s.destroy_graph()
        for _ in range(reps):
            for k in KS:
                for pdl in (False, True):
                    key = f"{k}{'p' if pdl else ''}"
                    s.flush_l2()
                    t = s.run_batched(k, N // k, pdl=pdl)
                    out["full"].setdefault(key, []).append(1e6 * t.gpu_s / N)
                    out["clk"].setdefault(key, []).append(clk())
                    s.build_graph(k, pdl=pdl)
                    s.flush_l2()
                    e = s.run_graph(N // k)
                    out["exec"].setdefault(key, []).append(1e6 * e.gpu_s / N)
                    s.destroy_graph()
    finally:
        s.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--reps", type=int, default=12)
    ap.add_argument("--procs", type=int, default=3)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(child(a.dtype, a.reps)))
        return
    runs = []
    for _ in range(a.procs):
        p = subprocess.run([sys.executable, __file__, "--child", "--dtype", a.dtype, "--reps", str(a.reps)],
                           capture_output=True, text=True, timeout=900)
        if p.returncode != 0:
            print(p.stderr[-2000:], file=sys.stderr)
            continue
        runs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    summary = {}
    for key in runs[0]["full"] if runs else []:
        full = [v for r in runs for v in r["full"][key]]
        ex = [v for r in runs for v in r["exec"][key]]
        med = statistics.median(full)
        summary[key] = {
            "full_median": round(med, 4), "full_min": round(min(full), 4), "full_max": round(max(full), 4),
            "slow_fraction": round(sum(v > 1.15 * min(full) for v in full) / len(full), 3),
            "per_process_median": [round(statistics.median(r["full"][key]), 4) for r in runs],
            "exec_median": round(statistics.median(ex), 4), "exec_max": round(max(ex), 4),
            "graph_bytes": [r["mem"].get(key) for r in runs],
            "sm_mhz": sorted({c for r in runs for c in r["clk"][key] if c is not None}),
        }
    print(json.dumps({"dtype": a.dtype, "reps": a.reps, "procs": len(runs), "summary": summary,
                      "runs": runs}))


if __name__ == "__main__":
    main()

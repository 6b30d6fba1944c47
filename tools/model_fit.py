"""Fit the paper's performance model to B200 sweeps with the REFERENCE's own code (build container).

    python tools/model_fit.py gpurun_out/evidence --round r01

Reads each sweep_<config>/{creation,execution,stream}.csv written by
``python -m paper_2501_09398_b200 sweep`` (the reference measurement schema) and the measured
constants in trace_<config>.json, then runs — unchanged, imported read-only from
/root/reference/pkg/src — ``fitting.fit_creation`` / ``fit_execution`` (with the 25% validity
filter), ``optimize.recommend_from_coefficients`` and ``model.measured_speedup``. Writes
profiles/<round>_model_fit.md. This is analysis tooling, not part of the product or its tests.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from iterbatch.fileio import parse_measurements  # noqa: E402
from iterbatch.fitting import fit_creation, fit_execution, fit_validity_filter  # noqa: E402
from iterbatch.model import SampleStats, measured_speedup  # noqa: E402
from iterbatch.optimize import recommend_from_coefficients  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = [("skeleton", 10000, "vector 2^14"), ("skeleton_pdl", 10000, "vector 2^14, PDL edges"),
           ("hotspot2d", 10000, "Hotspot2D 1024^2"), ("hotspot3d", 1000, "Hotspot3D 512x512x8"),
           ("fdtd", 2000, "FDTD 256^3 (2 kernels / iteration)"),
           ("fdtd_fused", 2000, "FDTD 256^3 fused (1 kernel / iteration)")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("evidence")
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    out = [f"# Performance-model fit on B200 ({a.round})", "",
           "Sweeps: `python -m paper_2501_09398_b200 sweep` (binary32, 5 repeats per K, every divisor of "
           "I_k up to 25% of I_k, host wall-clock T_C and T_E as in the paper; the driver's one-time "
           "graph-memory growth paid before the sweep; odd K on the ping-pong solvers builds ONE executable "
           "re-pointed per launch (`IB_FLAG_PATCH`), so T_C is one K-node graph as the linear creation "
           "model assumes). Fits and the optimum are "
           "computed by the reference's own `fit_creation`, `fit_execution` (validity filter 0.25 I_k, "
           "`fitting.py:104-134`) and `recommend_from_coefficients` (`optimize.py:135-165`), unchanged.", "",
           "| config | k_c (s/node) | b_c (s) | a (s·node) | b (s) | exec MAE (s) | K* (reference optimizer) | "
           "continuous sqrt(a/k_c) | predicted speed-up | measured best K (T_C+T_E) | measured speed-up at K* |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for key, total, label in CONFIGS:
        d = os.path.join(a.evidence, f"sweep_{key}")
        if not os.path.isdir(d):
            continue
        cre = fit_validity_filter(parse_measurements(os.path.join(d, "creation.csv")), 0.25, total)
        exe = fit_validity_filter(parse_measurements(os.path.join(d, "execution.csv")), 0.25, total)
        cf, ef = fit_creation(cre), fit_execution(exe)
        rec = recommend_from_coefficients(cf.slope, cf.intercept, ef.slope, ef.intercept, total)
        stream = {p.batch_size: p for p in parse_measurements(os.path.join(d, "stream.csv")).points}
        graph = {p.batch_size: p for p in exe.points}
        creat = {p.batch_size: p for p in cre.points}
        best_k = min(graph, key=lambda k: graph[k].mean() + creat[k].mean())
        k = rec.batch_size if rec.batch_size in graph else best_k
        tot = SampleStats.from_samples([g + c for g, c in zip(graph[k].samples, creat[k].samples)])
        sp = measured_speedup(SampleStats.from_samples(stream[k].samples), tot)
        cont = math.sqrt(ef.slope / cf.slope) if cf.slope > 0 and ef.slope > 0 else float("nan")
        out.append(f"| {label} | {cf.slope:.3e} | {cf.intercept:.3e} | {ef.slope:.3e} | {ef.intercept:.3e} | "
                   f"{ef.mae:.2e} | {rec.batch_size} | {cont:.1f} | {rec.predicted_speedup:.3f} | {best_k} | "
                   f"{sp.ratio:.3f} ± {sp.error:.3f} |")
    out += ["", "A100 (paper Table I, `PAPER.md:286-291`, 1e3 threads): k_c = 4.18e-6, b_c = 1.59e-4, "
            "a = 1.77e-2, b = 4.56e-2, S* = 80 (reference optimizer), predicted speed-up 1.367.", ""]
    traces = []
    for key, _, label in CONFIGS:
        p = os.path.join(a.evidence, f"trace_{key}.json")
        if os.path.exists(p):
            t = json.loads(open(p).read().strip().splitlines()[-1])
            traces.append(f"| {label} | {t['t_k']*1e6:.2f} | {t['t_i']*1e6:.2f} | {t['t_a']*1e6:.2f} | "
                          f"{t['t_b']*1e6:.2f} | {t['t_l']*1e6:.2f} | {t['k_c']*1e6:.2f} | {t['b_c']*1e6:.1f} |")
    if traces:
        out += ["## Measured timeline constants (CUPTI trace, `python -m paper_2501_09398_b200 trace`)", "",
                "Medians over one traced graph run (K = 100) and one traced stream run; µs. Observation I "
                "of the paper (`PAPER.md:208`) holds when t_i < t_a.", "",
                "| config | t_k | t_i (in-graph gap) | t_a (between graphs) | t_b (stream gap) | t_l (incl. CUPTI first-launch setup) | k_c | b_c |",
                "|---|---|---|---|---|---|---|---|"] + traces
    path = os.path.join(ROOT, "profiles", f"{a.round}_model_fit.md")
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()

"""Fit the paper's performance model to B200 measurements with the REFERENCE's own code.

    python tools/model_fit.py gpurun_out/evidence --round r02

Reads each sweep_<config>/{creation,execution,stream,total}.csv written by
``python -m paper_2501_09398_b200 sweep`` (the reference measurement schema) and each
trace_<config>/{graph_trace.csv,stream_trace.csv,params.txt} written by ``... trace``. Then, with
the reference package imported read-only (baseline/_ref, else /root/reference/pkg/src), unchanged:

* ``fitting.fit_creation`` / ``fit_execution`` (25% validity filter) and
  ``optimize.recommend_from_coefficients`` on the sweeps;
* ``iterbatch optimize --params params.txt --iterations I_K [--mem-cap B]`` (the reference CLI,
  cli.py:155-169) on the measured params file, with and without a memory cap;
* ``iterbatch speedup --baseline stream.csv --graph total.csv`` (cli.py:233-250);
* ``iterbatch simulate --params params.txt`` at the recommended K, against the measured total;
* ``fileio.parse_trace_csv`` + ``simulate.trace_summary`` on the real traces.

Writes profiles/<round>_model_fit.md. Analysis tooling, not product.
"""

from __future__ import annotations

import argparse
import contextlib
import io
import json
import math
import os
import statistics
import sys

sys.dont_write_bytecode = True
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "iterbatch")):
        sys.path.insert(0, cand)
        break

from iterbatch import cli as rcli  # noqa: E402
from iterbatch.fileio import parse_measurements, parse_params, parse_trace_csv  # noqa: E402
from iterbatch.fitting import fit_creation, fit_execution, fit_validity_filter  # noqa: E402
from iterbatch.model import BatchPlan, SampleStats, measured_speedup  # noqa: E402
from iterbatch.optimize import recommend_from_coefficients  # noqa: E402
from iterbatch.simulate import EventTrace, TraceMode, trace_summary  # noqa: E402

CONFIGS = [("skeleton", 10000, "vector 2^14 (binary32)"),
           ("hotspot2d_f64", 10000, "Hotspot2D 1024^2 (binary64)"),
           ("hotspot2d", 10000, "Hotspot2D 1024^2 (binary32)"),
           ("hotspot3d", 1000, "Hotspot3D 512x512x8 (binary32)"),
           ("fdtd", 2000, "FDTD 256^3, 2 kernels / iteration (binary32)"),
           ("fdtd_fused", 2000, "FDTD 256^3 fused, 1 kernel / iteration (binary32)")]


def ref_cli(*argv) -> tuple[int, str, str]:
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = rcli.main(list(argv))
    return code, out.getvalue().strip(), err.getvalue().strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("evidence")
    ap.add_argument("--round", default="r02")
    a = ap.parse_args()
    ev = a.evidence
    out = [f"# Performance-model fit on B200 ({a.round})", "",
           "Sweeps: `python -m paper_2501_09398_b200 sweep` (5 repeats per K, host wall-clock T_C and T_E as "
           "in the paper; odd K on the ping-pong solvers re-points ONE executable (`IB_FLAG_PATCH`) so T_C "
           "is one K-node graph). Traces: `python -m paper_2501_09398_b200 trace` (CUPTI kernel records + "
           "host events on the CUPTI clock; the first two launches of the traced executable, whose nodes "
           "CUPTI instruments on first launch, are dropped; FDTD's two launches per iteration are one model "
           "'kernel'; t_l from idle-device launches timed with CUDA events and no profiler attached, the "
           "CUPTI-timed value beside it; k_c / b_c a least-squares fit of "
           "the whole build time T_C at four batch sizes — the phases fit_creation uses; m_base / m_node a "
           "fit of the device memory a built graph holds at 1000-8000 iterations, where cudaMemGetInfo's "
           "2 MiB steps resolve it). Everything below is computed by "
           "the reference package itself (`tools/model_fit.py`), unchanged.", "",
           "## Sweep fits (reference `fit_creation` / `fit_execution`, validity filter 0.25 I_k, "
           "`recommend_from_coefficients`)", "",
           "| config | k_c (s/iter) | b_c (s) | a (s·iter) | b (s) | exec MAE (s) | K* | predicted speed-up | "
           "measured best K (T_C+T_E) | `iterbatch speedup` at K* (stream / total) |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for key, total, label in CONFIGS:
        d = os.path.join(ev, f"sweep_{key}")
        if not os.path.isdir(d):
            continue
        cre = fit_validity_filter(parse_measurements(os.path.join(d, "creation.csv")), 0.25, total)
        exe = fit_validity_filter(parse_measurements(os.path.join(d, "execution.csv")), 0.25, total)
        cf, ef = fit_creation(cre), fit_execution(exe)
        rec = recommend_from_coefficients(cf.slope, cf.intercept, ef.slope, ef.intercept, total)
        graph = {p.batch_size: p for p in exe.points}
        creat = {p.batch_size: p for p in cre.points}
        best_k = min(graph, key=lambda k: graph[k].mean() + creat[k].mean())
        k = rec.batch_size if rec.batch_size in graph else best_k
        sp = "n/a"
        tot_csv = os.path.join(d, "total.csv")
        if os.path.exists(tot_csv):
            code, txt, _ = ref_cli("speedup", "--baseline", os.path.join(d, "stream.csv"), "--graph", tot_csv)
            sizes = [p.batch_size for p in parse_measurements(tot_csv).points]
            if code == 0 and k in sizes:
                ratio, err = txt.splitlines()[sizes.index(k)].split(",")
                sp = f"{float(ratio):.3f} ± {float(err):.3f}"
        else:
            stream = {p.batch_size: p for p in parse_measurements(os.path.join(d, "stream.csv")).points}
            tot = SampleStats.from_samples([g + c for g, c in zip(graph[k].samples, creat[k].samples)])
            s = measured_speedup(SampleStats.from_samples(stream[k].samples), tot)
            sp = f"{s.ratio:.3f} ± {s.error:.3f}"
        out.append(f"| {label} | {cf.slope:.3e} | {cf.intercept:.3e} | {ef.slope:.3e} | {ef.intercept:.3e} | "
                   f"{ef.mae:.2e} | {rec.batch_size} | {rec.predicted_speedup:.3f} | {best_k} | {sp} |")
    out += ["", "A100 (paper Table I, `PAPER.md:286-291`): k_c = 4.18e-6, b_c = 1.59e-4, a = 1.77e-2, b = 4.56e-2, "
            "S* = 80, predicted speed-up 1.367.", ""]

    rows, opt_rows, sim_rows, rt_rows = [], [], [], []
    for key, total, label in CONFIGS:
        d = os.path.join(ev, f"trace_{key}")
        js = os.path.join(ev, f"trace_{key}.json")
        if not os.path.isdir(d) or not os.path.exists(js):
            continue
        t = json.loads(open(js).read().strip().splitlines()[-1])
        params_path = os.path.join(d, "params.txt")
        params, memory = parse_params(params_path)
        rows.append(f"| {label} | {t['t_k']*1e6:.2f} | {t['t_i']*1e6:.2f} | {t['t_a']*1e6:.2f} | "
                    f"{t['t_b']*1e6:.2f} | {t['t_l']*1e6:.2f} | {t.get('t_l_cupti', float('nan'))*1e6:.2f} | "
                    f"{t['k_c']*1e6:.3f} | {t['b_c']*1e6:.1f} | {t['k_c_node_add']*1e6:.2f} | "
                    f"{memory.base_bytes} | {memory.bytes_per_node} |")
        _, rec_txt, _ = ref_cli("optimize", "--params", params_path, "--iterations", str(total))
        k_star = int(rec_txt.split(",")[0]) if rec_txt else None  # recommendation_line: K,I,T,speedup,cont
        # a memory cap that binds: the bytes of a graph of K*/4 iterations
        cap = None
        if k_star:
            cap = memory.base_bytes + memory.bytes_per_node * max(1, k_star // 4)
            _, cap_txt, cap_err = ref_cli("optimize", "--params", params_path, "--iterations", str(total),
                                          "--mem-cap", str(cap))
        else:
            cap_txt = cap_err = ""
        opt_rows.append(f"| {label} | `{rec_txt}` | {cap} | `{cap_txt or cap_err}` |")
        # simulate the recommended plan with the measured constants, against the measured total
        sw = os.path.join(ev, f"sweep_{key}", "total.csv")
        if k_star and os.path.exists(sw):
            pts = {p.batch_size: p for p in parse_measurements(sw).points}
            kk = k_star if k_star in pts else min(pts, key=lambda x: abs(x - k_star))
            code, sim_txt, sim_err = ref_cli("simulate", "--params", params_path, "--iterations", str(total),
                                             "--batch-size", str(kk))
            sim_total = float(sim_txt.split(",")[2]) if code == 0 else None  # summary_line: T_C,T_E,T
            meas = statistics.fmean(pts[kk].samples)
            sim_rows.append(f"| {label} | {kk} | `{sim_txt or sim_err}` | {meas:.6f} | "
                            + (f"{sim_total / meas:.3f} |" if sim_total else "n/a |"))
        # real traces through the reference's own reader and summary
        for mode in ("graph", "stream"):
            path = os.path.join(d, f"{mode}_trace.csv")
            events = parse_trace_csv(path)
            size = 1 + max(e.kernel_index for e in events if e.kernel_index is not None)
            num = 1 + max(e.batch_index for e in events if e.batch_index is not None)
            plan = BatchPlan(size * num, size, num)
            summ = trace_summary(EventTrace(events, TraceMode.GRAPH if mode == "graph" else TraceMode.BASELINE,
                                            plan, params))
            rt_rows.append(f"| {label} | {mode} | {len(events)} | {summ.creation_span:.6f} | "
                           f"{summ.execution_span:.6f} | {summ.total:.6f} |")
    if rows:
        out += ["## Measured platform constants (`trace`; µs unless stated)", "",
                "Observation I of the paper (`PAPER.md:208`) holds when t_i < t_a.", "",
                "| config | t_k (per iteration) | t_i (in-graph gap) | t_a (between graphs) | t_b (stream gap) | "
                "t_l (idle launch, no profiler: CUDA events) | t_l (idle launch, CUPTI) | k_c (T_C fit, per iteration) | b_c | node-add interval "
                "| m_base (B) | m_node (B/iteration) |",
                "|---|---|---|---|---|---|---|---|---|---|---|---|"] + rows + [""]
        out += ["## `iterbatch optimize` (reference CLI) on the measured params files", "",
                "| config | `optimize --params params.txt --iterations I_k` | --mem-cap (bytes of a K*/4 graph) | "
                "`optimize ... --mem-cap` |", "|---|---|---|---|"] + opt_rows + [""]
        out += ["## `iterbatch simulate` with the measured constants vs the measured total (sweep)", "",
                "| config | K | `simulate --params ... --batch-size K` | measured T_C+T_E (s) | simulated / measured |",
                "|---|---|---|---|---|"] + sim_rows + [""]
        out += ["## Real traces through the reference reader (`parse_trace_csv` + `trace_summary`)", "",
                "| config | trace | events | creation span (s) | execution span (s) | total (s) |",
                "|---|---|---|---|---|---|"] + rt_rows + [""]
    path = os.path.join(ROOT, "profiles", f"{a.round}_model_fit.md")
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()

"""B200 measurements read back by the REFERENCE's own readers and model.

tests/golden/b200_fit/ holds a small canned output of this repo's ``sweep`` and ``trace`` commands
recorded on a B200 (Hotspot2D 1024^2 binary64, I_k = 200; tools/evidence_fit.sh, the ``canned``
lines): the four measurement CSVs, the graph / stream traces and the params file. They must go
through the unmodified reference package — parse_measurements + fit_creation / fit_execution
(fileio.py:128, fitting.py:104-134), parse_trace_csv + trace_summary (fileio.py:205,
simulate.py:161-192), parse_params + MemoryModel (fileio.py:70-125, model.py:130-142) and the
``optimize`` / ``speedup`` / ``simulate`` subcommands (cli.py:140-169,233-250) — with no adaptor.
The reference is imported from baseline/_ref (build()) or /root/reference; skipped when neither
exists (the GPU box has neither). Also checks the writer side on synthetic data: the product's
``write_trace_csv`` / ``write_params`` / ``derive_parameters`` (paper_2501_09398_b200/trace.py).
"""

import contextlib
import io
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "b200_fit")


def _ref():
    for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "iterbatch")):
            if cand not in sys.path:
                sys.path.append(cand)
            import iterbatch  # noqa: F401

            return True
    return False


needs_ref = pytest.mark.skipif(not _ref(), reason="reference package not present (baseline/_ref or /root/reference)")


def _cli(*argv):
    from iterbatch import cli as rcli

    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = rcli.main(list(argv))
    return code, out.getvalue().strip(), err.getvalue().strip()


@needs_ref
def test_sweep_csvs_fit_with_the_reference():
    from iterbatch.fileio import parse_measurements
    from iterbatch.fitting import fit_creation, fit_execution

    series = {k: parse_measurements(os.path.join(FIX, f"{k}.csv"))
              for k in ("creation", "execution", "stream", "total")}
    sizes = [p.batch_size for p in series["creation"].points]
    assert sizes == [2, 4, 10, 20, 50]
    for s in series.values():
        assert all(len(p.samples) == 5 and min(p.samples) > 0 for p in s.points)
    c = fit_creation(series["creation"])
    e = fit_execution(series["execution"])
    # T_C grows with the node count; T_E falls with the batch size (fewer graph launches)
    assert c.slope > 0 and e.slope > 0
    assert np.isfinite([c.slope, c.intercept, e.slope, e.intercept]).all()
    for kind in ("creation", "execution"):
        code, out, err = _cli("fit", "--input", os.path.join(FIX, f"{kind}.csv"), "--kind", kind,
                              "--total-iterations", "200")
        assert code == 0 and out, err
    code, out, err = _cli("speedup", "--baseline", os.path.join(FIX, "stream.csv"),
                          "--graph", os.path.join(FIX, "total.csv"))
    assert code == 0, err
    ratios = [float(line.split(",")[0]) for line in out.splitlines()]
    assert len(ratios) == 5
    speed = max(ratios)
    assert speed > 1.0  # graph batching wins at this launch-bound size


@needs_ref
def test_real_traces_summarise_with_the_reference():
    from iterbatch.fileio import parse_params, parse_trace_csv
    from iterbatch.model import BatchPlan
    from iterbatch.simulate import EventKind, EventTrace, TraceMode, trace_summary

    params, _ = parse_params(os.path.join(FIX, "params.txt"))
    for name, mode in (("graph_trace.csv", TraceMode.GRAPH), ("stream_trace.csv", TraceMode.BASELINE)):
        events = parse_trace_csv(os.path.join(FIX, name))
        started = sum(e.kind is EventKind.KERNEL_STARTED for e in events)
        ended = sum(e.kind is EventKind.KERNEL_ENDED for e in events)
        assert started == ended == 200  # every kernel of the I_k = 200 run, once
        size = 1 + max(e.kernel_index for e in events if e.kernel_index is not None)
        num = 1 + max(e.batch_index for e in events if e.batch_index is not None)
        plan = BatchPlan(size * num, size, num)
        s = trace_summary(EventTrace(events, mode, plan, params))  # validates order and indices
        assert s.execution_span > 0 and s.total >= s.execution_span
        if mode is TraceMode.GRAPH:
            assert (size, num) == (20, 10)
            assert 0 < s.creation_span < s.execution_span
            launches = sum(e.kind is EventKind.GRAPH_LAUNCHED for e in events)
            assert launches == num
        else:
            assert s.creation_span == 0.0
    g = trace_summary(EventTrace(parse_trace_csv(os.path.join(FIX, "graph_trace.csv")), TraceMode.GRAPH,
                                 BatchPlan(200, 20, 10), params))
    b_events = parse_trace_csv(os.path.join(FIX, "stream_trace.csv"))
    b = trace_summary(EventTrace(b_events, TraceMode.BASELINE, BatchPlan(200, 1, 200), params))
    assert g.execution_span < b.execution_span  # the graph's execution beats per-kernel launches


@needs_ref
def test_params_file_drives_the_reference_optimizer():
    from iterbatch.fileio import parse_params

    path = os.path.join(FIX, "params.txt")
    params, memory = parse_params(path)
    assert 0 < params.kernel_time < 1e-3 and 0 <= params.intra_graph_gap < params.inter_graph_gap
    assert params.creation_per_node > 0 and memory is not None
    code, out, err = _cli("optimize", "--params", path, "--iterations", "200")
    assert code == 0, err
    k_star = int(out.split(",")[0])
    assert 200 % k_star == 0
    code, out, err = _cli("simulate", "--params", path, "--iterations", "200", "--batch-size", str(k_star))
    assert code == 0, err
    creation, execution, total = (float(x) for x in out.split(","))
    assert creation > 0 and execution > 0 and abs(total - creation - execution) < 3e-9  # 9-decimal output


def test_writers_emit_the_reference_schema(tmp_path):
    """The product's trace writer / params writer / parameter derivation on a synthetic timeline
    (no GPU): 3 batches of 4 two-kernel iterations."""
    from paper_2501_09398_b200 import trace as tr

    kpi, size, num = 2, 4, 3
    kern, t = [], 1e-3
    for b in range(num):
        for i in range(size * kpi):
            kern.append((t, t + 10e-6))
            t += 10e-6 + (0.2e-6 if i + 1 < size * kpi else 6e-6)
    kern = np.asarray(kern)
    events = [(0.0, "node_added", None, k) for k in range(size * kpi)]
    events += [(2e-4, "graph_instantiated", None, None), (3e-4, "graph_uploaded", None, None)]
    for b in range(num):
        events.append((kern[b * size * kpi, 0] - 5e-6, "graph_launched", b, None))
    for idx, (a, e) in enumerate(kern):
        bi, ki = divmod(idx, size * kpi)
        events += [(a, "kernel_started", bi, ki), (e, "kernel_ended", bi, ki)]
    events.sort(key=lambda x: x[0])
    g = tr.RealTrace("graph", size * kpi, num, events, kern)
    s_k = np.asarray([(1e-3 + i * 12e-6, 1e-3 + i * 12e-6 + 10e-6) for i in range(size * kpi * num)])
    st = tr.RealTrace("baseline", 1, len(s_k), [], s_k)
    p = tr.derive_parameters(g, st, kernels_per_iteration=kpi)
    assert p["t_k"] == pytest.approx(20.2e-6)  # one iteration: H, 0.2 us gap, E
    assert p["t_i"] == pytest.approx(0.2e-6) and p["t_a"] == pytest.approx(6e-6)
    assert p["t_b"] == pytest.approx(2e-6)  # iteration-to-iteration gap of the stream run
    path = tmp_path / "params.txt"
    p.update({"t_l": 2e-5, "k_c": 2e-6, "b_c": 8e-5})
    tr.write_params(path, p, {"m_base": 4096, "m_node": 2048})
    text = path.read_text().splitlines()
    assert text[0] == "# schema=1"
    keys = [ln.split("=")[0].strip() for ln in text if "=" in ln and not ln.startswith("#")]
    assert keys == ["t_k", "t_i", "t_a", "t_l", "t_b", "k_c", "b_c", "m_base", "m_node"]
    csv = tmp_path / "graph_trace.csv"
    tr.write_trace_csv(g, csv)
    lines = csv.read_text().splitlines()
    assert lines[:2] == ["# schema=1", tr.TRACE_HEADER]
    assert len(lines) == 2 + len(events)
    if _ref():
        from iterbatch.fileio import parse_params, parse_trace_csv

        params, memory = parse_params(path)
        assert params.kernel_time == pytest.approx(20.2e-6, rel=1e-6)
        assert memory.base_bytes == 4096 and memory.bytes_per_node == 2048
        assert len(parse_trace_csv(csv)) == len(events)

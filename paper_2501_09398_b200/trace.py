"""Real B200 timelines in the reference's EventTrace schema, and the timing parameters they imply.

The reference only *simulates* the Fig. 1 timelines (pkg/src/iterbatch/simulate.py:28-125) and
reads measured platform constants from a ``key = value`` params file (fileio.py:34-45,70-125).
This module records the real thing:

* ``capture_graph`` / ``capture_stream`` arm the runtime's trace (``ib_trace_enable``): CUPTI
  activity records give every solver kernel's [start, end] (the mechanism nsys uses; the kernels
  carry no instrumentation), and the host events of the build and launch calls are stamped on the
  same CUPTI timebase;
* ``write_trace_csv`` writes them in the reference trace-CSV schema (``# schema=1``,
  ``timestamp,kind,batch_index,kernel_index``, 9-decimal seconds, fileio.py:48,193-205), with the
  clock starting at zero at the build start as the simulator's does; ``iterbatch``'s
  ``parse_trace_csv`` / ``trace_summary`` read it unchanged;
* ``derive_parameters`` reduces a graph trace and a stream trace to the model's constants
  t_k, t_i, t_a, t_l, t_b (model.py:48-74), k_c, b_c from the build events, and
  ``write_params`` writes the params file ``iterbatch optimize`` consumes.
"""

from __future__ import annotations

import ctypes
import math
import statistics
from dataclasses import dataclass

import numpy as np

from . import _lib

# reference EventKind values (simulate.py:28-36), indexed by the runtime's IB_EV_* codes
KIND = {
    0: "node_added",
    1: "graph_instantiated",
    2: "graph_uploaded",
    3: "graph_launched",
    4: "kernel_started",
    5: "kernel_ended",
    6: "batch_gap_started",
    7: "baseline_kernel_launched",
}
BUILD_STARTED = 100
TRACE_HEADER = "timestamp,kind,batch_index,kernel_index"


@dataclass
class RealTrace:
    """Events as (seconds since the build/run start, kind, batch_index | None, kernel_index | None)."""

    mode: str  # "graph" | "baseline"
    batch_size: int  # nodes per batch (kernels per graph launch); 1 for baseline
    num_batches: int
    events: list
    kernels: np.ndarray  # (n, 2) kernel [start, end] seconds on the same clock


def _arm(solver, capacity: int) -> None:
    _lib.check(_lib.lib().ib_trace_enable(solver.ctx, int(capacity)))


def _arm_warm(solver, capacity: int) -> None:
    """Arm, absorb CUPTI's one-off setup costs (first traced kernel launch, first traced graph
    launch: milliseconds each) with a throwaway stream launch and a throwaway 2-iteration graph
    (even, so the state parity is unchanged), then re-arm (clears the records)."""
    _arm(solver, capacity)
    solver.run_stream(2)
    solver.build_graph(2)
    solver.run_graph(1)
    solver.destroy_graph()
    _arm(solver, capacity)


def _collect(solver, capacity: int):
    L = _lib.lib()
    buf = np.zeros(2 * capacity, dtype=np.int64)
    n = L.ib_trace_kernels(solver.ctx, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), capacity)
    if n < 0:
        _lib.check(int(n))
    kern = buf[: 2 * min(n, capacity)].reshape(-1, 2)
    m = L.ib_trace_host_events(solver.ctx, None, 0)
    rows = np.zeros(4 * max(m, 1), dtype=np.int64)
    L.ib_trace_host_events(solver.ctx, rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), m)
    _arm(solver, 0)
    return kern, rows[: 4 * m].reshape(-1, 4), int(n)


def capture_graph(solver, batch_size: int, num_batches: int, pdl: bool = False, warm: int = 2) -> RealTrace:
    """Build a batch_size-iteration graph and replay it num_batches times, traced.

    The first launch of a newly instantiated executable under CUPTI kernel tracing pays CUPTI's
    instrumentation of its nodes (~3 ms at 100 nodes, seen as a 3 ms first-launch latency), which an
    untraced run never pays. So the executable is launched ``warm`` times first (two: both parity
    executables of an odd K, and the state parity is unchanged) and those launches' kernel records
    and launch events are dropped; the build events are kept."""
    kpi = solver.kernels_per_iteration
    per = batch_size * kpi
    cap = per * (num_batches + warm)
    _arm_warm(solver, cap)
    solver.build_graph(batch_size, pdl=pdl)
    solver.run_graph(warm)
    solver.run_graph(num_batches)
    solver.destroy_graph()
    kern, host, n = _collect(solver, cap)
    if n != cap:
        raise RuntimeError(f"trace recorded {n} kernels, expected {cap}")
    kern = kern[warm * per:]
    keep, seen = [], 0
    for row in host:
        if row[1] == 3:  # graph_launched: drop the warm launches, renumber the rest from 0
            seen += 1
            if seen <= warm:
                continue
            row = row.copy()
            row[2] = seen - warm - 1
        keep.append(row)
    return _assemble("graph", per, num_batches, kern, np.asarray(keep, dtype=np.int64))


def capture_stream(solver, iterations: int, pdl: bool = False) -> RealTrace:
    """Listing 1 (one launch per kernel), traced; each kernel is its own 'batch'."""
    kpi = solver.kernels_per_iteration
    cap = iterations * kpi
    _arm_warm(solver, cap)
    solver.run_stream(iterations, pdl=pdl)
    kern, host, n = _collect(solver, cap)
    if n != cap:
        raise RuntimeError(f"trace recorded {n} kernels, expected {cap}")
    return _assemble("baseline", 1, cap, kern, host)


def capture_launch_latency(solver, batch_size: int, reps: int = 7) -> list:
    """t_l, the first-launch latency of the model (model.py:48-74), measured as the paper defines
    it: graph launch call -> first kernel start with the device idle. The graph is built first and
    launched ``reps`` times, each launch synchronised before the next (ib_graph_run waits for its
    end event), so no launch queues behind another; the CUPTI set-up of the first traced launch is
    absorbed by _arm_warm. Returns the per-launch latencies in seconds."""
    per = batch_size * solver.kernels_per_iteration
    cap = reps * per
    _arm_warm(solver, cap)
    solver.build_graph(batch_size)
    for _ in range(reps):
        solver.run_graph(1)
    solver.destroy_graph()
    kern, host, n = _collect(solver, cap)
    if n != cap:
        raise RuntimeError(f"trace recorded {n} kernels, expected {cap}")
    launches = sorted(int(t) for t, kind, _, _ in host if kind == 3)
    return [(int(kern[i * per, 0]) - t) * 1e-9 for i, t in enumerate(launches)]


def launch_latency_untraced(solver, batch_size: int, t_a: float, t_k: float = 0.0, reps: int = 7) -> float:
    """t_l without any profiler attached: the device time of ONE graph launch on an idle device
    (CUDA events on the launch stream: the start event is stamped as soon as the host enqueues it,
    before the launch call returns) minus the steady per-graph time of back-to-back launches, plus
    the inter-graph gap t_a those back-to-back launches contain instead of t_l. The graph is cut
    to ~200 us of kernels (at least 2 iterations, even) so the run-to-run noise of the execution
    stays well below the latency being measured. Returns seconds."""
    if t_k > 0:
        short = max(2, int(math.ceil(200e-6 / t_k)))
        batch_size = min(batch_size, short + (short & 1))
    solver.build_graph(batch_size)
    solver.run_graph(2)  # first launches of the executable(s)
    steady = statistics.median(solver.run_graph(20).gpu_s / 20 for _ in range(3))
    single = statistics.median(solver.run_graph(1).gpu_s for _ in range(reps))
    solver.destroy_graph()
    return max(0.0, single - steady + t_a)


def fit_line(xs, ys) -> tuple[float, float]:
    """Least-squares slope and intercept."""
    x = np.asarray(xs, dtype=np.float64)
    y = np.asarray(ys, dtype=np.float64)
    slope, intercept = np.polyfit(x, y, 1)
    return float(slope), float(intercept)


def _assemble(mode, size, num, kern, host) -> RealTrace:
    starts = [r for r in host if r[1] == BUILD_STARTED]
    t0 = int(starts[0][0]) if starts else int(min(host[0][0] if len(host) else kern[0, 0], kern[0, 0]))
    ev = []
    launch_i = 0
    for t, kind, batch, kernel in host:
        if kind == BUILD_STARTED:
            continue
        if kind == 7:  # baseline launches: one per kernel, indexed as batches of size 1
            ev.append(((t - t0) * 1e-9, KIND[7], launch_i, 0))
            launch_i += 1
            continue
        if kind == 0:  # an odd-K hotspot graph has a second (swapped-parity) executable
            kernel = kernel % size
        ev.append(((t - t0) * 1e-9, KIND[int(kind)], None if batch < 0 else int(batch),
                   None if kernel < 0 else int(kernel)))
    ks = (kern - t0) * 1e-9
    for idx, (a, b) in enumerate(ks):
        bi, ki = divmod(idx, size)
        if mode == "graph" and ki == 0 and bi > 0:
            ev.append((ks[idx - 1, 1], KIND[6], bi, None))
        ev.append((a, KIND[4], bi, ki))
        ev.append((b, KIND[5], bi, ki))
    order = {k: i for i, k in enumerate(KIND.values())}
    ev.sort(key=lambda e: (e[0], order[e[1]]))
    return RealTrace(mode, size, num, ev, ks)


def write_trace_csv(trace: RealTrace, path) -> None:
    with open(path, "w") as fh:
        fh.write("# schema=1\n")
        fh.write(TRACE_HEADER + "\n")
        for t, kind, batch, kernel in trace.events:
            b = "" if batch is None else str(batch)
            k = "" if kernel is None else str(kernel)
            fh.write(f"{max(t, 0.0):.9f},{kind},{b},{k}\n")


def _per_iteration(k: np.ndarray, kpi: int) -> np.ndarray:
    """[start, end] of each iteration (its first kernel's start, its last kernel's end)."""
    if kpi <= 1:
        return k
    n = len(k) // kpi
    return np.stack([k[0:n * kpi:kpi, 0], k[kpi - 1:n * kpi:kpi, 1]], axis=1)


def derive_parameters(graph: RealTrace, stream: RealTrace, kernels_per_iteration: int = 1) -> dict:
    """The model's platform constants (model.py:48-74) measured from real traces.

    t_k kernel duration; t_i gap between consecutive kernels inside a graph; t_a gap between the
    last kernel of a graph and the first of the next; t_l first launch call -> first kernel start
    of this run (the trace command replaces it with the idle-device measurement of
    capture_launch_latency); t_b kernel-to-kernel gap of the plain launch loop; k_c / b_c here are
    the node-add interval and the add->upload tail of ONE build (the trace command replaces them
    with a fit of the whole build time T_C over several batch sizes, the phases the sweep fits).

    ``kernels_per_iteration`` > 1 (FDTD's H then E launches): the model's unit of work is one
    iteration, as in the sweeps and fits (batch sizes count iterations), so t_k is an iteration's
    span (first kernel start -> last kernel end, the H->E gap inside) and the gaps are between
    iterations.
    """
    kpi = max(1, int(kernels_per_iteration))
    g = _per_iteration(graph.kernels, kpi)
    size = max(1, graph.batch_size // kpi)
    dur = g[:, 1] - g[:, 0]
    gaps = g[1:, 0] - g[:-1, 1]
    idx = np.arange(1, len(g))
    intra = gaps[(idx % size) != 0]
    inter = gaps[(idx % size) == 0]
    s = _per_iteration(stream.kernels, kpi)
    sgaps = s[1:, 0] - s[:-1, 1]
    launches = [e[0] for e in graph.events if e[1] == "graph_launched"]
    nodes = sorted(e[0] for e in graph.events if e[1] == "node_added")
    inst = [e[0] for e in graph.events if e[1] == "graph_instantiated"]
    upl = [e[0] for e in graph.events if e[1] == "graph_uploaded"]
    k_c = (nodes[-1] - nodes[0]) / max(1, len(nodes) - 1) if len(nodes) > 1 else 0.0
    b_c = (upl[-1] - nodes[-1]) if (upl and nodes) else 0.0
    med = lambda a: float(statistics.median(a)) if len(a) else 0.0  # noqa: E731
    return {
        "t_k": med(dur),
        "t_i": med(intra) if len(intra) else 0.0,
        "t_a": med(inter) if len(inter) else 0.0,
        "t_l": float(g[0, 0] - launches[0]) if launches else 0.0,
        "t_b": med(sgaps),
        "k_c": float(k_c),
        "b_c": float(max(b_c, 0.0)),
        "kernels_graph": int(len(g)),
        "kernels_stream": int(len(s)),
        "instantiate_s": float(inst[-1] - nodes[-1]) if (inst and nodes) else 0.0,
    }


def write_params(path, params: dict, memory: dict | None = None) -> None:
    """The reference's params file (fileio.py:34-45): t_k t_i t_a t_l t_b k_c b_c [m_base m_node]."""
    with open(path, "w") as fh:
        fh.write("# schema=1\n# measured on B200 by paper_2501_09398_b200.trace\n")
        for key in ("t_k", "t_i", "t_a", "t_l", "t_b", "k_c", "b_c"):
            fh.write(f"{key} = {max(params[key], 0.0):.6e}\n")
        if memory:
            fh.write(f"m_base = {int(memory['m_base'])}\n")
            fh.write(f"m_node = {int(memory['m_node'])}\n")

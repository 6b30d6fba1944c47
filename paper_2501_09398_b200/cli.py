"""Command line front end: ``python -m paper_2501_09398_b200 <command>``.

``run-workload`` mirrors the reference's subcommand (pkg/src/iterbatch/cli.py:97-115,172-230):
same flags, same seeded inputs (seed 20240817, cli.py:42,172-199), same checksum line and
measurement CSV, executed on the B200 runtime. Extra flags: --dtype, --build, --pdl, --devices.

``sweep`` runs the batch-size sweep the paper's model is fitted on: for every
feasible K it records creation (T_C), graph execution (T_E) and stream execution, and writes one
measurement CSV per kind in the reference schema, readable by ``iterbatch fit`` / ``speedup``.

Exit codes as the reference (cli.py:3-4,253-263): 0 ok, 1 data errors (ValueError/OSError),
2 usage errors.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

from .fitting import MeasurementPoint, MeasurementSeries, write_measurements_csv
from .model import BatchPlan, feasible_batch_sizes

WORKLOAD_SEED = 20240817  # cli.py:42


class UsageError(Exception):
    pass


def _comma_sizes(text: str) -> list[int]:
    try:
        sizes = [int(part) for part in text.split(",")]
    except ValueError:
        raise argparse.ArgumentTypeError(f"sizes must be integers, got {text!r}")
    if not sizes or any(s < 1 for s in sizes):
        raise argparse.ArgumentTypeError(f"sizes must be positive, got {text!r}")
    return sizes


def build_workload(family: str, sizes: list[int]):
    """The reference's synthetic inputs, value for value (cli.py:172-199)."""
    from . import workloads as wl

    rng = np.random.default_rng(WORKLOAD_SEED)
    if family == "vector":
        if len(sizes) != 1:
            raise UsageError("vector takes one size: N")
        return wl.VectorWorkload(rng.random(sizes[0]), 0.9999)
    if family == "hotspot2d":
        if len(sizes) not in (1, 2):
            raise UsageError("hotspot2d takes N or N,N2 (rows, cols)")
        shape = (sizes[0], sizes[-1])
        return wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, 0.1)
    if family == "hotspot3d":
        if len(sizes) == 1:
            shape = (sizes[0],) * 3
        elif len(sizes) == 2:  # grid edge plus layer count
            shape = (sizes[0], sizes[0], sizes[1])
        elif len(sizes) == 3:
            shape = tuple(sizes)
        else:
            raise UsageError("hotspot3d takes N, N,LAYERS, or N,N2,N3")
        return wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, 0.1)
    if family != "fdtd":
        raise UsageError(f"unknown workload {family!r}")
    if len(sizes) == 1:
        nx = ny = nz = sizes[0]
    elif len(sizes) == 3:
        nx, ny, nz = sizes
    else:
        raise UsageError("fdtd takes N or N,N2,N3 (cells per axis)")
    return wl.te101_cavity(nx, ny, nz)


def programs():
    from . import workloads as wl

    return {
        "vector": wl.vector_program,
        "hotspot2d": wl.hotspot_program,
        "hotspot3d": wl.hotspot_program,
        "fdtd": wl.fdtd_program,
    }


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="iterbatch-b200",
        description="Iteration-batched CUDA-graph execution of solver kernels on B200.",
    )
    commands = parser.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--workload", choices=["vector", "hotspot2d", "hotspot3d", "fdtd"], required=True)
        p.add_argument("--size", type=_comma_sizes, required=True, metavar="N[,N2[,N3]]")
        p.add_argument("--iterations", type=int, required=True, metavar="I_K")
        p.add_argument("--dtype", choices=["f64", "f32"], default="f64")
        p.add_argument("--build", choices=["manual", "capture"], default="manual")
        p.add_argument("--pdl", action="store_true", help="programmatic dependent launch edges")
        p.add_argument("--fuse", action="store_true",
                       help="fdtd: one fused kernel per iteration (H then E, double-buffered lattice)")
        p.add_argument("--devices", type=_comma_sizes, default=None,
                       help="device id per axis-0 slab (hotspot only), e.g. 0,0 or 0,1,2,3")

    run = commands.add_parser("run-workload", help="execute a workload and measure or checksum it")
    common(run)
    run.add_argument("--batch-size", type=int, required=True, metavar="S")
    run.add_argument("--mode", choices=["loop", "batched"], required=True)
    run.add_argument("--repeats", type=int, default=10)
    run.add_argument("--timings", metavar="OUT.csv", help="write measured seconds")
    run.add_argument("--checksum", action="store_true", help="print the final-state checksum")
    run.set_defaults(func=_cmd_run_workload)

    sw = commands.add_parser("sweep", help="measure T_C / T_E / stream time over batch sizes")
    common(sw)
    sw.add_argument("--batch-sizes", default="all",
                    help="comma list, or 'all' for every divisor <= --max-fraction * I_K")
    sw.add_argument("--max-fraction", type=float, default=0.25)
    sw.add_argument("--repeats", type=int, default=10)
    sw.add_argument("--out", required=True, metavar="DIR")
    sw.set_defaults(func=_cmd_sweep)

    tr = commands.add_parser("trace", help="record real graph/stream timelines in the reference "
                             "trace schema and write the measured model constants")
    common(tr)
    tr.add_argument("--batch-size", type=int, required=True, metavar="S")
    tr.add_argument("--out", required=True, metavar="DIR")
    tr.set_defaults(func=_cmd_trace)
    return parser


def _cmd_run_workload(args) -> int:
    from . import workloads as wl

    if not args.checksum and not args.timings:
        raise UsageError("nothing to do: pass --checksum and/or --timings")
    state = build_workload(args.workload, args.size)
    program = programs()[args.workload]()
    plan = BatchPlan.from_batch_size(args.iterations, args.batch_size)
    order = wl.ExecutionOrder(args.mode)
    kw = dict(dtype=args.dtype, devices=args.devices, fuse=args.fuse)
    if args.checksum:
        if order is wl.ExecutionOrder.LOOP:
            final = wl.run_loop(program, state, plan.total_kernel_executions, pdl=args.pdl, **kw)
        else:
            final = wl.run_batched(program, state, plan.batch_size, plan.num_batches,
                                   build=args.build, pdl=args.pdl, **kw)
        print(f"{wl.state_checksum(final):016x}")
    if args.timings:
        series = wl.time_workload(program, state, plan, order, repeats=args.repeats,
                                  label=args.workload, build=args.build, pdl=args.pdl, **kw)
        write_measurements_csv(series, args.timings)
    return 0


def _cmd_sweep(args) -> int:
    from . import workloads as wl

    state = build_workload(args.workload, args.size)
    program = programs()[args.workload]()
    total = args.iterations
    if args.batch_sizes == "all":
        sizes = [k for k in feasible_batch_sizes(total) if k <= args.max_fraction * total]
    else:
        sizes = _comma_sizes(args.batch_sizes)
    os.makedirs(args.out, exist_ok=True)
    kw = dict(dtype=args.dtype, devices=args.devices, build=args.build, pdl=args.pdl, fuse=args.fuse)
    # The driver grows its graph-executable memory the first time a process instantiates a graph
    # of a new size (tens of ms once; tools/build_phases.py) — a per-process cost, not part of
    # T_C(K) — so it is paid before the sweep, as bench.py does.
    with wl._solver(state, args.dtype, args.devices, args.fuse) as warm:
        warm.build_graph(max(sizes), build=args.build, pdl=args.pdl)
        warm.destroy_graph()
    creation, execution, total_, stream, summary = [], [], [], [], []
    for k in sizes:
        plan = BatchPlan.from_batch_size(total, k)
        # an odd K on a ping-pong solver would otherwise build two executables (one per start
        # parity): re-point one instead (IB_FLAG_PATCH), so T_C stays one graph of K nodes as the
        # paper's linear creation model assumes
        patch = bool(k & 1) and args.build == "manual" and not args.devices and (
            args.workload.startswith("hotspot") or args.fuse)
        g = wl.time_workload_phases(program, state, plan, wl.ExecutionOrder.BATCHED,
                                    args.repeats, meminfo=True, patch=patch, **kw)
        s = wl.time_workload_phases(program, state, plan, wl.ExecutionOrder.LOOP,
                                    args.repeats, **kw)
        creation.append(MeasurementPoint(k, tuple(g["creation"])))
        execution.append(MeasurementPoint(k, tuple(g["execution"])))
        total_.append(MeasurementPoint(k, tuple(c + e for c, e in zip(g["creation"], g["execution"]))))
        stream.append(MeasurementPoint(k, tuple(s["execution"])))
        row = {
            "batch_size": k,
            "creation_s": statistics.fmean(g["creation"]),
            "graph_exec_s": statistics.fmean(g["execution"]),
            "graph_gpu_s": statistics.fmean(g["gpu"]),
            "stream_exec_s": statistics.fmean(s["execution"]),
            "stream_gpu_s": statistics.fmean(s["gpu"]),
            "graph_bytes": g["times"][0][0].graph_bytes,
            "nodes": g["times"][0][0].nodes,
        }
        row["us_per_iter_graph"] = 1e6 * row["graph_exec_s"] / total
        row["us_per_iter_stream"] = 1e6 * row["stream_exec_s"] / total
        row["speedup_exec"] = row["stream_exec_s"] / row["graph_exec_s"]
        row["speedup_total"] = row["stream_exec_s"] / (row["graph_exec_s"] + row["creation_s"])
        summary.append(row)
        print(json.dumps(row), flush=True)
    label = args.workload
    write_measurements_csv(MeasurementSeries(tuple(creation), label), os.path.join(args.out, "creation.csv"))
    write_measurements_csv(MeasurementSeries(tuple(execution), label), os.path.join(args.out, "execution.csv"))
    write_measurements_csv(MeasurementSeries(tuple(stream), label), os.path.join(args.out, "stream.csv"))
    # T = T_C + T_E per repeat: `iterbatch speedup --baseline stream.csv --graph total.csv`
    write_measurements_csv(MeasurementSeries(tuple(total_), label), os.path.join(args.out, "total.csv"))
    with open(os.path.join(args.out, "summary.json"), "w") as fh:
        json.dump({"workload": args.workload, "size": args.size, "iterations": total,
                   "dtype": args.dtype, "build": args.build, "pdl": args.pdl, "fuse": args.fuse,
                   "rows": summary}, fh, indent=1)
    return 0


def free_device_bytes(device: int) -> int:
    import ctypes

    from . import _lib

    free = ctypes.c_int64()
    _lib.check(_lib.lib().ib_mem_info(device, ctypes.byref(free), None))
    return free.value


def graph_bytes(solver, size: int, base_free: int) -> int:
    """Device bytes held with a size-S graph instantiated: the free memory before the solver's
    first build minus the free memory now (cudaMemGetInfo)."""
    solver.build_graph(size)
    used = base_free - free_device_bytes(solver.devices[0] if solver.devices else 0)
    solver.destroy_graph()
    return used


def _cmd_trace(args) -> int:
    from . import trace as tr
    from . import workloads as wl

    state = build_workload(args.workload, args.size)
    plan = BatchPlan.from_batch_size(args.iterations, args.batch_size)
    os.makedirs(args.out, exist_ok=True)
    even = lambda x: max(2, x + (x & 1))  # noqa: E731
    k = plan.batch_size
    with wl.DeviceSolver(state, args.dtype, devices=args.devices, fuse=args.fuse) as s:
        # memory model m = m_base + m_node * S (model.py:130-142, memory_usage:266-269), probed
        # before this context built any graph: free device memory before the first build minus
        # free memory with the size-S graph instantiated — right whether the driver releases a
        # destroyed graph's memory or keeps it for the next (bigger) one. cudaMemGetInfo moves in
        # 2 MiB steps and a kernel node holds ~1-3 KB, so the probe sizes are thousands of nodes
        # (not the run's K) for the fit to resolve m_node
        msizes = [1000, 2000, 4000, 8000]
        base = free_device_bytes(s.devices[0] if s.devices else 0)
        mem = [graph_bytes(s, size, base) for size in msizes]
        s.run_batched(plan.batch_size, plan.num_batches, pdl=args.pdl)  # warm-up
        s.upload(state)
        g = tr.capture_graph(s, plan.batch_size, plan.num_batches, pdl=args.pdl)
        s.upload(state)
        st = tr.capture_stream(s, plan.total_kernel_executions)
        # t_l: launch call -> first kernel start on an idle device (the traced run above queues
        # launches behind each other, and its first traced launch pays CUPTI's set-up)
        s.upload(state)
        lat = tr.capture_launch_latency(s, plan.batch_size)
        # k_c, b_c: the whole build time T_C (create + instantiate + upload, the phases the sweep
        # and fit_creation use) at four batch sizes, least squares over the batch size S; even
        # sizes so a ping-pong solver builds one executable per size
        sizes = sorted({even(k // 2), even(k), even(2 * k), even(4 * k)})
        tc = []
        for size in sizes:
            samples = []
            for _ in range(3):
                samples.append(s.build_graph(size).build_s)
                s.destroy_graph()
            tc.append(statistics.median(samples))
        params = tr.derive_parameters(g, st, s.kernels_per_iteration)
        # t_l with no profiler attached (CUDA events), the value the params file carries; the
        # CUPTI-measured idle-launch latency is reported beside it
        s.upload(state)
        t_l = tr.launch_latency_untraced(s, plan.batch_size, params["t_a"], params["t_k"])
    params["t_l_traced_run"] = params["t_l"]
    params["t_l_cupti"] = statistics.median(lat)
    params["t_l"] = t_l
    params["k_c_node_add"] = params["k_c"]
    params["k_c"], params["b_c"] = tr.fit_line(sizes, tc)
    params["b_c"] = max(0.0, params["b_c"])
    params["creation_points"] = [[sz, t] for sz, t in zip(sizes, tc)]
    m_node, m_base = tr.fit_line(msizes, mem)
    memory = {"m_base": int(max(0.0, round(m_base))), "m_node": int(max(0.0, round(m_node)))}
    params["memory_points"] = [[sz, b] for sz, b in zip(msizes, mem)]
    tr.write_trace_csv(g, os.path.join(args.out, "graph_trace.csv"))
    tr.write_trace_csv(st, os.path.join(args.out, "stream_trace.csv"))
    tr.write_params(os.path.join(args.out, "params.txt"), params, memory)
    print(json.dumps({"workload": args.workload, "size": args.size, "iterations": args.iterations,
                      "batch_size": args.batch_size, "dtype": args.dtype, **params, **memory}))
    return 0


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 2
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""bench.py — iteration-batched CUDA-graph execution of solver kernels on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--only NAME]

Headline (BASELINE.json configs[1]): Rodinia Hotspot 2-D, 1024x1024 binary32, N = 10,000 timesteps,
graph mode at the measured optimal batch size K*. One bench STEP = one full run of the workload:
graph creation + instantiation + upload (T_C) and the N/K graph launches (T_E), timed on the
device with CUDA events (ib_run_batched), with L2 flushed (a 2x-L2 buffer written) before every
step. value = device time per step / N in microseconds per iteration (lower is better).

Also reported on the same line:
  speedup_vs_stream  per-iteration stream launch (Listing 1) time / graph time, same N, same flush
  roofline           per-iteration algorithmic bytes / per-iteration graph execution time (device)
                     against the measured HBM copy bandwidth (MEASURED_PEAKS.json)
  e2e                the public API with host buffers: pinned H2D of the inputs, the run, D2H of
                     the result, host wall clock
  cpu_baseline       the reference algorithm (numpy restatement, binary64, oracle/numpy_port.py)
                     on a bounded sample, on this host's cores (rank 0, N = 1 only)
  configs            the other BASELINE.json configs measured the same way (skeleton, Hotspot3D
                     512x512x8, FDTD 256^3, Hotspot3D 2048x2048x256)

N > 1 (torchrun): the headline path does not shard (launch-bound by design), so
each rank runs an independent replica on its own GPU ("replicas only", scaling "weak"); value is
the whole-job time per iteration = max-over-ranks step time / (N_iterations * world_size).

--impl reference: the reference CPU path (the numpy restatement of workloads.py, binary64, all host
threads via the reference's row-slab scheme) on the same config and metric, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "µs/iteration and graph-vs-stream speed-up vs batch size K; stencil HBM GB/s % of peak"
UNIT = "µs/iteration"

# BASELINE.json configs, in order. k_candidates: the divisors of N the in-bench sweep tries.
CONFIGS = {
    "skeleton": dict(workload="vector", size=[16384], iterations=10000,
                     label="Skeleton vector-scale 2^14 fp32, N=10000",
                     k_candidates=[10, 20, 50, 100, 200, 500, 1000, 2000]),
    "hotspot2d": dict(workload="hotspot2d", size=[1024], iterations=10000,
                      label="Rodinia Hotspot 2-D 1024x1024 fp32, N=10000",
                      k_candidates=[10, 20, 25, 40, 50, 80, 100, 125, 200, 250, 400, 500, 1000, 2000]),
    "hotspot3d": dict(workload="hotspot3d", size=[512, 8], iterations=1000,
                      label="Rodinia Hotspot3D 512x512x8 fp32, N=1000",
                      k_candidates=[10, 20, 25, 40, 50, 100, 125, 200, 250, 500, 1000]),
    "fdtd": dict(workload="fdtd", size=[256], iterations=2000,
                 label="FDTD Yee 256^3 fp32 (H+E per iteration), N=2000",
                 k_candidates=[10, 20, 50, 100, 200]),
    "fdtd_fused": dict(workload="fdtd", size=[256], iterations=2000, fuse=True,
                       label="FDTD Yee 256^3 fp32, H+E fused in one kernel per iteration, N=2000",
                       k_candidates=[10, 20, 50, 100, 200]),
    "hotspot3d_large": dict(workload="hotspot3d", size=[2048, 2048, 256], iterations=100,
                            label="Hotspot3D 2048x2048x256 fp32, N=100",
                            k_candidates=[5, 10, 20, 50, 100]),
}
HEADLINE = "hotspot2d"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------------------------
# distributed plumbing (torch only when launched under torchrun with WORLD_SIZE > 1)
# ---------------------------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.torch = None
        self.shared = False
        if self.world > 1:
            import torch
            import torch.distributed as td

            n = torch.cuda.device_count()
            if self.world > n:  # protocol check on a small box: ranks share GPUs, gloo for plumbing
                self.shared = True
                self.local = self.local % max(1, n)
                if n:  # (none at all: the reference arm, CPU only)
                    torch.cuda.set_device(self.local)
                td.init_process_group("gloo")
            else:
                torch.cuda.set_device(self.local)
                td.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.torch, self.td = torch, td

    def barrier(self):
        if self.torch is not None:
            self.td.barrier()

    def max(self, x: float) -> float:
        if self.torch is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cpu" if self.shared else "cuda")
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.torch is not None:
            self.td.destroy_process_group()


# ---------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------------
class Clocks:
    """SM clock and clock-event reasons sampled DURING a timed region: in-process NVML polling
    every 200 ms (an nvidia-smi child polling the driver slowed graph instantiation inside the
    region by milliseconds; each NVML query can still delay a concurrent build by ~0.1 ms, so
    sparse), nvidia-smi as the fallback. One more sample is taken at the region's end so short
    regions are covered."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self.lines = []
        self.start = 0
        self._stop = threading.Event()
        self.thread = None

    def _nvml_index(self) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if ids and all(v.isdigit() for v in ids) and self.device < len(ids):
            return int(ids[self.device])
        return self.device

    def _nvml_sample(self):
        n = self.nvml
        sm = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self.handle, n.NVML_CLOCK_SM)
        bits = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        flags = (n.nvmlClocksEventReasonHwSlowdown, n.nvmlClocksEventReasonHwThermalSlowdown,
                 n.nvmlClocksEventReasonSwThermalSlowdown, n.nvmlClocksEventReasonSwPowerCap)
        self.samples.append((float(sm), float(mx), {nm for nm, f in zip(self.NAMES, flags) if bits & f}))

    def _nvml_loop(self):
        while not self._stop.wait(0.2):
            try:
                self._nvml_sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a few hundred ms to print its first line: wait for it so a short
            # timed region is still sampled; keep only later lines
            t_end = time.monotonic() + 3.0
            while not self.lines and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        self.start = len(self.lines)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            self._stop.set()
            self.thread.join(timeout=2)
            try:
                self._nvml_sample()  # the region's end
                self.nvml.nvmlShutdown()
            except Exception:
                pass
            return
        if self.proc is not None:
            t_end = time.monotonic() + 0.3  # at least one sample from the region's end
            while len(self.lines) <= self.start and time.monotonic() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)
            for line in self.lines[self.start:]:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm, mx = float(parts[0]), float(parts[1])
                except ValueError:
                    continue
                self.samples.append((sm, mx, {nm for nm, f in zip(self.NAMES, parts[3:7])
                                              if f.lower() == "active"}))

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set().union(*(r for _, _, r in self.samples))
        return {"sm_mhz": statistics.median(sm for sm, _, _ in self.samples),
                "sm_max_mhz": self.samples[-1][1], "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def measured_peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(kernel_key: str):
    """DRAM bytes per launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(kernel_key)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def make_state(cfg):
    from paper_2501_09398_b200 import cli

    return cli.build_workload(cfg["workload"], cfg["size"])


def pick_k(solver, cfg, quick: bool) -> tuple[int, bool, list]:
    """In-bench batch-size sweep: minimise total device time T_C + T_E over candidate K (+PDL)."""
    n = cfg["iterations"]
    cands = [k for k in cfg["k_candidates"] if n % k == 0]
    if quick:
        cands = [k for k in cands if k in (10, 100, 1000)] or cands[:2]
    # The driver grows its graph-executable memory the first time a process instantiates a graph
    # of a new size (tools/build_phases.py: first K=2000 instantiate 60 ms, later ones 2.5 ms) —
    # a once-per-process cost, not part of T_C(K): pay it before the sweep.
    for pdl in (False, True):
        solver.build_graph(max(cands), pdl=pdl)
        solver.destroy_graph()
    reps = 1 if quick else 3  # median of 3: one host hiccup inside a graph build (T_C) would
    rows = []                 # otherwise mark a K as slow
    best = None
    for k in cands:
        for pdl in (False, True):
            ts = []
            for _ in range(reps):
                solver.flush_l2()
                ts.append(solver.run_batched(k, n // k, pdl=pdl))
            g = statistics.median(t.gpu_s for t in ts)
            rows.append({"K": k, "pdl": pdl, "us_per_iter": 1e6 * g / n,
                         "T_C_us": 1e6 * statistics.median(t.build_s for t in ts), "samples": reps})
            if best is None or g < best[0]:
                best = (g, k, pdl)
    return best[1], best[2], rows


def measure_ours(name, cfg, args, dist: Dist, device: int, headline: bool) -> dict:
    from paper_2501_09398_b200 import workloads as wl

    n = cfg["iterations"]
    state = make_state(cfg)
    solver = wl.DeviceSolver(state, "f32", devices=[device], fuse=cfg.get("fuse", False))
    try:
        k, pdl, sweep = pick_k(solver, cfg, args.quick)
        num = n // k
        for _ in range(args.warmup):
            solver.upload(state)
            solver.flush_l2()
            solver.run_batched(k, num, pdl=pdl)
        # ---- timed: K steps, each = one full run (T_C + T_E), L2 flushed before each ----------
        dist.barrier()
        solver.sync()
        step_s, tc_s = [], []
        small = sum(a.nbytes for a in state.state_arrays()) < (256 << 20)
        with Clocks(device) as clocks:
            for _ in range(args.steps):
                if small:  # fresh inputs each step (outside the timed interval)
                    solver.upload(state)
                solver.flush_l2()
                t = solver.run_batched(k, num, pdl=pdl)
                step_s.append(t.gpu_s)
                tc_s.append(t.build_s)
        solver.sync()
        dist.barrier()
        step_mean = dist.max(statistics.fmean(step_s))
        # ---- graph execution only (for the roofline) and the stream baseline ------------------
        solver.build_graph(k, pdl=pdl)
        exec_s = []
        for _ in range(3):
            solver.flush_l2()
            exec_s.append(solver.run_graph(num).gpu_s)
        solver.destroy_graph()
        stream_s = []
        for _ in range(5):  # the host's launch rate varies run to run: 5 samples for the error bar
            solver.flush_l2()
            stream_s.append(solver.run_stream(n).gpu_s)
        stream_pdl = []
        for _ in range(2):
            solver.flush_l2()
            stream_pdl.append(solver.run_stream(n, pdl=True).gpu_s)
        stream_mean = statistics.fmean(stream_s)
        exec_mean = statistics.fmean(exec_s)
        it_bytes = solver.iteration_bytes
        state_bytes = sum(int(np.prod(shp)) for shp in solver.shapes) * np.dtype(solver.np_dtype).itemsize
        peak, peak_src = measured_peaks()
        achieved = it_bytes / (exec_mean / n) / 1e9
        kpi = solver.kernels_per_iteration
        out = {
            "name": name,
            "workload": cfg["label"],
            "iterations": n,
            "batch_size": k,
            "pdl": pdl,
            "us_per_iter": 1e6 * step_mean / n,
            "ms_per_step": 1e3 * step_mean,
            "T_C_us": 1e6 * statistics.fmean(tc_s),
            "graph_exec_us_per_iter": 1e6 * exec_mean / n,
            "stream_us_per_iter": 1e6 * stream_mean / n,
            "stream_pdl_us_per_iter": 1e6 * statistics.fmean(stream_pdl) / n,
            "speedup_vs_stream": stream_mean / step_mean,
            # the reference's error model (model.py:247-253): relative std errors in quadrature
            "speedup_vs_stream_err": (stream_mean / step_mean) * math.hypot(
                statistics.stdev(stream_s) / stream_mean if len(stream_s) > 1 else 0.0,
                statistics.stdev(step_s) / statistics.fmean(step_s) if len(step_s) > 1 else 0.0),
            "speedup_vs_stream_exec_only": stream_mean / exec_mean,
            "kernels_per_iter": kpi,
            "gpu_launches": args.steps * n * kpi,
            "roofline": {
                "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(name),
                "bytes_per_iter": it_bytes, "peak_source": peak_src,
                "note": "per-iteration algorithmic bytes / per-iteration graph execution time"
                        + ("; fused FDTD: each field read+written once = 48 B/cell" if cfg.get("fuse") else "")
                        + ("; the state (%.1f MB) stays L2-resident across iterations, so this per-launch "
                           "kernel is launch/latency-bound and the HBM roof is not the binding one "
                           "(DESIGN.md §4)" % (state_bytes / 1e6) if state_bytes < (96 << 20) else ""),
            },
            "k_sweep": sweep,
            "clocks": clocks.summary(),
            "launches": solver.describe(),  # the kernels one iteration ran (ib_describe)
        }
        if headline:
            out["e2e"] = measure_e2e(solver, state, k, num, n, pdl, args)
        return out
    finally:
        solver.close()


def measure_dist(name, cfg, args, dist: Dist) -> dict:
    """Strong scaling of one global hotspot grid over WORLD_SIZE GPUs (one process each): axis-0
    slabs; the stencil kernel stores its boundary planes straight into the neighbours' halo planes
    (CUDA IPC / NVLink peer stores) with device-counter ordering in the graph
    (IB_BENCH_EXCHANGE=nccl: the runtime's NCCL send/recv group instead)."""
    from paper_2501_09398_b200.distributed import DistributedSolver, unique_id

    n = cfg["iterations"]
    shape = list(cfg["size"])
    if len(shape) == 2:
        shape = [shape[0], shape[0], shape[1]]
    exchange = os.environ.get("IB_BENCH_EXCHANGE", "peer")  # peer: IPC halo stores; nccl: send/recv
    uid = [unique_id() if dist.rank == 0 and exchange == "nccl" else None]
    if dist.world > 1 and exchange == "nccl":
        dist.td.broadcast_object_list(uid, src=0)

    def allgather(blob):
        out = [None] * dist.world
        dist.td.all_gather_object(out, blob)
        return out

    s = DistributedSolver.from_seed(shape, 0.1, "f32", dist.rank, dist.world, dist.local, uid[0],
                                    exchange=exchange, allgather=allgather if dist.world > 1 else None)
    try:
        k = 20 if n % 20 == 0 else n
        for _ in range(args.warmup):
            s.run_batched(k, n // k)
        dist.barrier()
        steps = []
        with Clocks(dist.local) as clocks:
            for _ in range(args.steps):
                s.flush_l2()
                dist.barrier()
                steps.append(s.run_batched(k, n // k).gpu_s)
        step = dist.max(statistics.fmean(steps))
        local_bytes = s.iteration_bytes
        peak, src = measured_peaks()
        achieved = local_bytes / (step / n) / 1e9  # this rank's slab bytes over the max-over-ranks time
        how = ("halo planes stored into the neighbours' buffers by the stencil kernel over CUDA IPC, "
               "device-counter ordering in-graph" if exchange == "peer" else "NCCL send/recv halos in-graph")
        return {"name": name, "workload": cfg["label"] + f", {dist.world} GPUs (axis-0 slabs, {how})",
                "iterations": n, "batch_size": k, "us_per_iter": 1e6 * step / n, "ms_per_step": 1e3 * step,
                "scaling": "strong", "gpu_launches": args.steps * n * (3 if exchange == "peer" else 1),
                "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                             "frac": round(achieved / peak, 4), "traffic": None, "bytes_per_iter": local_bytes,
                             "peak_source": src, "note": "per GPU: its slab's algorithmic bytes / iteration time"},
                "clocks": clocks.summary()}
    finally:
        s.close()


def measure_e2e(solver, state, k, num, n, pdl, args) -> dict:
    """Public API with host buffers: pinned H2D of every input field, the run, D2H of the result."""
    import ctypes

    from paper_2501_09398_b200 import _lib

    L = _lib.lib()
    pinned, ptrs = [], []
    for a in solver.host_arrays(state):
        p = ctypes.c_void_p()
        _lib.check(L.ib_host_alloc(ctypes.byref(p), a.nbytes))
        ptrs.append(p)
        view = np.ctypeslib.as_array((ctypes.c_byte * a.nbytes).from_address(p.value))
        view = view.view(a.dtype).reshape(a.shape)
        view[...] = a
        pinned.append(view)
    out_buf = np.ctypeslib.as_array(
        (ctypes.c_byte * pinned[0].nbytes).from_address(ptrs[0].value)).view(pinned[0].dtype).reshape(pinned[0].shape)
    written = [0] if solver.kind.startswith("hotspot") else list(range(solver.nfields))
    h2d = sum(a.nbytes for a in pinned)
    d2h = sum(pinned[f].nbytes for f in written)
    samples = []
    try:
        for rep in range(args.warmup + args.steps):
            solver.flush_l2()
            t0 = time.perf_counter()
            solver.upload(pinned)
            solver.run_batched(k, num, pdl=pdl)
            for f in written:
                solver.download_field(f, out_buf if f == 0 else None)
            dt = time.perf_counter() - t0
            if rep >= args.warmup:
                samples.append(dt)
    finally:
        for p in ptrs:
            L.ib_host_free(p)
    return {"value": 1e6 * statistics.fmean(samples) / n, "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "note": "host wall clock: pinned H2D + build + run + D2H per step"}


# ---------------------------------------------------------------------------------------------
# CPU baseline / reference arm: the reference algorithm (numpy, binary64) on this host
# ---------------------------------------------------------------------------------------------
def cpu_sample(cfg, workers: int, budget_s: float, min_iters: int = 1) -> dict:
    from oracle import numpy_port as npo

    state = make_state(cfg)
    pool = npo.SlabPool(workers)
    try:
        def run(iters):
            if cfg["workload"] == "vector":
                v = state.values
                t0 = time.perf_counter()
                npo.run_vector(v, state.scale_constant, iters, pool)
            elif cfg["workload"].startswith("hotspot"):
                t0 = time.perf_counter()
                npo.run_hotspot(state.temperature, state.power, state.diffusion_coefficient, iters, pool)
            else:
                c_h, c_e = npo.fdtd_coefficients(state.cell_size, state.time_step)
                t0 = time.perf_counter()
                npo.run_fdtd(state.state_arrays(), state.cell_size, c_h, c_e, iters, pool)
            return time.perf_counter() - t0

        probe = run(1)
        iters = max(min_iters, min(cfg["iterations"], int(budget_s / max(probe, 1e-9))))
        dt = run(iters)
    finally:
        pool.close()
    return {"us_per_iter": 1e6 * dt / iters, "iterations": iters, "seconds": dt, "workers": workers}


def cpu_baseline(cfg, budget_s: float) -> dict:
    cores = len(os.sched_getaffinity(0))
    single = cpu_sample(cfg, 1, budget_s / 2)
    multi = cpu_sample(cfg, cores, budget_s / 2) if cores > 1 else single
    best = multi if multi["us_per_iter"] < single["us_per_iter"] else single
    return {"value": round(best["us_per_iter"], 2), "unit": UNIT, "cores": best["workers"],
            "kind": "port",
            "sample": (f"{best['iterations']} of {cfg['iterations']} iterations of {cfg['label']} in "
                       f"binary64 (the reference's numpy algorithm, oracle/numpy_port.py, row slabs over "
                       f"{best['workers']} threads); 1-thread: {single['us_per_iter']:.1f} us/iter"),
            "cpu": cpu_model()}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, dist: Dist) -> int:
    cfg = CONFIGS[args.only or HEADLINE]
    if dist.rank != 0:
        return 0
    from oracle import numpy_port as npo

    cores = len(os.sched_getaffinity(0))
    state = make_state(cfg)
    pool = npo.SlabPool(cores)
    sample_iters = {"vector": 2000, "hotspot2d": 20, "hotspot3d": 5, "fdtd": 1}[cfg["workload"]]
    if cfg["size"] == [2048, 2048, 256]:
        sample_iters = 1

    def step():
        t0 = time.perf_counter()
        if cfg["workload"] == "vector":
            npo.run_vector(state.values, state.scale_constant, sample_iters, pool)
        elif cfg["workload"].startswith("hotspot"):
            npo.run_hotspot(state.temperature, state.power, state.diffusion_coefficient, sample_iters, pool)
        else:
            c_h, c_e = npo.fdtd_coefficients(state.cell_size, state.time_step)
            npo.run_fdtd(state.state_arrays(), state.cell_size, c_h, c_e, sample_iters, pool)
        return time.perf_counter() - t0

    try:
        for _ in range(args.warmup):
            step()
        samples = [step() for _ in range(args.steps)]
    finally:
        pool.close()
    mean = statistics.fmean(samples)
    value = 1e6 * mean / sample_iters
    sample = (f"each step = {sample_iters} of the {cfg['iterations']} iterations of {cfg['label']}, "
              f"binary64, reference numpy algorithm (oracle/numpy_port.py) over {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * mean, 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seed 20240817)",
        "config": {"workload": cfg["label"], "iterations": cfg["iterations"], "parallelism": "cpu-threads"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--only", choices=sorted(CONFIGS), default=None,
                    help="measure just this config (as the headline)")
    ap.add_argument("--no-extra", action="store_true", help="skip the non-headline configs")
    ap.add_argument("--quick", action="store_true", help="small K sweep")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU baseline work")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    dist = Dist()
    try:
        if args.impl == "reference":
            return run_reference(args, dist)
        return run_ours(args, dist)
    finally:
        dist.close()


def run_ours(args, dist: Dist) -> int:
    from paper_2501_09398_b200 import _lib

    _lib.lib()
    if _lib.device_count() < 1:
        raise RuntimeError("bench.py needs a CUDA device (no CPU fallback)")
    device = dist.local
    head_name = args.only or HEADLINE
    if head_name == "hotspot3d_large" and dist.world > 1:  # the sharded config alone
        r = measure_dist(head_name, CONFIGS[head_name], args, dist)
        if dist.rank == 0:
            print(json.dumps({"metric": METRIC, "value": round(r["us_per_iter"], 3), "unit": UNIT,
                              "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
                              "ms_per_step": round(r["ms_per_step"], 3), "higher_is_better": False,
                              "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                              "data": "synthetic (reference generator, seed 20240817)",
                              "config": {"workload": r["workload"], "iterations": r["iterations"],
                                         "batch_size": r["batch_size"],
                                         "parallelism": f"axis-0 slabs x{dist.world}"
                                         + (" (ranks share GPUs: protocol check only)" if dist.shared else "")},
                              "roofline": r["roofline"], "gpu_launches": r["gpu_launches"],
                              "clocks": r["clocks"]}), flush=True)
        return 0
    head = measure_ours(head_name, CONFIGS[head_name], args, dist, device, headline=True)
    log(f"[{head_name}] {head['us_per_iter']:.3f} us/iter at K={head['batch_size']} "
        f"(stream {head['stream_us_per_iter']:.3f}, x{head['speedup_vs_stream']:.2f})")
    extra = {}
    if not args.no_extra and args.only is None:
        for name, cfg in CONFIGS.items():
            if name == head_name:
                continue
            try:
                if name == "hotspot3d_large" and dist.world > 1:
                    extra[name] = measure_dist(name, cfg, args, dist)
                    continue
                r = measure_ours(name, cfg, args, dist, device, headline=False)
                r.pop("k_sweep", None)
                extra[name] = r
                log(f"[{name}] {r['us_per_iter']:.3f} us/iter at K={r['batch_size']} "
                    f"(stream {r['stream_us_per_iter']:.3f}, x{r['speedup_vs_stream']:.2f}) "
                    f"roofline {r['roofline']['frac']:.3f}")
            except MemoryError as exc:
                extra[name] = {"skipped": f"out of device memory: {exc}"}
    cpu = None
    if dist.rank == 0 and args.gpus == 1 and dist.world == 1:
        cpu = cpu_baseline(CONFIGS[head_name], args.cpu_budget)
    world = dist.world
    value = head["us_per_iter"] / world
    line = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(head["ms_per_step"], 4),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (reference generator cli.py:172-199, seed 20240817)",
        "config": {
            "workload": head["workload"] + " (one step = one full run: graph build T_C + N/K launches)",
            "iterations": head["iterations"],
            "batch_size": head["batch_size"],
            "graph_edges": "programmatic (PDL)" if head["pdl"] else "plain",
            "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
            "l2": "flushed before every step (2x L2 buffer written); the 12.6 MB working set then "
                  "stays L2-resident across the run's iterations as in the real application",
        },
        "speedup_vs_stream": round(head["speedup_vs_stream"], 3),
        "speedup_vs_stream_err": round(head["speedup_vs_stream_err"], 4),
        "stream_us_per_iter": round(head["stream_us_per_iter"], 4),
        "stream_pdl_us_per_iter": round(head["stream_pdl_us_per_iter"], 4),
        "graph_exec_us_per_iter": round(head["graph_exec_us_per_iter"], 4),
        "T_C_us": round(head["T_C_us"], 1),
        "roofline": head["roofline"],
        "cpu_baseline": cpu,
        "e2e": head["e2e"],
        "gpu_launches": head["gpu_launches"],
        "clocks": head["clocks"],
        "k_sweep": head["k_sweep"],
        "configs": extra,
    }
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

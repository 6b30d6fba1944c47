"""GPU: the ``run-workload`` command end to end, and the host-side contracts round 2 added.

* ``run-workload --checksum`` in loop and batched modes prints the reference's own checksum for
  every App. B.4 KAT row (tests/golden/kats.json) — the reference's gate compares loop and batched
  checksums through its CLI (pkg/tests/test_cli.py:197-260, cli.py:210-230).
* ``--timings`` writes the reference measurement CSV (fileio.py:184-190: ``# schema=1``, header
  ``batch_size,run_index,seconds``, one row per repeat, 9 decimals).
* The drop-in functions are thread-safe like the reference's pure functions (a context is checked
  out exclusively while a call uses it).
* Tall, narrow grids (grid.y clamp of the scalar kernel), odd-K WHILE launches over several batches.
"""

import csv
import os
import threading

import numpy as np
import pytest

from oracle import cpu as ocpu
from paper_2501_09398_b200 import cli
from paper_2501_09398_b200 import workloads as wl
from tests.test_gpu_parity import KATS, _kat_id

pytestmark = pytest.mark.gpu

# every KAT whose binary64 run finishes in well under a second on the device
CLI_KATS = [k for k in KATS if k["size"] not in ("256",)]


def _run_cli(capsys, *argv):
    code = cli.main(list(argv))
    out, err = capsys.readouterr()
    return code, out, err


@pytest.mark.parametrize("mode", ["loop", "batched"])
@pytest.mark.parametrize("kat", CLI_KATS, ids=[_kat_id(k) for k in CLI_KATS])
def test_run_workload_checksum_matches_reference(gpu, capsys, kat, mode):
    code, out, err = _run_cli(capsys, "run-workload", "--workload", kat["workload"], "--size", kat["size"],
                              "--iterations", str(kat["iterations"]), "--batch-size", str(kat["batch_size"]),
                              "--mode", mode, "--checksum")
    assert code == 0, err
    assert out.strip() == kat["checksum"]


def test_run_workload_fdtd_256_checksum_matches_oracle(gpu, capsys):
    (kat,) = [k for k in KATS if k["workload"] == "fdtd" and k["size"] == "256"]
    code, out, err = _run_cli(capsys, "run-workload", "--workload", "fdtd", "--size", "256", "--iterations",
                              str(kat["iterations"]), "--batch-size", str(kat["batch_size"]), "--mode",
                              "batched", "--checksum", "--fuse")
    assert code == 0, err
    assert out.strip() == kat["checksum"]


@pytest.mark.parametrize("mode", ["loop", "batched"])
def test_run_workload_timings_follow_the_reference_schema(gpu, capsys, tmp_path, mode):
    path = tmp_path / "t.csv"
    code, _, err = _run_cli(capsys, "run-workload", "--workload", "hotspot2d", "--size", "64,48", "--iterations",
                            "100", "--batch-size", "10", "--mode", mode, "--repeats", "3", "--timings", str(path))
    assert code == 0, err
    lines = path.read_text().splitlines()
    assert lines[0] == "# schema=1" and lines[1] == "batch_size,run_index,seconds"
    rows = list(csv.reader(lines[2:]))
    assert [int(r[0]) for r in rows] == [10, 10, 10]
    assert [int(r[1]) for r in rows] == [0, 1, 2]
    for r in rows:
        assert float(r[2]) > 0 and len(r[2].split(".")[1]) == 9


def test_run_workload_usage_and_data_errors(gpu, capsys):
    code, _, err = _run_cli(capsys, "run-workload", "--workload", "vector", "--size", "64", "--iterations", "4",
                            "--batch-size", "2", "--mode", "loop")
    assert code == 2 and "usage error" in err
    code, _, err = _run_cli(capsys, "run-workload", "--workload", "vector", "--size", "64", "--iterations", "10",
                            "--batch-size", "3", "--mode", "batched", "--checksum")
    assert code == 1 and "error:" in err  # BatchPlan: 3 does not divide 10


# ---- thread safety of the drop-in functions --------------------------------------------------------
def test_drop_in_functions_are_thread_safe(gpu):
    """Eight threads, three shapes (more than the context cache holds), concurrent runs: every
    result equals the serial one (the reference functions are pure)."""
    shapes = [(40, 33), (40, 33), (24, 17), (31, 8)]
    states = [wl.HotspotWorkload(np.random.default_rng(i).random(s), np.random.default_rng(i + 9).random(s) * 1e-3,
                                 0.1) for i, s in enumerate(shapes)]
    prog = wl.hotspot_program()
    want = [wl.state_checksum(wl.run_loop(prog, s, 24)) for s in states]
    errors, got = [], {}

    def work(t):
        try:
            for r in range(6):
                i = (t + r) % len(states)
                fn = wl.run_batched if (t + r) % 2 else wl.run_peeled
                out = fn(prog, states[i], 4, 6) if fn is wl.run_batched else fn(prog, states[i], 24, 5)
                got[(t, r)] = (i, wl.state_checksum(out))
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for (_, _), (i, h) in got.items():
        assert h == want[i]
    wl.release_cached_contexts()


# ---- shapes and modes -------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_tall_narrow_hotspot_grid(gpu, dtype):
    """100000 x 4: the vector kernels refuse > 65535 rows and the scalar kernel's row chunks must
    keep grid.y <= 65535 — the reference handles the shape, so must the device path."""
    rng = np.random.default_rng(5)
    t, p = rng.random((100000, 4)), rng.random((100000, 4)) * 1e-3
    state = wl.HotspotWorkload(t, p, 0.1)
    np_dt = np.float64 if dtype == "f64" else np.float32
    out = wl.run_batched(wl.hotspot_program(), state, 3, 2, dtype=dtype)
    ref = ocpu.hotspot(t, p, 0.1, 6, np_dt)
    assert np.array_equal(np.asarray(out.temperature, np_dt), ref)


@pytest.mark.parametrize("workload,size", [("hotspot2d", [37, 29]), ("hotspot3d", [20, 16, 8]),
                                           ("fdtd", [7, 5, 6])])
@pytest.mark.parametrize("k,batches", [(3, 5), (5, 2), (7, 1), (1, 4)])
def test_while_loop_odd_k_many_batches(gpu, workload, size, k, batches):
    """WHILE node with an odd K on a ping-pong solver: the body runs two batches (the second, of
    the other buffer parity, inside an IF node) — any number of batches in ONE graph launch."""
    state = cli.build_workload(workload, size)
    fuse = workload == "fdtd"  # the fused FDTD solver ping-pongs its lattice
    prog = cli.programs()[workload]()
    want = wl.state_checksum(wl.run_loop(prog, state, k * batches, fuse=fuse))
    with wl.DeviceSolver(state, "f64", fuse=fuse) as s:
        s.build_graph(k, while_loop=True)
        t = s.run_graph(batches)
        assert t.launches == 1
        assert wl.state_checksum(s.download(state)) == want
        s.run_graph(batches)  # the parity moved by `batches`: the run continues on the right buffer
        want2 = wl.state_checksum(wl.run_loop(prog, state, 2 * k * batches, fuse=fuse))
        assert wl.state_checksum(s.download(state)) == want2


# ---- the `trace` command: measured model constants for `iterbatch optimize` -------------------------
@pytest.mark.parametrize("workload,size,kpi", [("hotspot2d", "256", 1), ("fdtd", "16", 2)])
def test_trace_command_writes_the_measured_model(gpu, capsys, tmp_path, workload, size, kpi):
    """`trace` end to end: the graph trace holds exactly the traced run (the two CUPTI warm-up
    launches dropped, batches renumbered from 0), the params file carries every key the reference
    parser reads (fileio.py:70-125) with t_l measured without a profiler and m_node from graph
    memory, and FDTD's two launches per iteration make one model 'kernel' (t_k per iteration)."""
    out = tmp_path / "tr"
    code, stdout, err = _run_cli(capsys, "trace", "--workload", workload, "--size", size, "--iterations", "200",
                                 "--batch-size", "20", "--out", str(out))
    assert code == 0, err
    import json

    rep = json.loads(stdout.strip().splitlines()[-1])
    keys = {}
    for line in (out / "params.txt").read_text().splitlines():
        if "=" in line and not line.startswith("#"):
            k, v = line.split("=")
            keys[k.strip()] = float(v)
    assert list(keys) == ["t_k", "t_i", "t_a", "t_l", "t_b", "k_c", "b_c", "m_base", "m_node"]
    assert 0 < keys["t_k"] < 1e-3 and 0 < keys["t_l"] < 1e-3 and keys["k_c"] > 0
    assert keys["m_node"] > 0  # a kernel node holds ~2.4 KB of device memory per iteration
    assert rep["t_l_cupti"] > 0 and len(rep["memory_points"]) == 4
    rows = list(csv.reader(open(out / "graph_trace.csv")))[2:]
    kinds = [r[1] for r in rows]
    assert kinds.count("kernel_started") == kinds.count("kernel_ended") == 200 * kpi
    launched = [int(r[2]) for r in rows if r[1] == "graph_launched"]
    assert launched == list(range(10))  # 200 / 20 batches, the warm-up launches dropped
    ts = [float(r[0]) for r in rows]
    assert ts == sorted(ts)
    if kpi == 2:  # one model 'kernel' = one iteration = the H and the E launch
        one = [float(r[0]) for r in rows if r[1] in ("kernel_started", "kernel_ended")]
        assert keys["t_k"] > 0.5 * (one[3] - one[0])


# ---- device memory exhaustion -------------------------------------------------------------------
def test_out_of_device_memory_raises_memory_error_and_leaks_nothing(gpu):
    """A grid larger than the device (Hotspot3D 4096 x 4096 x 512 binary64: 3 x 68.7 GB) fails
    ib_create with IB_ENOMEM -> MemoryError (the reference's exception for allocation failure),
    frees what it had allocated, and the device stays usable."""
    import ctypes

    from paper_2501_09398_b200 import _lib

    class _Shape:  # shape-only state: no host memory behind it
        def __init__(self, shape):
            self.temperature = np.lib.stride_tricks.as_strided(np.zeros(1), shape, [0] * len(shape))
            self.power = self.temperature
            self.diffusion_coefficient = 0.1

    wl.release_cached_contexts()
    L = _lib.lib()
    free0 = ctypes.c_int64()
    _lib.check(L.ib_mem_info(0, ctypes.byref(free0), None))
    with pytest.raises(MemoryError):
        wl.DeviceSolver(_Shape((4096, 4096, 512)), "f64", upload=False)
    free1 = ctypes.c_int64()
    _lib.check(L.ib_mem_info(0, ctypes.byref(free1), None))
    assert free1.value >= free0.value - (64 << 20)  # nothing left allocated (allocator granularity)
    state = cli.build_workload("hotspot2d", [64])
    want = ocpu.hotspot(state.temperature, state.power, state.diffusion_coefficient, 3, np.float64)
    got = wl.run_batched(wl.hotspot_program(), state, 3, 1).temperature
    assert np.array_equal(got, want)

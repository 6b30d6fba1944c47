"""The reference's property and physics tests, run against the device path.

Restated from /root/reference/pkg/tests/test_workloads.py (hotspot properties, vector laws),
test_fdtd.py (energy invariant, E<->H swap, TE101 frequency) and test_acceptance.py:296-342
(cavity physics gate). binary64 keeps the reference's bounds (1e-12 energy drift); the binary32
bound is 1e-6 (measured 2.9e-7 in SURVEY.md App. B.1).
"""

import math

import numpy as np
import pytest

from oracle import cpu as ocpu
from paper_2501_09398_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def electric_energy(w):
    squares = np.sum(w.ex**2) + np.sum(w.ey**2) + np.sum(w.ez**2)
    return 0.5 * wl.VACUUM_PERMITTIVITY * w.cell_size**3 * float(squares)


def magnetic_cross_energy(before, after):
    dots = np.sum(before.hx * after.hx) + np.sum(before.hy * after.hy) + np.sum(before.hz * after.hz)
    return 0.5 * wl.VACUUM_PERMEABILITY * before.cell_size**3 * float(dots)


@pytest.mark.parametrize("dtype,bound", [("f64", 1e-12), ("f32", 1e-6)])
def test_energy_is_conserved(gpu, dtype, bound):
    # test_fdtd.py:178-189
    state = wl.te101_cavity(16, 8, 16)
    energies = []
    for _ in range(300):
        after_h = wl.fdtd_h_step(state, dtype=dtype)
        energies.append(electric_energy(state) + magnetic_cross_energy(state, after_h))
        state = wl.fdtd_e_step(after_h, dtype=dtype)
    drift = (max(energies) - min(energies)) / energies[0]
    assert energies[0] > 0.0 and drift < bound


def test_energy_swaps_between_field_types(gpu):
    # test_fdtd.py:192-205
    w = wl.te101_cavity(16, 8, 16)
    freq = (wl.VACUUM_LIGHT_SPEED / 2.0) * math.hypot(1.0 / 16.0, 1.0 / 16.0)
    quarter = int(round(0.25 / (freq * w.time_step)))
    state = wl.run_loop(wl.fdtd_program(), w, quarter)
    after_h = wl.fdtd_h_step(state)
    share = magnetic_cross_energy(state, after_h) / (
        electric_energy(state) + magnetic_cross_energy(state, after_h))
    assert share > 0.9


@pytest.mark.parametrize("dims,steps", [((16, 4, 16), 2048), ((32, 8, 32), 4096)])
def test_resonant_frequency_matches_analytic_mode(gpu, dims, steps):
    # test_fdtd.py:208-222 and test_acceptance.py:296-321; the probe is read from the device
    # state after every iteration of one resident context
    nx, ny, nz = dims
    w = wl.te101_cavity(nx, ny, nz)
    s = wl.DeviceSolver(w, "f64")
    ey_shape = w.ey.shape
    probe = np.empty(steps)
    buf = np.empty(ey_shape)
    for n in range(steps):
        s.run_stream(1)
        probe[n] = s.download_field(1, buf)[nx // 2, ny // 2, nz // 2]
    s.close()
    spectrum = np.abs(np.fft.rfft(probe))
    peak = int(np.argmax(spectrum[1:])) + 1
    measured = peak / (steps * w.time_step)
    analytic = (wl.VACUUM_LIGHT_SPEED / 2.0) * math.hypot(1.0 / (nx * w.cell_size), 1.0 / (nz * w.cell_size))
    assert abs(measured - analytic) / analytic < 0.02


def test_quiet_cavity_stays_quiet(gpu):
    out = wl.run_loop(wl.fdtd_program(), wl.fdtd_cavity(5, 4, 3), 5)
    for arr in out.state_arrays():
        assert not arr.any()


def test_e_step_grounds_tangential_walls(gpu):
    base = wl.fdtd_cavity(6, 5, 4)
    dirty = wl.FdtdWorkload(np.ones_like(base.ex), np.ones_like(base.ey), np.ones_like(base.ez),
                            base.hx, base.hy, base.hz, base.cell_size, base.time_step)
    out = wl.fdtd_e_step(dirty)
    assert not out.ex[:, 0, :].any() and not out.ex[:, -1, :].any()
    assert not out.ex[:, :, 0].any() and not out.ex[:, :, -1].any()
    assert not out.ey[0].any() and not out.ey[-1].any()
    assert not out.ey[:, :, 0].any() and not out.ey[:, :, -1].any()
    assert not out.ez[0].any() and not out.ez[-1].any()
    assert not out.ez[:, 0, :].any() and not out.ez[:, -1, :].any()


# ---- hotspot properties (test_workloads.py:114-159) ---------------------------------------------
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_hotspot_uniform_field_is_fixed_point(gpu, dtype):
    w = wl.HotspotWorkload(np.full((9, 7), 3.25), np.zeros((9, 7)), 0.25)
    out = wl.run_loop(wl.hotspot_program(), w, 5, dtype=dtype)
    assert np.array_equal(out.temperature, w.temperature)


def test_hotspot_zero_power_respects_maximum_principle(gpu):
    rng = np.random.default_rng(7)
    cur = wl.HotspotWorkload(rng.random((12, 9)), np.zeros((12, 9)), 0.25)
    for _ in range(10):
        nxt = wl.hotspot_step(cur)
        assert nxt.temperature.max() <= cur.temperature.max() + 1e-15
        assert nxt.temperature.min() >= cur.temperature.min() - 1e-15
        cur = nxt


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_hotspot_2d_preserves_grid_symmetry_exactly(gpu, dtype):
    temp = np.zeros((9, 9))
    temp[4, 4] = 1.0
    temp[2, 4] = temp[6, 4] = 0.25
    temp[4, 2] = temp[4, 6] = 0.25
    out = wl.run_loop(wl.hotspot_program(), wl.HotspotWorkload(temp, np.zeros_like(temp), 0.25), 6,
                      dtype=dtype)
    t = out.temperature
    assert np.array_equal(t, t[::-1, :]) and np.array_equal(t, t[:, ::-1]) and np.array_equal(t, t.T)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_hotspot_3d_preserves_grid_symmetry_exactly(gpu, dtype):
    temp = np.zeros((7, 7, 7))
    temp[3, 3, 3] = 1.0
    out = wl.run_loop(wl.hotspot_program(), wl.HotspotWorkload(temp, np.zeros_like(temp), 1.0 / 6.0),
                      4, dtype=dtype)
    t = out.temperature
    for axis in range(3):
        assert np.array_equal(t, np.flip(t, axis=axis))
    assert np.array_equal(t, t.transpose(1, 0, 2))


def test_hotspot_energy_budget_with_insulated_edges(gpu):
    rng = np.random.default_rng(7)
    w = wl.HotspotWorkload(rng.random((12, 9)), rng.random((12, 9)) * 1e-3, 0.25)
    out = wl.run_loop(wl.hotspot_program(), w, 8)
    assert out.temperature.sum() == pytest.approx(w.temperature.sum() + 8 * w.power.sum(), rel=1e-12)


def test_vector_laws(gpu):
    rng = np.random.default_rng(3)
    w = wl.VectorWorkload(rng.random(64), 1.0)
    assert np.array_equal(wl.run_loop(wl.vector_program(), w, 10).values, w.values)
    w = wl.VectorWorkload(rng.random(64), 0.5)
    assert np.array_equal(wl.run_loop(wl.vector_program(), w, 8).values, w.values * 0.5**8)
    w = wl.VectorWorkload(rng.random(64), 3.0)
    np.testing.assert_allclose(wl.run_loop(wl.vector_program(), w, 12).values, w.values * 3.0**12,
                               rtol=1e-12)


def test_driver_edge_cases(gpu):
    w = wl.VectorWorkload(np.arange(1.0, 9.0), 0.5)
    assert wl.run_loop(wl.vector_program(), w, 0) is w
    assert wl.run_batched(wl.vector_program(), w, 3, 0) is w
    with pytest.raises(ValueError):
        wl.run_loop(wl.vector_program(), w, -1)
    with pytest.raises(ValueError):
        wl.run_batched(wl.vector_program(), w, 0, 5)
    with pytest.raises(ValueError):
        wl.run_batched(wl.vector_program(), w, 2, -1)
    with pytest.raises(ValueError):  # program/state mismatch
        wl.run_loop(wl.hotspot_program(), w, 1)
    s = wl.DeviceSolver(w)
    with pytest.raises(RuntimeError):  # run before build
        s.run_graph(1)
    with pytest.raises(ValueError):  # wrong host size
        s.upload([np.zeros(3)])
    s.close()


def test_time_workload_series(gpu):
    w = wl.VectorWorkload(np.random.default_rng(1).random(32), 0.9)
    plan = wl.BatchPlan(6, 2, 3)
    series = wl.time_workload(wl.vector_program(), w, plan, wl.ExecutionOrder.BATCHED, repeats=4,
                              label="demo")
    assert series.label == "demo" and len(series.points) == 1
    assert series.points[0].batch_size == 2 and len(series.points[0].samples) == 4
    assert all(s > 0 for s in series.points[0].samples)
    ph = wl.time_workload_phases(wl.vector_program(), w, plan, wl.ExecutionOrder.BATCHED, 3)
    assert all(c > 0 for c in ph["creation"]) and all(e > 0 for e in ph["execution"])
    assert all(t[0].nodes == 2 for t in ph["times"])


def test_real_trace_is_consistent(gpu, tmp_path):
    """Traced graph and stream runs: one record per kernel, ordered, in the reference schema."""
    from paper_2501_09398_b200 import cli, trace as tr

    state = cli.build_workload("hotspot2d", [256])
    s = wl.DeviceSolver(state, "f32")
    g = tr.capture_graph(s, 25, 4)
    st = tr.capture_stream(s, 100)
    assert g.kernels.shape == (100, 2) and st.kernels.shape == (100, 2)
    for k in (g.kernels, st.kernels):
        assert np.all(k[:, 1] >= k[:, 0]) and np.all(k[1:, 0] >= k[:-1, 0])
    ts = [e[0] for e in g.events]
    assert ts == sorted(ts)
    kinds = {e[1] for e in g.events}
    assert {"node_added", "graph_instantiated", "graph_uploaded", "graph_launched",
            "kernel_started", "kernel_ended", "batch_gap_started"} <= kinds
    p = tr.derive_parameters(g, st)
    # CUPTI stamps kernel ends a few tens of ns late, so back-to-back graph kernels can show a
    # slightly negative gap; the params file clamps at 0 (write_params)
    assert 0 < p["t_k"] < 1e-3 and p["t_i"] > -0.5e-6 and p["t_b"] > -0.5e-6 and p["k_c"] > 0
    path = tmp_path / "g.csv"
    tr.write_trace_csv(g, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "# schema=1" and lines[1] == "timestamp,kind,batch_index,kernel_index"
    # tracing off again: results unaffected, no records
    want = ocpu.hotspot(state.temperature, state.power, state.diffusion_coefficient, 10, np.float32)
    ref = wl.run_loop(wl.hotspot_program(), state, 10, dtype="f32")
    assert np.array_equal(np.asarray(ref.temperature, np.float32), want), "cached-context run_loop"
    s.upload(state)
    s.run_stream(10)
    got = s.download(state)
    assert np.array_equal(np.asarray(got.temperature, np.float32), want), "traced solver after tracing"
    assert s.checksum() != 0
    s.close()


def test_contexts_release_their_device_memory(gpu):
    """Create / run / destroy contexts of every solver repeatedly: device memory returns to its
    starting level (no leaked fields, lattices, graphs or IPC / counter blocks)."""
    import ctypes

    from paper_2501_09398_b200 import _lib, cli

    wl.release_cached_contexts()
    L = _lib.lib()

    def free_bytes():
        f, t = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.ib_mem_info(0, ctypes.byref(f), ctypes.byref(t)))
        return f.value

    def cycle():
        for w, size, kw in (("vector", [4096], {}), ("hotspot2d", [64, 96], {}), ("hotspot3d", [24, 16, 8], {}),
                            ("fdtd", [12, 9, 14], {}), ("fdtd", [12, 9, 14], {"fuse": True}),
                            ("hotspot3d", [40, 16, 8], {"devices": [0, 0, 0]})):
            s = wl.DeviceSolver(cli.build_workload(w, size), "f32", **kw)
            s.run_batched(3, 2, pdl=True)
            s.build_graph(5, while_loop=("devices" not in kw))
            s.run_graph(1)
            s.close()

    cycle()  # first use: lazy module loading, driver pools
    before = free_bytes()
    for _ in range(5):
        cycle()
    after = free_bytes()
    assert before - after < (64 << 20), (before, after)

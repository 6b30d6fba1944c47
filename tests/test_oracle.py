"""The CPU oracle is pinned to the reference before anything is checked against it.

* C oracle (binary64) final-state checksums == the reference's golden checksums (kats.json)
* C oracle == reference fixtures (fixtures.npz), array for array
* numpy port == C oracle bit for bit, in binary64 and binary32 (two independent restatements)
* C FNV-1a == the reference's pure-Python FNV-1a (workloads.py:513-517)
"""

import numpy as np
import pytest

from oracle import cpu as ocpu
from oracle import numpy_port as npo
from paper_2501_09398_b200 import cli


def _fnv_py(data: bytes, h=0xCBF29CE484222325):  # workloads.py:513-517, verbatim algorithm
    for byte in data:
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _oracle_state(name, state, n, dtype=np.float64):
    if name == "vector":
        return (ocpu.vector(state.values, state.scale_constant, n, dtype),)
    if name.startswith("hotspot"):
        return (ocpu.hotspot(state.temperature, state.power, state.diffusion_coefficient, n, dtype),
                np.asarray(state.power, dtype))
    d, dt = state.cell_size, state.time_step
    c_h, c_e = npo.fdtd_coefficients(d, dt)
    return ocpu.fdtd(state.state_arrays(), d, c_h, c_e, n, dtype)


def _cells(workload, size):
    s = [int(x) for x in size.split(",")]
    if workload == "vector":
        return s[0]
    if workload == "hotspot2d":
        return s[0] * s[-1]
    if workload == "hotspot3d":
        return {1: s[0] ** 3, 2: s[0] * s[0] * s[-1], 3: int(np.prod(s))}[len(s)]
    return 6 * (s[0] ** 3 if len(s) == 1 else int(np.prod(s)))


def _cheap(k):
    return _cells(k["workload"], k["size"]) * k["iterations"] <= 1.2e9


def test_fnv_matches_reference_algorithm():
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 8, 1000):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert ocpu.fnv1a64(b) == _fnv_py(b)
    a = rng.random(37).astype(np.float32)
    assert ocpu.checksum([a]) == _fnv_py(a.astype("<f8").tobytes())


def test_oracle_matches_reference_checksums(kats):
    checked = 0
    for k in kats:
        if not _cheap(k):
            continue
        state = cli.build_workload(k["workload"], [int(x) for x in k["size"].split(",")])
        got = ocpu.checksum(_oracle_state(k["workload"], state, k["iterations"]))
        assert f"{got:016x}" == k["checksum"], k
        checked += 1
    assert checked >= 20


def test_oracle_matches_reference_fixtures(fixtures):
    f = fixtures
    assert np.array_equal(ocpu.vector(f["vector_in"], 0.9999, 60), f["vector_out60"])
    assert np.array_equal(ocpu.hotspot(f["hot2_T"], f["hot2_P"], 0.2, 12), f["hot2_out12"])
    assert np.array_equal(ocpu.hotspot(f["hot3_T"], f["hot3_P"], 0.125, 5), f["hot3_out5"])
    names = ("ex", "ey", "ez", "hx", "hy", "hz")
    for tag, n_steps, out in (("fdtd_in_", 12, "fdtd_out12_"), ("dirty_in_", 3, "dirty_out3_")):
        sc = f["fdtd_scalars"] if tag == "fdtd_in_" else f["dirty_scalars"]
        c_h, c_e = npo.fdtd_coefficients(*sc)
        got = ocpu.fdtd([f[tag + n] for n in names], sc[0], c_h, c_e, n_steps)
        for n, a in zip(names, got):
            assert np.array_equal(a, f[out + n]), (tag, n)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_numpy_port_equals_c_oracle_bitwise(dtype):
    rng = np.random.default_rng(12)
    v = rng.random(1001)
    want = ocpu.vector(v, 0.9999, 40, dtype)
    assert np.array_equal(npo.run_vector(v.astype(dtype), 0.9999, 40), want)
    for shape in ((17, 23), (9, 11, 5), (1, 1), (1, 6, 1)):
        t, p = rng.random(shape), rng.random(shape) * 1e-3
        k = 0.1
        want = ocpu.hotspot(t, p, k, 15, dtype)
        got = npo.run_hotspot(t.astype(dtype), p.astype(dtype), k, 15)
        assert np.array_equal(got, want), shape
    w = cli.build_workload("fdtd", [7, 5, 6])
    c_h, c_e = npo.fdtd_coefficients(w.cell_size, w.time_step)
    fields = [a.astype(dtype) for a in w.state_arrays()]
    got = npo.run_fdtd(fields, w.cell_size, c_h, c_e, 20)
    want = ocpu.fdtd(w.state_arrays(), w.cell_size, c_h, c_e, 20, dtype)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_numpy_port_slab_threading_is_bit_identical():
    rng = np.random.default_rng(4)
    t, p = rng.random((40, 30)), rng.random((40, 30)) * 1e-3
    ref = npo.run_hotspot(t, p, 0.2, 6)
    pool = npo.SlabPool(3)
    try:
        assert np.array_equal(npo.run_hotspot(t, p, 0.2, 6, pool), ref)
    finally:
        pool.close()

"""Randomised shapes, batch sizes and launch options for every solver, bit-exact against the C
oracle (binary32 and binary64). Seeded: a failure prints its case and reproduces."""

import os

import numpy as np
import pytest

from oracle import cpu as ocpu
from paper_2501_09398_b200 import workloads as wl
from tests.conftest import spread

pytestmark = pytest.mark.gpu


def _cases(n, seed):
    """n cases (IB_FUZZ_SCALE multiplies them for a long soak; the seed stays the same, so a
    failing case reproduces by its index)."""
    rng = np.random.default_rng(seed)
    for c in range(n * int(os.environ.get("IB_FUZZ_SCALE", "1"))):
        yield c, rng


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_fuzz_hotspot(gpu, dtype):
    npd = np.float32 if dtype == "f32" else np.float64
    for c, rng in _cases(40, 101 if dtype == "f32" else 102):
        d3 = bool(rng.integers(2))
        if d3:
            shape = (int(rng.integers(1, 40)), int(rng.integers(1, 40)), int(rng.choice([1, 2, 3, 4, 8, 12, 16, 64])))
        else:
            shape = (int(rng.integers(1, 70)), int(rng.choice([1, 3, 4, 8, 32, 100, 128, 256, 260])))
        k = float(rng.choice([0.05, 0.1, 0.15])) if d3 else float(rng.choice([0.1, 0.2, 0.25]))
        st = wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, k)
        kk = int(rng.integers(1, 6))
        nb = int(rng.integers(1, 4))
        slabs = int(rng.integers(1, 4)) if shape[0] >= 3 else 1
        pdl = bool(rng.integers(2))
        want = ocpu.hotspot(st.temperature, st.power, k, kk * nb, npd)
        got = wl.run_batched(wl.hotspot_program(), st, kk, nb, dtype=dtype, pdl=pdl and slabs == 1,
                             devices=spread(slabs) if slabs > 1 else None,
                             build="capture" if slabs > 1 else "manual").temperature
        assert np.array_equal(np.asarray(got, npd), want), (c, shape, k, kk, nb, slabs, pdl)
    wl.release_cached_contexts()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_fuzz_fdtd(gpu, dtype):
    npd = np.float32 if dtype == "f32" else np.float64
    for c, rng in _cases(30, 201 if dtype == "f32" else 202):
        dims = tuple(int(x) for x in rng.integers(1, 24, size=3))
        d = float(rng.choice([1.0, 1.0, 0.5, 0.37]))
        base = wl.fdtd_cavity(*dims, cell_size=d)
        st = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()], base.cell_size,
                             base.time_step)
        kk = int(rng.integers(1, 5))
        nb = int(rng.integers(1, 3))
        fuse = bool(rng.integers(2))
        slabs = 1 if fuse or dims[0] < 2 else int(rng.integers(1, 4))
        dt = st.time_step
        want = ocpu.fdtd(st.state_arrays(), d, dt / wl.VACUUM_PERMEABILITY, dt / wl.VACUUM_PERMITTIVITY,
                         kk * nb, npd)
        got = wl.run_batched(wl.fdtd_program(), st, kk, nb, dtype=dtype, fuse=fuse,
                             devices=spread(slabs) if slabs > 1 else None,
                             build="capture" if slabs > 1 else "manual").state_arrays()
        for g, w in zip(got, want):
            assert np.array_equal(np.asarray(g, npd), w), (c, dims, d, kk, nb, fuse, slabs)
    wl.release_cached_contexts()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_fuzz_vector(gpu, dtype):
    npd = np.float32 if dtype == "f32" else np.float64
    for c, rng in _cases(20, 301 if dtype == "f32" else 302):
        n = int(rng.integers(1, 5000))
        cst = float(rng.choice([0.9999, 0.5, 1.0, 0.75]))
        st = wl.VectorWorkload(rng.random(n), cst)
        kk, nb = int(rng.integers(1, 8)), int(rng.integers(1, 4))
        want = ocpu.vector(st.values, cst, kk * nb, npd)
        got = wl.run_batched(wl.vector_program(), st, kk, nb, dtype=dtype, pdl=bool(rng.integers(2))).values
        assert np.array_equal(np.asarray(got, npd), want), (c, n, cst, kk, nb)
    wl.release_cached_contexts()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_large_vector_grid_stride(gpu, dtype):
    """Vectors beyond one wave of threads take 1024-thread CTAs and a grid-stride loop."""
    npd = np.float32 if dtype == "f32" else np.float64
    rng = np.random.default_rng(7)
    for n in (5_000_003, 3 * 1024 * 1024 * 4 + 2):
        st = wl.VectorWorkload(rng.random(n), 0.9999)
        want = ocpu.vector(st.values, 0.9999, 6, npd)
        got = wl.run_batched(wl.vector_program(), st, 3, 2, dtype=dtype, pdl=True).values
        assert np.array_equal(np.asarray(got, npd), want), n
    wl.release_cached_contexts()

"""Every kernel variant the launch layer can pick is bit-identical to the oracle.

The runtime chooses between kernel variants by shape and size: for hotspot the
scalar march, the 16-byte vectorised row kernel and the cp.async.bulk (TMA) plane-march pipeline;
for FDTD the staged k_fdtd_lf modes (fused, H, E) at every tile height / chunking and the lean
fallback. IB_HOTSPOT_KERNEL / IB_HOTSPOT_VEC_ROWS / IB_HOTSPOT_RPC / IB_TMA_STAGES /
IB_FDTD_KERNEL / IB_FDTD_TJ / IB_FDTD_CHUNKS / IB_FDTD_TILES / IB_FDTD_CTAS force a choice, so
each variant is checked here at
shapes its automatic choice would not reach (ragged tiles, tiny chunks, slabs, binary64).
"""

import os

import numpy as np
import pytest

from oracle import cpu as ocpu
from paper_2501_09398_b200 import workloads as wl
from tests.conftest import spread

pytestmark = pytest.mark.gpu


@pytest.fixture
def env():
    saved = {}

    def set_(**kw):
        for k, v in kw.items():
            saved.setdefault(k, os.environ.get(k))
            os.environ[k] = str(v)

    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    wl.release_cached_contexts()


HOT_SHAPES = [(64, 48), (33, 1024), (7, 4100), (1, 8), (40, 12, 8), (9, 20, 256), (5, 3, 512),
              (17, 6, 4), (2, 2, 4), (11, 7, 16), (3, 1, 8), (1, 1, 16), (13, 16)]


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kernel", ["scalar", "vec", "tma"])
@pytest.mark.parametrize("shape", HOT_SHAPES, ids=["x".join(map(str, s)) for s in HOT_SHAPES])
def test_hotspot_variant_bitwise(gpu, env, shape, kernel, dtype):
    env(IB_HOTSPOT_KERNEL=kernel)
    rng = np.random.default_rng(len(shape) * 1000 + shape[0])
    k = 0.1 if len(shape) == 3 else 0.2
    state = wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, k)
    npd = np.float32 if dtype == "f32" else np.float64
    want = ocpu.hotspot(state.temperature, state.power, k, 7, npd)
    got = wl.run_batched(wl.hotspot_program(), state, 7, 1, dtype=dtype).temperature
    assert np.array_equal(np.asarray(got, npd), want)
    got = wl.run_loop(wl.hotspot_program(), state, 7, dtype=dtype, pdl=True).temperature
    assert np.array_equal(np.asarray(got, npd), want)


@pytest.mark.parametrize("rpc,stages", [(1, 3), (2, 3), (3, 4), (5, 8), (64, 4)])
def test_hotspot_tma_chunking_and_ring_depth(gpu, env, rpc, stages):
    env(IB_HOTSPOT_KERNEL="tma", IB_HOTSPOT_RPC=rpc, IB_TMA_STAGES=stages)
    rng = np.random.default_rng(rpc * 31 + stages)
    for shape in ((23, 16, 256), (29, 40, 8), (31, 2048)):
        state = wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, 0.1)
        want = ocpu.hotspot(state.temperature, state.power, 0.1, 5, np.float32)
        got = wl.run_batched(wl.hotspot_program(), state, 5, 1, dtype="f32").temperature
        assert np.array_equal(np.asarray(got, np.float32), want), shape


@pytest.mark.parametrize("bx", [32, 256])
@pytest.mark.parametrize("shuffle", [0, 1, 2])
@pytest.mark.parametrize("rows,block", [(1, 256), (2, 256), (4, 256), (1, 1024), (2, 512), (4, 64)])
def test_hotspot_vec_rows_per_thread(gpu, env, rows, block, shuffle, bx):
    """The vectorised kernel with every rows-per-thread choice and 2-D CTA shapes (row-blocks
    per CTA, CTA width capped at bx threads), ragged last row chunk and partially idle CTAs
    included."""
    env(IB_HOTSPOT_KERNEL="vec", IB_HOTSPOT_VEC_ROWS=rows, IB_HOTSPOT_BLOCK=block, IB_HOTSPOT_SHUFFLE=shuffle,
        IB_HOTSPOT_BX=bx)
    rng = np.random.default_rng(rows)
    # shapes with whole warps per row (the shuffle path: 32 groups of 4/2 cells) and without
    for shape in ((23, 16, 8), (30, 5, 4), (9, 3, 16), (31, 64), (6, 8), (7, 64, 8), (5, 32, 16),
                  (9, 128, 4), (6, 256), (4, 512, 32), (3, 3, 128), (11, 2048)):
        for dtype, npd in (("f32", np.float32), ("f64", np.float64)):
            state = wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, 0.1)
            want = ocpu.hotspot(state.temperature, state.power, 0.1, 5, npd)
            got = wl.run_batched(wl.hotspot_program(), state, 5, 1, dtype=dtype, pdl=True).temperature
            assert np.array_equal(np.asarray(got, npd), want), (shape, dtype)


@pytest.mark.parametrize("kernel", ["vec", "tma", "scalar"])
@pytest.mark.parametrize("slabs", [2, 3, 5])
def test_hotspot_variants_with_slabs(gpu, env, kernel, slabs):
    env(IB_HOTSPOT_KERNEL=kernel, IB_HOTSPOT_RPC=3)
    rng = np.random.default_rng(slabs)
    for shape in ((30, 12, 8), (41, 64)):
        state = wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, 0.1)
        want = ocpu.hotspot(state.temperature, state.power, 0.1, 6, np.float64)
        got = wl.run_batched(wl.hotspot_program(), state, 3, 2, devices=spread(slabs), build="capture")
        assert np.array_equal(got.temperature, want), shape


@pytest.mark.parametrize("kernel", ["vec", "tma", "scalar"])
@pytest.mark.parametrize("slabs", [2, 3])
def test_hotspot_slabs_copy_exchange(gpu, env, kernel, slabs):
    """IB_HALO_COPY: the slab kernels write only their own rows and
    cudaMemcpyPeerAsync moves the halo faces — == oracle in stream mode, per-step calls and
    captured graphs at odd and even K, and equal to the fused-store exchange (v2)."""
    env(IB_HOTSPOT_KERNEL=kernel, IB_HOTSPOT_RPC=3)
    rng = np.random.default_rng(40 + slabs)
    for shape in ((30, 12, 8), (41, 64)):
        state = wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, 0.1)
        want = ocpu.hotspot(state.temperature, state.power, 0.1, 6, np.float64)
        with wl.DeviceSolver(state, "f64", devices=spread(slabs), halo="copy") as s:
            d = s.describe()  # kernels plus the peer-copy nodes after each (2 per interior slab)
            assert sum(e.get("memcpy_nodes", 0) for e in d) == 2 * (slabs - 1)
            s.run_stream(6)
            assert np.array_equal(s.download(state).temperature, want), shape
            s.upload(state)
            for _ in range(6):
                s.run_step(0)
            assert np.array_equal(s.download(state).temperature, want), shape
            for k, n in ((3, 2), (2, 3), (6, 1)):
                s.upload(state)
                s.run_batched(k, n, build="capture", pdl=True)
                assert np.array_equal(s.download(state).temperature, want), (shape, k)
        got = wl.run_batched(wl.hotspot_program(), state, 3, 2, devices=spread(slabs), build="capture",
                             halo="copy")  # the module-level drivers take the option too
        assert np.array_equal(got.temperature, want), shape
        with wl.DeviceSolver(state, "f32", devices=spread(slabs), halo="copy") as s, \
                wl.DeviceSolver(state, "f32", devices=spread(slabs)) as v2:
            s.run_batched(3, 2, build="capture")
            v2.run_batched(3, 2, build="capture")
            assert np.array_equal(s.download(state).temperature, v2.download(state).temperature)


def test_halo_mode_validation(gpu):
    rng = np.random.default_rng(3)
    hot = wl.HotspotWorkload(rng.random((8, 16)), rng.random((8, 16)) * 1e-3, 0.1)
    with pytest.raises(ValueError):
        wl.DeviceSolver(hot, "f32", halo="nvlink")
    with wl.DeviceSolver(hot, "f32", halo="copy") as s:  # one slab: accepted, nothing to exchange
        s.run_stream(2)
    with wl.DeviceSolver(wl.fdtd_cavity(6, 4, 6), "f32", devices=spread(2), halo="copy") as s:
        s.run_stream(2)  # FDTD slabs take the copy exchange too


@pytest.mark.parametrize("halo", ["store", "copy"])
@pytest.mark.parametrize("fuse", [False, True], ids=["two-half-steps", "fused"])
def test_fdtd_slabs_peeled_and_per_step(gpu, fuse, halo):
    """Slabs through the other drivers: loop peeling (N not divisible by K, a remainder graph) and
    the per-step API (ib_run_step) == the oracle, for both FDTD solvers and both halo exchanges."""
    base = wl.fdtd_cavity(9, 5, 11)
    rng = np.random.default_rng(77)
    state = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()], base.cell_size,
                            base.time_step)
    dt = state.time_step
    want = ocpu.fdtd(state.state_arrays(), 1.0, dt / wl.VACUUM_PERMEABILITY,
                     dt / wl.VACUUM_PERMITTIVITY, 7, np.float64)
    got = wl.run_peeled(wl.fdtd_program(), state, 7, 3, devices=spread(3), fuse=fuse, halo=halo,
                        build="capture")
    for g, w in zip(got.state_arrays(), want):
        assert np.array_equal(g, w)
    with wl.DeviceSolver(state, "f64", devices=spread(3), fuse=fuse, halo=halo) as s:
        for _ in range(7):
            for step in range(1 if fuse else 2):
                s.run_step(step)
        for g, w in zip(s.download(state).state_arrays(), want):
            assert np.array_equal(g, w)


FDTD_DIMS = [(8, 4, 8), (5, 6, 7), (1, 1, 1), (3, 1, 9), (16, 9, 33), (2, 40, 3)]


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kernel,tj,chunks", [("lean", 0, 0), ("lean-scalar", 0, 0), ("staged", 0, 0), ("staged", 1, 0),
                                              ("staged", 2, 3), ("staged", 3, 1), ("staged", 4, 2)])
@pytest.mark.parametrize("dims", FDTD_DIMS, ids=["x".join(map(str, d)) for d in FDTD_DIMS])
def test_fdtd_variant_bitwise(gpu, env, dims, kernel, tj, chunks, dtype):
    """The two half-step launches per iteration (in place on the padded lattice): the staged
    k_fdtd_lf H / E modes at every tile height and chunking, and the lean fallback, == oracle."""
    env(IB_FDTD_KERNEL=kernel.split("-")[0], IB_FDTD_TJ=tj, IB_FDTD_CHUNKS=chunks,
        IB_FDTD_LEANV=0 if kernel == "lean-scalar" else 1)
    base = wl.fdtd_cavity(*dims)
    rng = np.random.default_rng(sum(dims) + tj + chunks)
    state = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()],
                            base.cell_size, base.time_step)
    npd = np.float32 if dtype == "f32" else np.float64
    dt = state.time_step
    want = ocpu.fdtd(state.state_arrays(), 1.0, dt / wl.VACUUM_PERMEABILITY,
                     dt / wl.VACUUM_PERMITTIVITY, 4, npd)
    got = wl.run_batched(wl.fdtd_program(), state, 2, 2, dtype=dtype, pdl=True)
    for g, w in zip(got.state_arrays(), want):
        assert np.array_equal(np.asarray(g, npd), w)
    got = wl.run_loop(wl.fdtd_program(), state, 4, dtype=dtype)
    for g, w in zip(got.state_arrays(), want):
        assert np.array_equal(np.asarray(g, npd), w)


def test_fdtd_non_unit_cell_size(gpu, env):
    """d != 1 exercises the division path (skipped exactly when d == 1)."""
    for kernel in ("lean", "staged"):
        env(IB_FDTD_KERNEL=kernel)
        w = wl.te101_cavity(6, 5, 7, cell_size=0.37)
        dt = w.time_step
        want = ocpu.fdtd(w.state_arrays(), 0.37, dt / wl.VACUUM_PERMEABILITY,
                         dt / wl.VACUUM_PERMITTIVITY, 9, np.float64)
        got = wl.run_loop(wl.fdtd_program(), w, 9)
        for g, ww in zip(got.state_arrays(), want):
            assert np.array_equal(g, ww)


def test_fdtd_long_z_rows_fall_back_to_lean(gpu):
    """z rows too long for the staged kernel's CTA: the two-launch solver takes the lean kernels,
    the fused solver refuses with ValueError (no silent change of algorithm)."""
    base = wl.fdtd_cavity(2, 2, 1600)
    rng = np.random.default_rng(5)
    state = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()],
                            base.cell_size, base.time_step)
    dt = state.time_step
    want = ocpu.fdtd(state.state_arrays(), 1.0, dt / wl.VACUUM_PERMEABILITY,
                     dt / wl.VACUUM_PERMITTIVITY, 3, np.float32)
    got = wl.run_loop(wl.fdtd_program(), state, 3, dtype="f32")
    for g, w in zip(got.state_arrays(), want):
        assert np.array_equal(np.asarray(g, np.float32), w)
    with pytest.raises(ValueError):
        wl.run_loop(wl.fdtd_program(), state, 3, dtype="f32", fuse=True)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("tj,ctas,chunks,tiles", [(0, 0, 0, 0), (1, 0, 0, 0), (2, 5, 0, 0), (3, 1, 0, 0),
                                                  (4, 7, 0, 0), (4, 13, 0, 0), (2, 0, 3, 0), (4, 0, 1, 0),
                                                  (1, 0, 4, 0), (4, 0, 2, 3), (3, 0, 1, 7), (4, 9, 0, 5)])
@pytest.mark.parametrize("dims", FDTD_DIMS + [(40, 9, 70), (7, 17, 31)],
                         ids=["x".join(map(str, d)) for d in FDTD_DIMS + [(40, 9, 70), (7, 17, 31)]])
def test_fdtd_fused_bitwise(gpu, env, dims, tj, ctas, chunks, tiles, dtype):
    """One kernel per iteration (H then E fused, double-buffered padded lattice) == the oracle,
    bitwise, for every tile height, uneven row splits (tiles of h <= TJ rows), lockstep chunk
    grids and CTA counts that split the (tile, plane) units into runs starting mid-tile (the
    recomputed seed plane) and spanning several tiles."""
    env(IB_FDTD_TJ=tj, IB_FDTD_CTAS=ctas, IB_FDTD_CHUNKS=chunks, IB_FDTD_TILES=tiles)
    base = wl.fdtd_cavity(*dims)
    rng = np.random.default_rng(sum(dims) * 7 + tj + ctas + chunks + tiles)
    state = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()],
                            base.cell_size, base.time_step)
    npd = np.float32 if dtype == "f32" else np.float64
    dt = state.time_step
    want = ocpu.fdtd(state.state_arrays(), 1.0, dt / wl.VACUUM_PERMEABILITY,
                     dt / wl.VACUUM_PERMITTIVITY, 5, npd)
    for kw in ({"build": "manual"}, {"build": "capture", "pdl": True}):
        got = wl.run_batched(wl.fdtd_program(), state, 5, 1, dtype=dtype, fuse=True, **kw)  # odd K
        for g, w in zip(got.state_arrays(), want):
            assert np.array_equal(np.asarray(g, npd), w)
    got = wl.run_loop(wl.fdtd_program(), state, 5, dtype=dtype, fuse=True)
    for g, w in zip(got.state_arrays(), want):
        assert np.array_equal(np.asarray(g, npd), w)


@pytest.mark.parametrize("ctas", [0, 3])
def test_fdtd_fused_non_unit_cell_size(gpu, env, ctas):
    """Fused leapfrog with d != 1 (the division path) == the oracle, bitwise."""
    env(IB_FDTD_CTAS=ctas)
    w = wl.te101_cavity(6, 5, 7, cell_size=0.37)
    dt = w.time_step
    for dtype, npd in (("f64", np.float64), ("f32", np.float32)):
        want = ocpu.fdtd(w.state_arrays(), 0.37, dt / wl.VACUUM_PERMEABILITY,
                         dt / wl.VACUUM_PERMITTIVITY, 9, npd)
        got = wl.run_loop(wl.fdtd_program(), w, 9, dtype=dtype, fuse=True)
        for g, ww in zip(got.state_arrays(), want):
            assert np.array_equal(np.asarray(g, npd), ww)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("slabs", [2, 3, 5])
@pytest.mark.parametrize("dims", [(8, 4, 8), (16, 9, 33), (5, 6, 7), (40, 9, 70)],
                         ids=["8x4x8", "16x9x33", "5x6x7", "40x9x70"])
def test_fused_fdtd_slabs_equal_one_domain(gpu, env, dims, slabs, dtype):
    """The fused leapfrog split into axis-0 lattice slabs (each slab ping-pongs its planes plus a
    halo plane each side; the kernel stores its last plane's new E and H into the next slab's
    seed plane and its first plane's new E into the previous slab's upper halo) == one domain ==
    the oracle, bit for bit: graph (capture) at even and odd K, stream mode, tile / chunk
    variants."""
    if slabs > dims[0] + 1:
        pytest.skip("more slabs than planes")
    base = wl.fdtd_cavity(*dims)
    rng = np.random.default_rng(100 + sum(dims) + slabs)
    state = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()],
                            base.cell_size, base.time_step)
    npd = np.float32 if dtype == "f32" else np.float64
    dt = state.time_step
    want = ocpu.fdtd(state.state_arrays(), 1.0, dt / wl.VACUUM_PERMEABILITY,
                     dt / wl.VACUUM_PERMITTIVITY, 6, npd)
    devs = spread(slabs)
    for tj, chunks in ((0, 0), (1, 2), (3, 1)):
        env(IB_FDTD_TJ=tj, IB_FDTD_CHUNKS=chunks)
        for k, n in ((3, 2), (2, 3)):
            got = wl.run_batched(wl.fdtd_program(), state, k, n, dtype=dtype, devices=devs, build="capture",
                                 fuse=True)
            for g, w in zip(got.state_arrays(), want):
                assert np.array_equal(np.asarray(g, npd), w), (tj, chunks, k)
        got = wl.run_loop(wl.fdtd_program(), state, 6, dtype=dtype, devices=devs, fuse=True)
        for g, w in zip(got.state_arrays(), want):
            assert np.array_equal(np.asarray(g, npd), w), (tj, chunks)
    env(IB_FDTD_TJ=0, IB_FDTD_CHUNKS=0)
    for run in (lambda: wl.run_batched(wl.fdtd_program(), state, 3, 2, dtype=dtype, devices=devs,
                                       build="capture", fuse=True, halo="copy"),
                lambda: wl.run_loop(wl.fdtd_program(), state, 6, dtype=dtype, devices=devs, fuse=True,
                                    halo="copy")):
        for g, w in zip(run().state_arrays(), want):  # IB_HALO_COPY: peer-copy nodes move the halos
            assert np.array_equal(np.asarray(g, npd), w)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("slabs", [2, 3, 5])
@pytest.mark.parametrize("dims", [(8, 4, 8), (16, 9, 33), (5, 6, 7), (40, 9, 70)],
                         ids=["8x4x8", "16x9x33", "5x6x7", "40x9x70"])
def test_fdtd_slabs_equal_one_domain(gpu, env, dims, slabs, dtype):
    """FDTD split into axis-0 slabs of the lattice (halo planes pushed by the H / E launches
    into the neighbours, cross-slab graph edges) == one domain == the oracle, bit for bit, in
    graph (capture) and stream mode, with tile / chunk variants."""
    if slabs > dims[0] + 1:
        pytest.skip("more slabs than planes")
    base = wl.fdtd_cavity(*dims)
    rng = np.random.default_rng(sum(dims) + slabs)
    state = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()],
                            base.cell_size, base.time_step)
    npd = np.float32 if dtype == "f32" else np.float64
    dt = state.time_step
    want = ocpu.fdtd(state.state_arrays(), 1.0, dt / wl.VACUUM_PERMEABILITY,
                     dt / wl.VACUUM_PERMITTIVITY, 6, npd)
    devs = spread(slabs)
    for tj, chunks in ((0, 0), (1, 2), (3, 1)):
        env(IB_FDTD_TJ=tj, IB_FDTD_CHUNKS=chunks)
        got = wl.run_batched(wl.fdtd_program(), state, 3, 2, dtype=dtype, devices=devs, build="capture")
        for g, w in zip(got.state_arrays(), want):
            assert np.array_equal(np.asarray(g, npd), w), (tj, chunks)
        got = wl.run_loop(wl.fdtd_program(), state, 6, dtype=dtype, devices=devs)
        for g, w in zip(got.state_arrays(), want):
            assert np.array_equal(np.asarray(g, npd), w), (tj, chunks)
    env(IB_FDTD_TJ=0, IB_FDTD_CHUNKS=0)
    for run in (lambda: wl.run_batched(wl.fdtd_program(), state, 3, 2, dtype=dtype, devices=devs,
                                       build="capture", halo="copy"),
                lambda: wl.run_loop(wl.fdtd_program(), state, 6, dtype=dtype, devices=devs, halo="copy")):
        for g, w in zip(run().state_arrays(), want):  # IB_HALO_COPY: peer-copy nodes move the halos
            assert np.array_equal(np.asarray(g, npd), w)


def test_fdtd_shallow_staged_shape_takes_lean_kernels(gpu, env):
    """binary64 rows of 384 cells leave the staged kernel a 1-row tile or a 3-stage ring: the
    two-half-step solver runs the lean kernels there — still == oracle; forcing
    IB_FDTD_KERNEL=staged keeps the staged kernel."""
    base = wl.fdtd_cavity(48, 256, 384)  # 233 MB lattice in binary64: above the L2-resident lean rule
    rng = np.random.default_rng(11)
    state = wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()], base.cell_size,
                            base.time_step)
    with wl.DeviceSolver(state, "f64") as s:
        names = [d["kernel"] for d in s.describe()]
    assert names and all(any(f"k_fdtd_{m}" in n for m in ("h2", "e2", "h4", "e4")) for n in names), names
    env(IB_FDTD_KERNEL="staged")
    with wl.DeviceSolver(state, "f64") as s:
        assert all("k_fdtd_lf" in d["kernel"] for d in s.describe())
    dt = state.time_step
    want = ocpu.fdtd(state.state_arrays(), 1.0, dt / wl.VACUUM_PERMEABILITY, dt / wl.VACUUM_PERMITTIVITY, 2,
                     np.float64)
    for kernel in ("staged", "lean"):
        env(IB_FDTD_KERNEL=kernel)
        got = wl.run_batched(wl.fdtd_program(), state, 2, 1)
        for g, w in zip(got.state_arrays(), want):
            assert np.array_equal(g, w), kernel

"""Multi-process slabs on GPUs (ib_create_dist). World 1 runs everywhere; the NCCL halo path needs
>= 2 GPUs (one process per GPU, like torchrun) and is skipped on a single-GPU box."""

import os
import socket

import numpy as np
import pytest

from paper_2501_09398_b200 import _lib
from paper_2501_09398_b200 import workloads as wl
from paper_2501_09398_b200.distributed import DistributedSolver, unique_id

pytestmark = pytest.mark.gpu


def _state(shape, seed=3):
    rng = np.random.default_rng(seed)
    return wl.HotspotWorkload(rng.random(shape), rng.random(shape) * 1e-3, 0.1)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_world_one_equals_device_solver(gpu, dtype):
    st = _state((24, 16, 8))
    ref = wl.run_batched(wl.hotspot_program(), st, 5, 2, dtype=dtype).temperature
    d = DistributedSolver(st, dtype, rank=0, world=1, device=0, uid=None)
    d.run_batched(5, 2)
    assert np.array_equal(d.local_temperature().astype(np.float64), ref)
    d.close()


def test_nccl_is_loadable(gpu):
    uid = unique_id()
    assert len(uid) == 128 and any(uid)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, shape, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        st = _state(shape)
        d = DistributedSolver(st, "f32", rank=rank, world=world, device=rank, uid=obj[0])
        d.run_batched(5, 2)          # graph mode: kernel + NCCL group per iteration, captured
        d.run_stream(3)              # stream mode, same exchange
        parts = [None] * world
        dist.all_gather_object(parts, (d.lo, d.hi, d.local_temperature()))
        d.close()
        if rank == 0:
            full = np.empty(shape, np.float32)
            for a, b, arr in parts:
                full[a:b] = arr
            q.put(full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(64, 24, 8), (33, 40)])
def test_multi_rank_nccl_halo_equals_single_gpu(gpu, shape):
    n = _lib.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU)")
    import torch.multiprocessing as mp

    world = min(n, 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    st = _state(shape)
    want = wl.run_loop(wl.hotspot_program(), st, 13, dtype="f32").temperature
    assert np.array_equal(got.astype(np.float64), want)


def _rank_main_peer(rank, world, port, shape, kernel, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), IB_HOTSPOT_KERNEL=kernel,
                      IB_DIST_TIMEOUT_MS="60000")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def allgather(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out

        st = _state(shape)
        device = rank % _lib.device_count()  # one GPU: every rank shares device 0 (IPC still works)
        d = DistributedSolver(st, "f32", rank=rank, world=world, device=device, exchange="peer",
                              allgather=allgather)
        d.run_batched(5, 2)          # graph: wait / stencil with peer halo stores / signal
        d.run_stream(3)              # stream mode, same protocol
        first = d.local_temperature()
        d.upload(st)                 # a second run from the initial state (counters keep going)
        d.run_batched(4, 3, pdl=True)
        d.run_stream(1)
        parts = [None] * world
        dist.all_gather_object(parts, (d.lo, d.hi, first, d.local_temperature()))
        d.close()
        if rank == 0:
            a = np.empty(shape, np.float32)
            b = np.empty(shape, np.float32)
            for lo, hi, x, y in parts:
                a[lo:hi] = x
                b[lo:hi] = y
            q.put((a, b))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kernel", ["vec", "tma", "scalar"])
@pytest.mark.parametrize("world,shape", [(2, (64, 24, 8)), (3, (33, 40)), (2, (12, 16, 256)), (8, (40, 24, 8))])
def test_multi_rank_peer_halo_equals_single_gpu(gpu, kernel, world, shape):
    """One process per rank, halo planes stored straight into the neighbours' buffers (CUDA IPC)
    and ordered by device counters: == the single-domain result, bit for bit. On a one-GPU box
    the ranks share the device (IPC between processes on one device is legal), which checks the
    protocol, not the NVLink speed."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main_peer, args=(r, world, port, shape, kernel, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        a, b = q.get(timeout=240)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    st = _state(shape)
    os.environ["IB_HOTSPOT_KERNEL"] = kernel
    try:
        want_a = wl.run_loop(wl.hotspot_program(), st, 13, dtype="f32").temperature
        want_b = wl.run_loop(wl.hotspot_program(), st, 13, dtype="f32").temperature
    finally:
        os.environ.pop("IB_HOTSPOT_KERNEL", None)
        wl.release_cached_contexts()
    assert np.array_equal(a.astype(np.float64), want_a)
    assert np.array_equal(b.astype(np.float64), want_b)


def _fdtd_state(dims, seed=11):
    base = wl.fdtd_cavity(*dims)
    rng = np.random.default_rng(seed)
    return wl.FdtdWorkload(*[rng.random(a.shape) for a in base.state_arrays()], base.cell_size,
                           base.time_step)


def _rank_main_fdtd(rank, world, port, dims, dtype, q, fuse=False):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), IB_DIST_TIMEOUT_MS="60000")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def allgather(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out

        st = _fdtd_state(dims)
        device = rank % _lib.device_count()
        d = DistributedSolver(st, dtype, rank=rank, world=world, device=device, exchange="peer",
                              allgather=allgather, fuse=fuse)
        d.run_batched(3, 2)   # graph: per half-step wait / H or E with halo stores / signal
        d.run_stream(1)       # stream mode
        parts = [None] * world
        dist.all_gather_object(parts, (d.lo, d.hi, d.local_fields()))
        d.close()
        if rank == 0:
            out = [np.empty(a.shape) for a in st.state_arrays()]
            for lo, hi, fields in parts:
                for o, a in zip(out, fields):
                    o[min(lo, o.shape[0]):min(lo, o.shape[0]) + a.shape[0]] = a
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fuse", [False, True], ids=["two-half-steps", "fused"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("world,dims", [(2, (8, 4, 8)), (3, (16, 9, 33)), (2, (5, 6, 7)), (8, (20, 5, 6))])
def test_multi_rank_fdtd_peer_equals_single_domain(gpu, world, dims, dtype, fuse):
    """FDTD lattice split into one slab per process, halo planes stored into the neighbours'
    buffers through CUDA IPC with counter ordering (per half-step; per iteration for the fused
    leapfrog, whose slabs ping-pong) == one domain."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main_fdtd, args=(r, world, port, dims, dtype, q, fuse))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = q.get(timeout=240)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    st = _fdtd_state(dims)
    want = wl.run_loop(wl.fdtd_program(), st, 7, dtype=dtype).state_arrays()
    wl.release_cached_contexts()
    for g, w in zip(got, want):
        assert np.array_equal(g, w)

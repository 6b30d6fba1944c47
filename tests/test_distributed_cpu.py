"""Multi-process slab protocol on CPU (gloo, world_size 2 and 3): host-side logic of §8e.

Each rank owns rows slab_bounds(rows, world, rank) of a global Hotspot grid plus halo planes,
steps its slab, and exchanges boundary planes with its neighbours following exchange_plan — the
exact plan the runtime's NCCL group executes after every kernel (runtime.cu: nccl_exchange).
The gathered result must equal the single-domain CPU oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu as ocpu
from paper_2501_09398_b200.distributed import exchange_plan, halo_window, slab_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _local_step(buf, power, k, top_edge, bot_edge):
    """One hotspot step of the owned rows of a halo'd slab buffer (rows 0 and -1 are halos)."""
    if top_edge:
        buf[0] = buf[1]  # global edge: clamp (np.pad mode="edge", workloads.py:177)
    if bot_edge:
        buf[-1] = buf[-2]
    c = buf[1:-1]
    pad_axes = [(0, 0)] + [(1, 1)] * (buf.ndim - 1)
    p = np.pad(c, pad_axes, mode="edge")
    if buf.ndim == 2:
        y = p[:, :-2] + p[:, 2:]
        s = (buf[:-2] + buf[2:]) + y
        loss = 4.0
    else:
        y = p[:, :-2, 1:-1] + p[:, 2:, 1:-1]
        z = p[:, 1:-1, :-2] + p[:, 1:-1, 2:]
        s = ((buf[:-2] + buf[2:]) + y) + z
        loss = 6.0
    out = np.empty_like(buf)
    out[1:-1] = c + k * (s - loss * c) + power
    return out


def _worker(rank, world, port, shape, steps, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        T = rng.random(shape)
        P = rng.random(shape) * 1e-3
        rows = shape[0]
        lo, hi = slab_bounds(rows, world, rank)
        wlo, whi = halo_window(rows, world, rank)
        n = hi - lo
        buf = np.zeros((n + 2,) + shape[1:])
        buf[1 - (lo - wlo): n + 1 + (whi - hi)] = T[wlo:whi]  # halos present only at interior faces
        for _ in range(steps):
            buf = _local_step(buf, P[lo:hi], k, rank == 0, rank == world - 1)
            reqs = []
            for op, peer, row in exchange_plan(rows, world, rank):
                t = torch.from_numpy(np.ascontiguousarray(buf[row]))
                if op == "send":
                    reqs.append(dist.isend(t, peer))
                else:
                    reqs.append((dist.irecv(t, peer), row, t))
            for r in reqs:
                if isinstance(r, tuple):
                    r[0].wait()
                    buf[r[1]] = r[2].numpy()
                else:
                    r.wait()
        mine = torch.from_numpy(np.ascontiguousarray(buf[1:n + 1]))
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, mine.numpy()))
        if rank == 0:
            full = np.empty(shape)
            for a, b, arr in parts:
                full[a:b] = arr
            q.put(full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (17, 9)), (3, (20, 6, 4)), (2, (5, 3, 8)), (8, (21, 5, 4))])
def test_gloo_slab_protocol_matches_single_domain(world, shape):
    steps, k = 6, 0.1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, steps, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    T = rng.random(shape)
    P = rng.random(shape) * 1e-3
    want = ocpu.hotspot(T, P, k, steps)
    assert np.array_equal(got, want)


def test_slab_bounds_and_windows_cover_the_grid():
    for rows in (1, 2, 7, 2048):
        for world in range(1, min(rows, 9) + 1):
            spans = [slab_bounds(rows, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            for r in range(world):
                wlo, whi = halo_window(rows, world, r)
                lo, hi = spans[r]
                assert wlo == lo - (r > 0) and whi == hi + (r < world - 1)
    with pytest.raises(ValueError):
        slab_bounds(3, 4, 0)


def test_exchange_plan_pairs_every_send_with_a_recv():
    rows, world = 2048, 8
    sends, recvs = [], []
    for r in range(world):
        lo, hi = slab_bounds(rows, world, r)
        for op, peer, row in exchange_plan(rows, world, r):
            (sends if op == "send" else recvs).append((r, peer, row, hi - lo))
    assert len(sends) == len(recvs) == 2 * (world - 1)
    for r, peer, row, n in sends:  # my first owned row lands in the upper rank's bottom halo
        match = [x for x in recvs if x[0] == peer and x[1] == r]
        assert len(match) == 1
        assert (row == 1 and match[0][2] == match[0][3] + 1) or (row == n and match[0][2] == 0)


@pytest.mark.parametrize("shape,world", [((11, 4, 3), 3), ((8, 5), 2), ((2048, 4), 8)])
def test_seeded_window_equals_slicing_the_reference_generator(shape, world):
    from paper_2501_09398_b200.cli import WORKLOAD_SEED
    from paper_2501_09398_b200.distributed import seeded_window

    rng = np.random.default_rng(WORKLOAD_SEED)
    T = rng.random(shape)
    P = rng.random(shape) * 1e-3
    for rank in range(world):
        t, p = seeded_window(shape, rank, world)
        lo, hi = slab_bounds(shape[0], world, rank)
        wlo, whi = halo_window(shape[0], world, rank)
        assert np.array_equal(t, T[wlo:whi]) and np.array_equal(p, P[lo:hi])

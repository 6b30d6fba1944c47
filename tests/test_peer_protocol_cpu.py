"""The peer halo exchange's ordering protocol, restated on CPU with one thread per rank.

runtime.cu / kernels.cuh (k_dist_wait, k_dist_signal): before iteration t a rank waits until both
neighbours have completed t iterations, then computes its owned rows from buf[p] into buf[p^1]
and stores its first / last output row straight into the neighbours' buf[p^1] halo planes, then
publishes t+1. Here every rank is a thread sharing numpy buffers, with random delays injected
between the protocol steps; the gathered result must equal the single-domain oracle bit for bit
for every schedule — i.e. the wait condition alone rules out the RAW race (reading a halo before
the neighbour wrote it) and the WAR race (overwriting a neighbour's halo it is still reading).
"""

import random
import threading
import time

import numpy as np
import pytest

from oracle import cpu as ocpu
from paper_2501_09398_b200.distributed import slab_bounds


def _step(src, dst, power, k, top_edge, bot_edge):
    """Owned rows of one hotspot step on a halo'd slab buffer (numpy, binary64)."""
    buf = src.copy()
    if top_edge:
        buf[0] = buf[1]
    if bot_edge:
        buf[-1] = buf[-2]
    c = buf[1:-1]
    p = np.pad(c, [(0, 0)] + [(1, 1)] * (buf.ndim - 1), mode="edge")
    if buf.ndim == 2:
        s = (buf[:-2] + buf[2:]) + (p[:, :-2] + p[:, 2:])
        loss = 4.0
    else:
        s = ((buf[:-2] + buf[2:]) + (p[:, :-2, 1:-1] + p[:, 2:, 1:-1])) + (p[:, 1:-1, :-2] + p[:, 1:-1, 2:])
        loss = 6.0
    dst[1:-1] = c + k * (s - loss * c) + power


def _run(T, P, k, world, iters, seed):
    rows = T.shape[0]
    rng = random.Random(seed)
    delays = [[rng.random() * 1e-3 for _ in range(3 * iters)] for _ in range(world)]
    ranks = []
    for r in range(world):
        lo, hi = slab_bounds(rows, world, r)
        b = [np.zeros((hi - lo + 2,) + T.shape[1:]) for _ in range(2)]
        wlo, whi = lo - (r > 0), hi + (r < world - 1)
        b[0][1 - (r > 0): 1 - (r > 0) + (whi - wlo)] = T[wlo:whi]
        ranks.append({"lo": lo, "hi": hi, "buf": b, "P": P[lo:hi], "done": 0})
    counts = [0] * world
    lock = threading.Lock()
    errors = []

    def worker(r):
        me = ranks[r]
        try:
            for t in range(iters):
                time.sleep(delays[r][3 * t])
                while True:  # k_dist_wait: neighbours' completed counts >= mine
                    with lock:
                        ok = all(counts[q] >= t for q in (r - 1, r + 1) if 0 <= q < world)
                    if ok:
                        break
                    time.sleep(1e-5)
                p = t & 1
                src, dst = me["buf"][p], me["buf"][p ^ 1]
                _step(src, dst, me["P"], k, r == 0, r == world - 1)
                time.sleep(delays[r][3 * t + 1])
                if r > 0:  # first owned output row -> up neighbour's bottom halo (peer store)
                    ranks[r - 1]["buf"][p ^ 1][-1] = dst[1]
                if r < world - 1:  # last owned output row -> down neighbour's top halo
                    ranks[r + 1]["buf"][p ^ 1][0] = dst[-2]
                time.sleep(delays[r][3 * t + 2])
                with lock:  # k_dist_signal
                    counts[r] = t + 1
        except Exception as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=120)
    assert not errors
    out = np.empty_like(T)
    for me in ranks:
        out[me["lo"]:me["hi"]] = me["buf"][iters & 1][1:-1]
    return out


@pytest.mark.parametrize("world,shape,seed", [(2, (12, 6), 1), (3, (17, 5, 4), 2), (4, (9, 7), 3),
                                               (3, (6, 4, 3), 4)])
def test_peer_protocol_equals_single_domain_under_random_schedules(world, shape, seed):
    rng = np.random.default_rng(seed)
    T = rng.random(shape)
    P = rng.random(shape) * 1e-3
    iters = 9
    want = ocpu.hotspot(T, P, 0.1, iters, np.float64)
    got = _run(T, P, 0.1, world, iters, seed)
    assert np.array_equal(got, want)

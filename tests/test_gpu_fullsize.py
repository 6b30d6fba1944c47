"""Parity at BASELINE.json's full sizes, where the CPU oracle cannot run the whole grid.

Hotspot3D 2048x2048x256 (binary32, 12.9 GB on the device, the cp.async.bulk plane-march kernel):
* light-cone windows: after N steps a cell depends only on cells within N of it, so the C oracle
  run on a window grown by N (real grid edges where the window touches them) must equal the
  device result on the window's interior, bit for bit — corners, edges, and interior windows
  that straddle the kernel's tile and row-chunk boundaries;
* graph (programmatic edges, odd K) == stream, and 3 axis-0 slabs == 1 slab, bit for bit.
FDTD 256^3 (binary32): fused leapfrog == two half-steps == C oracle, bit for bit, and the
graph path == the stream path. (binary64 at 256^3 is pinned to the reference checksum at N = 20 in
test_gpu_parity.py.)
"""

import numpy as np
import pytest

from oracle import cpu as ocpu
from paper_2501_09398_b200 import workloads as wl
from tests.conftest import spread

pytestmark = pytest.mark.gpu

SHAPE = (2048, 2048, 256)
K_DIFF = 0.1


class _Shape:
    """Shape-only stand-in for the global state (the arrays are uploaded as binary32 directly)."""

    def __init__(self, shape, k):
        self.temperature = np.lib.stride_tricks.as_strided(np.zeros(1), shape, [0] * len(shape))
        self.power = self.temperature
        self.diffusion_coefficient = float(k)


@pytest.fixture(scope="module")
def big():
    rng = np.random.default_rng(20240817)
    t = rng.random(SHAPE, dtype=np.float32)
    p = rng.random(SHAPE, dtype=np.float32) * np.float32(1e-3)
    return t, p


def _run(t, p, how, n, devices=None):
    s = wl.DeviceSolver(_Shape(SHAPE, K_DIFF), "f32", devices=devices, upload=False)
    try:
        s.upload([t, p])
        if how == "stream":
            s.run_stream(n)
        else:
            k = how
            s.run_batched(k, n // k, pdl=True)
        return s.download_field(0)
    finally:
        s.close()


def _window_check(t, p, got, r0, c0, w, n):
    R, C, _ = SHAPE
    ra, rb = max(0, r0 - n), min(R, r0 + w + n)
    ca, cb = max(0, c0 - n), min(C, c0 + w + n)
    want = ocpu.hotspot(t[ra:rb, ca:cb], p[ra:rb, ca:cb], K_DIFF, n, np.float32)
    g = got[r0:r0 + w, c0:c0 + w]
    wv = want[r0 - ra:r0 - ra + w, c0 - ca:c0 - ca + w]
    assert np.array_equal(g, wv), (r0, c0)


def test_hotspot3d_2048_light_cone_windows_and_modes(gpu, big):
    t, p = big
    n = 5
    got = _run(t, p, 5, n)  # odd K: the swapped-parity executable as well
    R, C, _ = SHAPE
    w = 20
    for r0, c0 in ((0, 0), (0, C - w), (R - w, 0), (R - w, C - w), (1000, 1013), (1531, 7),
                   (127, 1024), (2000, 500)):
        _window_check(t, p, got, r0, c0, w, n)
    assert np.array_equal(got, _run(t, p, "stream", n))
    assert np.array_equal(got, _run(t, p, 5, n, devices=spread(3)))


@pytest.fixture(scope="module")
def fdtd256():
    base = wl.te101_cavity(256, 256, 256)
    rng = np.random.default_rng(3)
    arrs = [a + 1e-3 * rng.random(a.shape) for a in base.state_arrays()]  # break the mode's symmetry
    return wl.FdtdWorkload(*arrs, base.cell_size, base.time_step)


def test_fdtd_256_two_half_steps_fused_and_oracle(gpu, fdtd256):
    st = fdtd256
    n = 3
    dt = st.time_step
    want = ocpu.fdtd(st.state_arrays(), st.cell_size, dt / wl.VACUUM_PERMEABILITY,
                     dt / wl.VACUUM_PERMITTIVITY, n, np.float32)
    two = wl.run_batched(wl.fdtd_program(), st, 3, 1, dtype="f32").state_arrays()
    fused = wl.run_batched(wl.fdtd_program(), st, 3, 1, dtype="f32", fuse=True).state_arrays()
    stream = wl.run_loop(wl.fdtd_program(), st, n, dtype="f32", fuse=True).state_arrays()
    wl.release_cached_contexts()
    for a, b, c, w in zip(two, fused, stream, want):
        assert np.array_equal(np.asarray(a, np.float32), w)
        assert np.array_equal(np.asarray(b, np.float32), w)
        assert np.array_equal(np.asarray(c, np.float32), w)


def test_fdtd_256_binary32_within_tolerance_at_the_baseline_horizon(gpu):
    """BASELINE config FDTD 256^3, N = 2000: binary32 vs the binary64 run (which reproduces the
    reference bit for bit, pinned by its checksum at N = 20) within 1e-5 in normalised L-inf
    (pointwise max-rel is undefined on TE101's exact zeros)."""
    st = wl.te101_cavity(256, 256, 256)
    prog = wl.fdtd_program()
    ref = wl.run_batched(prog, st, 100, 20).state_arrays()
    got = wl.run_batched(prog, st, 100, 20, dtype="f32", fuse=True).state_arrays()
    wl.release_cached_contexts()
    scale = max(float(np.max(np.abs(a))) for a in ref[:3])  # E amplitude
    hscale = max(float(np.max(np.abs(a))) for a in ref[3:])
    for i, (g, r) in enumerate(zip(got, ref)):
        s = scale if i < 3 else hscale
        assert float(np.max(np.abs(g - r))) / s <= 1e-5, i


def test_hotspot3d_2048_binary32_within_tolerance_at_n100(gpu):
    """BASELINE config Hotspot3D 2048x2048x256, N = 100: binary32 vs binary64 (bit-exact to the
    reference algorithm), max-rel <= 1e-5."""
    rng = np.random.default_rng(20240817)
    t = rng.random(SHAPE)
    p = rng.random(SHAPE) * 1e-3
    outs = {}
    for dtype in ("f64", "f32"):
        s = wl.DeviceSolver(_Shape(SHAPE, K_DIFF), dtype, upload=False)
        try:
            npd = np.float64 if dtype == "f64" else np.float32
            s.upload([t.astype(npd, copy=False), p.astype(npd, copy=False)])
            s.run_batched(20, 5, pdl=True)
            outs[dtype] = s.download_field(0)
        finally:
            s.close()
    rel = np.max(np.abs(outs["f32"].astype(np.float64) - outs["f64"]) / np.abs(outs["f64"]))
    assert rel <= 1e-5, rel

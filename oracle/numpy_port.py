"""numpy restatement of the reference steps. TEST INFRASTRUCTURE / CPU BASELINE ONLY.

Restates /root/reference/pkg/src/iterbatch/workloads.py expression for expression, generic over
the array dtype. In binary64 this is the reference algorithm (same numpy calls, same grouping,
same np.pad edge mode, same row-slab threading) and is what bench.py times as the CPU baseline
(kind "port"). In binary32 the scalars stay Python floats so numpy (NEP 50) keeps every op in
binary32 with the scalar rounded once — the semantics of the binary32 CUDA kernels.

The vector binary32 rule is the exception: the constant stays binary64 and the product is rounded
on store, matching k_vector_f32.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

VACUUM_LIGHT_SPEED = 299792458.0  # workloads.py:48-50
VACUUM_PERMEABILITY = 4.0e-7 * math.pi
VACUUM_PERMITTIVITY = 1.0 / (VACUUM_PERMEABILITY * VACUUM_LIGHT_SPEED**2)


class SlabPool:
    """Row-slab threading of workloads.py:60-69 with a persistent pool.

    The reference re-creates its ThreadPoolExecutor every step (workloads.py:67); the bounds
    formula n*i//workers is the same. A persistent pool makes the baseline faster, never slower,
    so the CPU numbers reported beside the GPU are conservative.
    """

    def __init__(self, workers: int | None):
        self.workers = workers if workers and workers > 1 else None
        self.pool = ThreadPoolExecutor(max_workers=self.workers) if self.workers else None

    def fill(self, n_rows: int, fill) -> None:
        if self.pool is None or n_rows <= 1:
            fill(0, n_rows)
            return
        w = self.workers
        bounds = [n_rows * i // w for i in range(w + 1)]
        spans = [(lo, hi) for lo, hi in zip(bounds, bounds[1:]) if lo < hi]
        for _ in self.pool.map(lambda s: fill(*s), spans):
            pass

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


_SERIAL = SlabPool(None)


def vector_scale_step(values: np.ndarray, c: float, pool: SlabPool = _SERIAL) -> np.ndarray:
    """workloads.py:97-105."""
    out = np.empty_like(values)
    if values.dtype == np.float32:
        def fill(lo, hi):
            out[lo:hi] = (values[lo:hi].astype(np.float64) * c).astype(np.float32)
    else:
        def fill(lo, hi):
            out[lo:hi] = values[lo:hi] * c
    pool.fill(out.shape[0], fill)
    return out


def hotspot_step(temp: np.ndarray, power: np.ndarray, k: float, pool: SlabPool = _SERIAL):
    """workloads.py:167-207."""
    k = float(k)
    loss = 2.0 * temp.ndim
    padded = np.pad(temp, 1, mode="edge")
    out = np.empty_like(temp)
    if temp.ndim == 2:
        def fill(lo, hi):
            center = padded[lo + 1 : hi + 1, 1:-1]
            x_pair = padded[lo:hi, 1:-1] + padded[lo + 2 : hi + 2, 1:-1]
            y_pair = padded[lo + 1 : hi + 1, :-2] + padded[lo + 1 : hi + 1, 2:]
            out[lo:hi] = center + k * ((x_pair + y_pair) - loss * center) + power[lo:hi]
    else:
        def fill(lo, hi):
            center = padded[lo + 1 : hi + 1, 1:-1, 1:-1]
            x_pair = padded[lo:hi, 1:-1, 1:-1] + padded[lo + 2 : hi + 2, 1:-1, 1:-1]
            y_pair = padded[lo + 1 : hi + 1, :-2, 1:-1] + padded[lo + 1 : hi + 1, 2:, 1:-1]
            z_pair = padded[lo + 1 : hi + 1, 1:-1, :-2] + padded[lo + 1 : hi + 1, 1:-1, 2:]
            out[lo:hi] = center + k * (((x_pair + y_pair) + z_pair) - loss * center) + power[lo:hi]
    pool.fill(out.shape[0], fill)
    return out


def fdtd_h_step(f, d: float, c_h: float, pool: SlabPool = _SERIAL):
    """workloads.py:325-355; f = (ex, ey, ez, hx, hy, hz)."""
    ex, ey, ez, hx0, hy0, hz0 = f
    d, c_h = float(d), float(c_h)
    hx, hy, hz = np.empty_like(hx0), np.empty_like(hy0), np.empty_like(hz0)

    def fill_hx(lo, hi):
        hx[lo:hi] = hx0[lo:hi] + c_h * (
            (ey[lo:hi, :, 1:] - ey[lo:hi, :, :-1]) / d - (ez[lo:hi, 1:, :] - ez[lo:hi, :-1, :]) / d
        )

    def fill_hy(lo, hi):
        hy[lo:hi] = hy0[lo:hi] + c_h * (
            (ez[lo + 1 : hi + 1] - ez[lo:hi]) / d - (ex[lo:hi, :, 1:] - ex[lo:hi, :, :-1]) / d
        )

    def fill_hz(lo, hi):
        hz[lo:hi] = hz0[lo:hi] + c_h * (
            (ex[lo:hi, 1:, :] - ex[lo:hi, :-1, :]) / d - (ey[lo + 1 : hi + 1] - ey[lo:hi]) / d
        )

    pool.fill(hx.shape[0], fill_hx)
    pool.fill(hy.shape[0], fill_hy)
    pool.fill(hz.shape[0], fill_hz)
    return (ex, ey, ez, hx, hy, hz)


def fdtd_e_step(f, d: float, c_e: float, pool: SlabPool = _SERIAL):
    """workloads.py:358-413."""
    ex0, ey0, ez0, hx, hy, hz = f
    d, c_e = float(d), float(c_e)
    ex, ey, ez = ex0.copy(), ey0.copy(), ez0.copy()
    nx, ny, nz = ex0.shape[0], ex0.shape[1] - 1, ex0.shape[2] - 1

    def fill_ex(lo, hi):
        ex[lo:hi, 1:-1, 1:-1] = ex0[lo:hi, 1:-1, 1:-1] + c_e * (
            (hz[lo:hi, 1:, 1:-1] - hz[lo:hi, :-1, 1:-1]) / d
            - (hy[lo:hi, 1:-1, 1:] - hy[lo:hi, 1:-1, :-1]) / d
        )

    def fill_ey(lo, hi):
        lo_i, hi_i = max(lo, 1), min(hi, nx)
        if lo_i >= hi_i:
            return
        ey[lo_i:hi_i, :, 1:-1] = ey0[lo_i:hi_i, :, 1:-1] + c_e * (
            (hx[lo_i:hi_i, :, 1:] - hx[lo_i:hi_i, :, :-1]) / d
            - (hz[lo_i:hi_i, :, 1:-1] - hz[lo_i - 1 : hi_i - 1, :, 1:-1]) / d
        )

    def fill_ez(lo, hi):
        lo_i, hi_i = max(lo, 1), min(hi, nx)
        if lo_i >= hi_i:
            return
        ez[lo_i:hi_i, 1:-1, :] = ez0[lo_i:hi_i, 1:-1, :] + c_e * (
            (hy[lo_i:hi_i, 1:-1, :] - hy[lo_i - 1 : hi_i - 1, 1:-1, :]) / d
            - (hx[lo_i:hi_i, 1:, :] - hx[lo_i:hi_i, :-1, :]) / d
        )

    pool.fill(ex.shape[0], fill_ex)
    pool.fill(ey.shape[0], fill_ey)
    pool.fill(ez.shape[0], fill_ez)
    ex[:, 0, :] = 0.0
    ex[:, -1, :] = 0.0
    ex[:, :, 0] = 0.0
    ex[:, :, -1] = 0.0
    ey[0, :, :] = 0.0
    ey[-1, :, :] = 0.0
    ey[:, :, 0] = 0.0
    ey[:, :, -1] = 0.0
    ez[0, :, :] = 0.0
    ez[-1, :, :] = 0.0
    ez[:, 0, :] = 0.0
    ez[:, -1, :] = 0.0
    return (ex, ey, ez, hx, hy, hz)


def run_vector(values, c, steps, pool: SlabPool = _SERIAL):
    for _ in range(steps):
        values = vector_scale_step(values, c, pool)
    return values


def run_hotspot(temp, power, k, steps, pool: SlabPool = _SERIAL):
    for _ in range(steps):
        temp = hotspot_step(temp, power, k, pool)
    return temp


def run_fdtd(fields, d, c_h, c_e, steps, pool: SlabPool = _SERIAL):
    for _ in range(steps):
        fields = fdtd_e_step(fdtd_h_step(fields, d, c_h, pool), d, c_e, pool)
    return fields


def fdtd_coefficients(cell_size: float, time_step: float) -> tuple[float, float]:
    """c_h = dt/mu0 (workloads.py:328), c_e = dt/eps0 (workloads.py:365)."""
    return time_step / VACUUM_PERMEABILITY, time_step / VACUUM_PERMITTIVITY

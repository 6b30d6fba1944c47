"""ctypes binding of the C oracle (oracle/ib_oracle.c). TEST INFRASTRUCTURE ONLY.

Each function takes fp64 or fp32 numpy arrays (the dtype selects the C restatement), works on
copies and returns new arrays, mirroring the pure-function style of the reference steps
(workloads.py:97-105, 167-207, 325-413).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libib_oracle.so")
_lib = None

FNV_OFFSET = 0xCBF29CE484222325


def build() -> str:
    """Compile the oracle with its Makefile (gcc only; no CUDA)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        p, i64, d, f, u64, sz = (
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_double,
            ctypes.c_float,
            ctypes.c_uint64,
            ctypes.c_size_t,
        )
        L.or_fnv1a64.argtypes = [p, sz, u64]
        L.or_fnv1a64.restype = u64
        L.or_fnv1a64_f32_as_f64.argtypes = [p, sz, u64]
        L.or_fnv1a64_f32_as_f64.restype = u64
        L.or_vector_f64.argtypes = [p, i64, d, i64]
        L.or_vector_f32.argtypes = [p, i64, d, i64]
        L.or_hotspot_f64.argtypes = [p, p, i64, i64, i64, ctypes.c_int, d, i64]
        L.or_hotspot_f32.argtypes = [p, p, i64, i64, i64, ctypes.c_int, f, i64]
        L.or_fdtd_f64.argtypes = [p] * 6 + [i64, i64, i64, d, d, d, i64]
        L.or_fdtd_f32.argtypes = [p] * 6 + [i64, i64, i64, f, f, f, i64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _tag(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise ValueError(f"oracle supports float32/float64, got {dt}")


def vector(values, c: float, steps: int, dtype=np.float64) -> np.ndarray:
    v = np.array(values, dtype=dtype, order="C", copy=True)
    getattr(lib(), "or_vector_" + _tag(dtype))(_ptr(v), v.size, float(c), int(steps))
    return v


def hotspot(temperature, power, k: float, steps: int, dtype=np.float64) -> np.ndarray:
    t = np.array(temperature, dtype=dtype, order="C", copy=True)
    p = np.ascontiguousarray(power, dtype=dtype)
    if t.ndim == 2:
        R, C = t.shape
        L, dims = 1, 2
    elif t.ndim == 3:
        R, C, L = t.shape
        dims = 3
    else:
        raise ValueError("hotspot oracle takes 2-D or 3-D grids")
    getattr(lib(), "or_hotspot_" + _tag(dtype))(
        _ptr(t), _ptr(p), R, C, L, dims, float(k), int(steps)
    )
    return t


def fdtd(fields, d: float, c_h: float, c_e: float, steps: int, dtype=np.float64):
    """fields = (ex, ey, ez, hx, hy, hz); returns new arrays after `steps` H+E iterations."""
    arrs = [np.array(a, dtype=dtype, order="C", copy=True) for a in fields]
    nx, nyp, nzp = arrs[0].shape
    getattr(lib(), "or_fdtd_" + _tag(dtype))(
        *[_ptr(a) for a in arrs], nx, nyp - 1, nzp - 1, float(d), float(c_h), float(c_e), int(steps)
    )
    return tuple(arrs)


def fnv1a64(data: bytes | np.ndarray, h: int = FNV_OFFSET) -> int:
    buf = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray)) else data
    buf = np.ascontiguousarray(buf)
    return int(lib().or_fnv1a64(_ptr(buf), buf.nbytes, h))


def checksum(arrays) -> int:
    """state_checksum (workloads.py:520-525) over arrays in state_arrays() order."""
    h = FNV_OFFSET
    for a in arrays:
        a = np.asarray(a)
        if a.dtype == np.float32:
            a = np.ascontiguousarray(a)
            h = int(lib().or_fnv1a64_f32_as_f64(_ptr(a), a.size, h))
        else:
            b = np.ascontiguousarray(a, dtype="<f8")
            h = int(lib().or_fnv1a64(_ptr(b), b.nbytes, h))
    return h

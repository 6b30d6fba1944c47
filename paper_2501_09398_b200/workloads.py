"""B200 drop-in for the reference solver API ``iterbatch.workloads``.

Same names, signatures, dataclasses, validation messages and error types as
/root/reference/pkg/src/iterbatch/workloads.py, with every step executed by the sm_100a runtime
(libiterbatch_b200.so, include/iterbatch_b200.h) instead of numpy:

=====================  ==========================================  ===============================
reference              here                                        device work
=====================  ==========================================  ===============================
vector_scale_step      workloads.py:97-105                         1 launch of k_vector
hotspot_step           workloads.py:167-207                        1 launch of k_hotspot_vec/tma
fdtd_h_step/e_step     workloads.py:325-413                        1 launch of k_fdtd_lf H / E mode
run_loop               workloads.py:442-450 (Listing 1)            N launches from a C++ loop
run_batched            workloads.py:453-471 (Listings 2/3)         K-iteration CUDA graph, I replays
time_workload          workloads.py:479-505                        timed T_C + T_E per repeat
state_checksum         workloads.py:508-525                        native FNV-1a (same algorithm)
=====================  ==========================================  ===============================

The boundary is per RUN: a run uploads the state once, keeps it in HBM for all iterations and
downloads it once. ``workers`` is accepted for signature compatibility and ignored (the device
grid replaces the row-slab threads). Keyword-only extensions: ``dtype`` ("f64" reproduces the
reference bit for bit; "f32" is the bandwidth-halving mode, parity tiers in DESIGN.md), ``devices``
(axis-0 slabs for hotspot grids and both FDTD solvers; ``halo="copy"`` moves hotspot halo planes
with peer-copy nodes instead of the kernel's own stores), ``fuse`` (FDTD: H and E in one kernel),
and graph options (``build``, ``pdl``, ``while_loop``, ``patch``).

There is no CPU fallback: without the library or a CUDA device every call raises.
Reference dataclasses are accepted too (duck-typed); results come back as the input's type.
"""

from __future__ import annotations

import ctypes
import math
import operator
import threading
import time
from collections import OrderedDict
from contextlib import contextmanager
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .fitting import MeasurementPoint, MeasurementSeries
from .model import BatchPlan

__all__ = [
    "VectorWorkload",
    "HotspotWorkload",
    "FdtdWorkload",
    "ChainProgram",
    "ExecutionOrder",
    "vector_scale_step",
    "hotspot_step",
    "fdtd_h_step",
    "fdtd_e_step",
    "vector_program",
    "hotspot_program",
    "fdtd_program",
    "fdtd_cavity",
    "te101_cavity",
    "run_loop",
    "run_batched",
    "run_peeled",
    "time_workload",
    "time_workload_phases",
    "state_checksum",
    "DeviceSolver",
    "release_cached_contexts",
    "VACUUM_LIGHT_SPEED",
    "VACUUM_PERMEABILITY",
    "VACUUM_PERMITTIVITY",
]

VACUUM_LIGHT_SPEED = 299792458.0
VACUUM_PERMEABILITY = 4.0e-7 * math.pi
VACUUM_PERMITTIVITY = 1.0 / (VACUUM_PERMEABILITY * VACUUM_LIGHT_SPEED**2)


def _as_float64(value, name: str) -> np.ndarray:
    arr = np.asarray(value, dtype=np.float64)
    if arr.size == 0:
        raise ValueError(f"{name} must not be empty")
    return arr


# ================================================================================================
# State dataclasses (host side, binary64 like the reference; workloads.py:72-273)
# ================================================================================================
@dataclass(frozen=True, eq=False)
class VectorWorkload:
    """A 1-D array repeatedly scaled by a constant."""

    values: np.ndarray
    scale_constant: float

    def __post_init__(self):
        values = _as_float64(self.values, "values")
        if values.ndim != 1:
            raise ValueError(f"values must be 1-D, got shape {values.shape}")
        object.__setattr__(self, "values", values)
        object.__setattr__(self, "scale_constant", float(self.scale_constant))

    @property
    def length(self) -> int:
        return self.values.shape[0]

    def copy(self) -> "VectorWorkload":
        return VectorWorkload(self.values.copy(), self.scale_constant)

    def state_arrays(self) -> tuple[np.ndarray, ...]:
        return (self.values,)


@dataclass(frozen=True, eq=False)
class HotspotWorkload:
    """Explicit heat diffusion with a source term on a 2-D or 3-D grid (edge-clamped)."""

    temperature: np.ndarray
    power: np.ndarray
    diffusion_coefficient: float

    def __post_init__(self):
        temperature = _as_float64(self.temperature, "temperature")
        power = _as_float64(self.power, "power")
        if temperature.ndim not in (2, 3):
            raise ValueError(f"temperature must be 2-D or 3-D, got {temperature.ndim}-D")
        if power.shape != temperature.shape:
            raise ValueError(
                f"power shape {power.shape} != temperature shape {temperature.shape}"
            )
        coeff = float(self.diffusion_coefficient)
        limit = 1.0 / (2.0 * temperature.ndim)
        if not 0.0 <= coeff <= limit:
            raise ValueError(
                f"diffusion_coefficient {coeff!r} outside stable range [0, {limit}] "
                f"for {temperature.ndim}-D"
            )
        object.__setattr__(self, "temperature", temperature)
        object.__setattr__(self, "power", power)
        object.__setattr__(self, "diffusion_coefficient", coeff)

    @property
    def dims(self) -> int:
        return self.temperature.ndim

    @property
    def rows(self) -> int:
        return self.temperature.shape[0]

    @property
    def cols(self) -> int:
        return self.temperature.shape[1]

    @property
    def layers(self) -> int:
        return self.temperature.shape[2] if self.dims == 3 else 1

    def copy(self) -> "HotspotWorkload":
        return HotspotWorkload(
            self.temperature.copy(), self.power.copy(), self.diffusion_coefficient
        )

    def state_arrays(self) -> tuple[np.ndarray, ...]:
        return (self.temperature, self.power)


@dataclass(frozen=True, eq=False)
class FdtdWorkload:
    """Staggered-grid electromagnetic fields in a closed conducting box (Yee lattice)."""

    ex: np.ndarray
    ey: np.ndarray
    ez: np.ndarray
    hx: np.ndarray
    hy: np.ndarray
    hz: np.ndarray
    cell_size: float
    time_step: float

    def __post_init__(self):
        for name in ("ex", "ey", "ez", "hx", "hy", "hz"):
            object.__setattr__(self, name, _as_float64(getattr(self, name), name))
        object.__setattr__(self, "cell_size", float(self.cell_size))
        object.__setattr__(self, "time_step", float(self.time_step))
        if self.cell_size <= 0.0:
            raise ValueError("cell_size must be positive")
        nx, ny, nz = self.dims
        expected = {
            "ex": (nx, ny + 1, nz + 1),
            "ey": (nx + 1, ny, nz + 1),
            "ez": (nx + 1, ny + 1, nz),
            "hx": (nx + 1, ny, nz),
            "hy": (nx, ny + 1, nz),
            "hz": (nx, ny, nz + 1),
        }
        for name, shape in expected.items():
            actual = getattr(self, name).shape
            if actual != shape:
                raise ValueError(f"{name} shape {actual} != expected {shape}")
        limit = self.cell_size / (VACUUM_LIGHT_SPEED * math.sqrt(3.0))
        if not 0.0 < self.time_step <= limit:
            raise ValueError(
                f"time_step {self.time_step!r} violates the stability limit {limit!r}"
            )

    @property
    def dims(self) -> tuple[int, int, int]:
        nx, nyp, nzp = self.ex.shape
        return nx, nyp - 1, nzp - 1

    def copy(self) -> "FdtdWorkload":
        return FdtdWorkload(
            self.ex.copy(), self.ey.copy(), self.ez.copy(),
            self.hx.copy(), self.hy.copy(), self.hz.copy(),
            self.cell_size, self.time_step,
        )

    def state_arrays(self) -> tuple[np.ndarray, ...]:
        return (self.ex, self.ey, self.ez, self.hx, self.hy, self.hz)


def fdtd_cavity(
    nx: int, ny: int, nz: int, cell_size: float = 1.0, courant: float = 0.99
) -> FdtdWorkload:
    """Zero-field box of nx*ny*nz cells at the given fraction of the limit (workloads.py:276-295)."""
    for n in (nx, ny, nz):
        if operator.index(n) < 1:
            raise ValueError("cell counts must be >= 1")
    if not 0.0 < courant <= 1.0:
        raise ValueError(f"courant must be in (0, 1], got {courant!r}")
    dt = courant * cell_size / (VACUUM_LIGHT_SPEED * math.sqrt(3.0))
    return FdtdWorkload(
        ex=np.zeros((nx, ny + 1, nz + 1)),
        ey=np.zeros((nx + 1, ny, nz + 1)),
        ez=np.zeros((nx + 1, ny + 1, nz)),
        hx=np.zeros((nx + 1, ny, nz)),
        hy=np.zeros((nx, ny + 1, nz)),
        hz=np.zeros((nx, ny, nz + 1)),
        cell_size=cell_size,
        time_step=dt,
    )


def te101_cavity(
    nx: int, ny: int, nz: int, cell_size: float = 1.0, courant: float = 0.99,
    amplitude: float = 1.0,
) -> FdtdWorkload:
    """Box seeded with the TE101 mode Ey = A sin(pi x/Lx) sin(pi z/Lz) (workloads.py:298-322)."""
    w = fdtd_cavity(nx, ny, nz, cell_size, courant)
    x_profile = np.sin(np.pi * np.arange(nx + 1) / nx)
    z_profile = np.sin(np.pi * np.arange(nz + 1) / nz)
    x_profile[0] = x_profile[-1] = 0.0  # sin(pi) rounds to ~1.2e-16: ground walls exactly
    z_profile[0] = z_profile[-1] = 0.0
    ey = np.empty_like(w.ey)
    ey[:] = amplitude * x_profile[:, None, None] * z_profile[None, None, :]
    return FdtdWorkload(w.ex, ey, w.ez, w.hx, w.hy, w.hz, w.cell_size, w.time_step)


# ================================================================================================
# Device solver: one HBM-resident solver instance (one ib_ctx)
# ================================================================================================
def _kind_of_state(state) -> str:
    if hasattr(state, "scale_constant") and hasattr(state, "values"):
        return "vector"
    if hasattr(state, "temperature") and hasattr(state, "diffusion_coefficient"):
        nd = np.ndim(state.temperature)
        if nd == 2:
            return "hotspot2d"
        if nd == 3:
            return "hotspot3d"
        raise ValueError(f"temperature must be 2-D or 3-D, got {nd}-D")
    if all(hasattr(state, n) for n in ("ex", "ey", "ez", "hx", "hy", "hz", "cell_size")):
        return "fdtd"
    raise ValueError(f"unsupported state type {type(state).__name__}")


def _dims_scalars(kind: str, state) -> tuple[tuple[int, ...], tuple[float, ...]]:
    if kind == "vector":
        return (int(np.shape(state.values)[0]),), (float(state.scale_constant),)
    if kind in ("hotspot2d", "hotspot3d"):
        return tuple(int(s) for s in np.shape(state.temperature)), (float(state.diffusion_coefficient),)
    nx, nyp, nzp = np.shape(state.ex)
    d, dt = float(state.cell_size), float(state.time_step)
    # computed exactly as the reference does, in binary64 (workloads.py:327-328, 364-365)
    return (nx, nyp - 1, nzp - 1), (d, dt / VACUUM_PERMEABILITY, dt / VACUUM_PERMITTIVITY)


_NP_DTYPE = {"f32": np.float32, "f64": np.float64}


def _norm_dtype(dtype) -> str:
    if dtype in ("f32", "float32", np.float32):
        return "f32"
    if dtype in ("f64", "float64", np.float64, None):
        return "f64"
    raise ValueError(f"dtype must be 'f32' or 'f64', got {dtype!r}")


@dataclass
class Times:
    """One runtime call's timings (see ib_times in include/iterbatch_b200.h)."""

    create_s: float = 0.0
    instantiate_s: float = 0.0
    upload_s: float = 0.0
    build_s: float = 0.0
    exec_s: float = 0.0
    gpu_s: float = 0.0
    kernels: int = 0
    launches: int = 0
    nodes: int = 0
    graph_bytes: int = 0

    @classmethod
    def from_c(cls, t: _lib.IbTimes) -> "Times":
        return cls(**t.as_dict())


_HALO_MODE = {"store": 0, "copy": 1}  # IB_HALO_STORE / IB_HALO_COPY


class DeviceSolver:
    """A solver instance resident in HBM: upload once, run many iterations, download once.

    ``DeviceSolver(state, dtype="f32")`` allocates device fields for the state's shape, uploads
    it, and exposes the two execution modes of the paper:
      * :meth:`run_stream` — Listing 1, one launch per kernel per iteration;
      * :meth:`build_graph` + :meth:`run_graph` — Listing 3, a K-iteration unrolled graph
        instantiated/uploaded once and replayed.
    """

    def __init__(self, state, dtype="f64", devices=None, upload: bool = True, fuse: bool = False,
                 halo: str = "store"):
        self.kind = _kind_of_state(state)
        if halo not in _HALO_MODE:
            raise ValueError(f"halo must be one of {sorted(_HALO_MODE)}, not {halo!r}")
        self.halo = halo
        self.fused = bool(fuse)
        if self.fused and self.kind != "fdtd":
            raise ValueError("fuse=True applies to FDTD (H and E half-steps in one kernel)")
        self.dtype = _norm_dtype(dtype)
        self.np_dtype = _NP_DTYPE[self.dtype]
        self.dims, self.scalars = _dims_scalars(self.kind, state)
        devs = list(devices) if devices else []
        self.devices = tuple(devs)
        L = _lib.lib()
        ctx = ctypes.c_void_p()
        dims = (ctypes.c_int64 * len(self.dims))(*self.dims)
        sc = (ctypes.c_double * len(self.scalars))(*self.scalars)
        dv = (ctypes.c_int * max(1, len(devs)))(*(devs or [0]))
        _lib.check(
            L.ib_create(ctypes.byref(ctx), _lib.SOLVER["fdtd_fused" if self.fused else self.kind],
                        _lib.DTYPE[self.dtype], dims,
                        len(self.dims), sc, len(self.scalars), dv if devs else None, len(devs))
        )
        self._ctx = ctx
        if halo != "store":  # multi-slab hotspot: peer-copy halo faces
            _lib.check(L.ib_set_halo_mode(ctx, _HALO_MODE[halo]))
        self.nfields = L.ib_num_fields(ctx)
        self.shapes = []
        for f in range(self.nfields):
            shp = (ctypes.c_int64 * 3)()
            nd = ctypes.c_int()
            _lib.check(L.ib_field_shape(ctx, f, shp, ctypes.byref(nd)))
            self.shapes.append(tuple(shp[: nd.value]))
        self.batch_size = 0
        if upload:
            self.upload(state)

    # -- lifecycle -------------------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_ctx", None):
            _lib.lib().ib_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def ctx(self):
        if not self._ctx:
            raise RuntimeError("DeviceSolver is closed")
        return self._ctx

    def matches(self, kind, dtype, dims, scalars, devices) -> bool:
        return (self.kind, self.dtype, self.dims, self.scalars, self.devices) == (
            kind, dtype, dims, scalars, devices)

    # -- data movement ---------------------------------------------------------------------------
    def host_arrays(self, state) -> list[np.ndarray]:
        """State arrays as C-contiguous arrays in the device dtype (the bytes to upload)."""
        return [np.ascontiguousarray(a, dtype=self.np_dtype) for a in state.state_arrays()]

    def upload(self, state, fields=None) -> None:
        arrs = state if isinstance(state, (list, tuple)) else self.host_arrays(state)
        L = _lib.lib()
        for f, a in enumerate(arrs):
            if fields is not None and f not in fields:
                continue
            a = np.ascontiguousarray(a, dtype=self.np_dtype)
            if a.shape != self.shapes[f]:
                raise ValueError(f"field {f} shape {a.shape} != device shape {self.shapes[f]}")
            _lib.check(L.ib_upload(self.ctx, f, a.ctypes.data_as(ctypes.c_void_p), a.nbytes))

    def download_field(self, f: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.shapes[f], dtype=self.np_dtype)
        if out.dtype != self.np_dtype or not out.flags.c_contiguous or out.shape != self.shapes[f]:
            raise ValueError("download buffer must be C-contiguous with the device shape and dtype")
        _lib.check(_lib.lib().ib_download(self.ctx, f, out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out

    def download(self, template, fields=None) -> object:
        """Return a new state of ``type(template)`` holding the device fields (binary64 arrays).

        Fields not listed in ``fields`` are passed through from the template unchanged (the
        reference returns the very same array objects for fields a step does not write).
        """
        arrs = list(template.state_arrays())
        for f in range(self.nfields):
            if fields is not None and f not in fields:
                continue
            a = self.download_field(f)
            arrs[f] = a if self.dtype == "f64" else a.astype(np.float64)
        return _rebuild(template, arrs)

    # -- execution -------------------------------------------------------------------------------
    def run_stream(self, iterations: int, pdl: bool = False) -> Times:
        t = _lib.IbTimes()
        _lib.check(_lib.lib().ib_run_stream(self.ctx, int(iterations), _lib.FLAG_PDL if pdl else 0,
                                            ctypes.byref(t)))
        return Times.from_c(t)

    def run_step(self, step: int) -> Times:
        t = _lib.IbTimes()
        _lib.check(_lib.lib().ib_run_step(self.ctx, int(step), ctypes.byref(t)))
        return Times.from_c(t)

    def build_graph(self, batch_size: int, build: str = "manual", pdl: bool = False,
                    device_launch: bool = False, upload: bool = True,
                    while_loop: bool = False, meminfo: bool = False, patch: bool = False) -> Times:
        """Unroll batch_size iterations into a graph, instantiate and upload it (T_C).

        ``meminfo`` also records the device memory the instantiated graph(s) took
        (``Times.graph_bytes``, the paper's memory probe); it costs milliseconds, so timing runs
        leave it off.
        """
        if build not in _lib.BUILD:
            raise ValueError(f"build must be one of {sorted(_lib.BUILD)}, got {build!r}")
        flags = ((_lib.FLAG_PDL if pdl else 0) | (_lib.FLAG_DEVICE_LAUNCH if device_launch else 0)
                 | (0 if upload else _lib.FLAG_NO_UPLOAD) | (_lib.FLAG_WHILE if while_loop else 0)
                 | (_lib.FLAG_MEMINFO if meminfo else 0) | (_lib.FLAG_PATCH if patch else 0))
        t = _lib.IbTimes()
        _lib.check(_lib.lib().ib_graph_build(self.ctx, int(batch_size), _lib.BUILD[build], flags,
                                             ctypes.byref(t)))
        self.batch_size = int(batch_size)
        return Times.from_c(t)

    def run_batched(self, batch_size: int, num_batches: int, build: str = "manual",
                    pdl: bool = False, while_loop: bool = False, patch: bool = False) -> Times:
        """Build + replay + destroy in one call; ``gpu_s`` is T = T_C + T_E on the device clock.

        ``patch``: an odd batch on a ping-pong solver uses ONE executable whose kernel nodes are
        re-pointed with cudaGraphExecKernelNodeSetParams between launches, instead of a second
        executable with the other buffer parity baked in.
        """
        flags = ((_lib.FLAG_PDL if pdl else 0) | (_lib.FLAG_WHILE if while_loop else 0)
                 | (_lib.FLAG_PATCH if patch else 0))
        t = _lib.IbTimes()
        _lib.check(_lib.lib().ib_run_batched(self.ctx, int(batch_size), int(num_batches),
                                             _lib.BUILD[build], flags, ctypes.byref(t)))
        return Times.from_c(t)

    def run_peeled(self, total_iterations: int, batch_size: int, build: str = "manual",
                   pdl: bool = False) -> Times:
        """floor(N/K) replays of a K-iteration graph + one remainder graph (loop peeling)."""
        t = _lib.IbTimes()
        _lib.check(_lib.lib().ib_run_peeled(self.ctx, int(total_iterations), int(batch_size),
                                            _lib.BUILD[build], _lib.FLAG_PDL if pdl else 0,
                                            ctypes.byref(t)))
        return Times.from_c(t)

    def run_graph(self, num_batches: int) -> Times:
        t = _lib.IbTimes()
        _lib.check(_lib.lib().ib_graph_run(self.ctx, int(num_batches), ctypes.byref(t)))
        return Times.from_c(t)

    def destroy_graph(self) -> None:
        _lib.check(_lib.lib().ib_graph_destroy(self.ctx))
        self.batch_size = 0

    def sync(self) -> None:
        _lib.check(_lib.lib().ib_sync(self.ctx))

    def flush_l2(self) -> None:
        _lib.check(_lib.lib().ib_flush_l2(self.ctx))

    def describe(self) -> list:
        """The kernel launches of one iteration as the runtime chose them for this shape:
        [{"kernel", "grid", "block", "smem", "slab", "step"}, ...] (ib_describe); with
        halo="copy", each launch is followed by {"memcpy_nodes", "slab", "step"}."""
        import json

        L = _lib.lib()
        n = int(L.ib_describe(self.ctx, None, 0))
        if n < 0:
            _lib.check(n)
        buf = ctypes.create_string_buffer(n)
        L.ib_describe(self.ctx, buf, n)
        return json.loads(buf.value.decode())

    @property
    def iteration_bytes(self) -> int:
        return int(_lib.lib().ib_iteration_bytes(self.ctx))

    @property
    def kernels_per_iteration(self) -> int:
        n = 2 if (self.kind == "fdtd" and not getattr(self, "fused", False)) else 1
        return n * max(1, len(self.devices))

    def checksum(self) -> int:
        """state_checksum of the device state without building a host dataclass."""
        h = _lib.FNV_OFFSET
        L = _lib.lib()
        for f in range(self.nfields):
            a = self.download_field(f)
            h = int(L.ib_fnv1a64_f64(a.ctypes.data_as(ctypes.c_void_p), a.size,
                                     _lib.DTYPE[self.dtype], h))
        return h


def _rebuild(template, arrs):
    """New state of the template's type with new state arrays (other fields carried over)."""
    cls = type(template)
    if hasattr(template, "scale_constant"):
        return cls(arrs[0], template.scale_constant)
    if hasattr(template, "temperature"):
        return cls(arrs[0], arrs[1], template.diffusion_coefficient)
    return cls(*arrs, template.cell_size, template.time_step)


_CACHE: "OrderedDict[tuple, DeviceSolver]" = OrderedDict()
_CACHE_SIZE = 2
_CACHE_LOCK = threading.Lock()


@contextmanager
def _solver(state, dtype, devices, fuse: bool = False, halo: str = "store"):
    """Check out a device context for this state's shape, with the state uploaded.

    The reference functions are pure and thread-safe, so the cache of live contexts is too: a
    context is removed from the cache while a call uses it (two threads on the same shape get two
    contexts), and only contexts sitting in the cache are ever evicted and closed.
    """
    kind = _kind_of_state(state)
    dt = _norm_dtype(dtype)
    dims, scalars = _dims_scalars(kind, state)
    devs = tuple(devices) if devices else ()
    key = (kind, dt, dims, scalars, devs, bool(fuse), halo)
    with _CACHE_LOCK:
        s = _CACHE.pop(key, None)
    if s is None:
        s = DeviceSolver(state, dt, devs, upload=False, fuse=fuse, halo=halo)
    try:
        s.upload(state)
        yield s
    finally:
        evicted = []
        with _CACHE_LOCK:
            if key in _CACHE:  # another thread checked in the same shape meanwhile: keep one
                evicted.append(s)
            else:
                _CACHE[key] = s
                while len(_CACHE) > _CACHE_SIZE:
                    evicted.append(_CACHE.popitem(last=False)[1])
        for old in evicted:
            old.close()


def release_cached_contexts() -> None:
    """Free the device memory held by cached (checked-in) solver contexts."""
    with _CACHE_LOCK:
        items = list(_CACHE.values())
        _CACHE.clear()
    for s in items:
        s.close()


# ================================================================================================
# Step protocol (per-step API parity; each call is upload -> 1 kernel -> download)
# ================================================================================================
def _one_step(w, step: int, writes, dtype="f64"):
    with _solver(w, dtype, None) as s:
        s.run_step(step)
        return s.download(w, fields=writes)


def vector_scale_step(w, workers: int | None = None, *, dtype="f64"):
    """out = values * c (workloads.py:97-105), on the GPU."""
    if _kind_of_state(w) != "vector":
        raise ValueError("vector_scale_step needs a VectorWorkload")
    return _one_step(w, 0, None, dtype)


def hotspot_step(w, workers: int | None = None, *, dtype="f64"):
    """One Jacobi update T + k*(neighbor_sum - 2*dims*T) + power (workloads.py:167-207), on the GPU."""
    if _kind_of_state(w) not in ("hotspot2d", "hotspot3d"):
        raise ValueError("hotspot_step needs a HotspotWorkload")
    return _one_step(w, 0, (0,), dtype)


def fdtd_h_step(w, workers: int | None = None, *, dtype="f64"):
    """Advance the magnetic field half a step from the curl of E (workloads.py:325-355)."""
    if _kind_of_state(w) != "fdtd":
        raise ValueError("fdtd_h_step needs an FdtdWorkload")
    return _one_step(w, 0, (3, 4, 5), dtype)


def fdtd_e_step(w, workers: int | None = None, *, dtype="f64"):
    """Advance E a full step from the curl of H; PEC walls pinned to 0 (workloads.py:358-413)."""
    if _kind_of_state(w) != "fdtd":
        raise ValueError("fdtd_e_step needs an FdtdWorkload")
    return _one_step(w, 1, (0, 1, 2), dtype)


@dataclass(frozen=True)
class ChainProgram:
    """The ordered steps making up one iteration of a workload (workloads.py:416-426)."""

    steps: tuple

    def __post_init__(self):
        steps = tuple(self.steps)
        if not steps:
            raise ValueError("a chain program needs at least one step")
        object.__setattr__(self, "steps", steps)


def vector_program() -> ChainProgram:
    return ChainProgram((vector_scale_step,))


def hotspot_program() -> ChainProgram:
    return ChainProgram((hotspot_step,))


def fdtd_program() -> ChainProgram:
    # magnetic half-step first, then electric: one full leapfrog iteration
    return ChainProgram((fdtd_h_step, fdtd_e_step))


_PROGRAM_STEPS = {
    ("vector_scale_step",): ("vector",),
    ("hotspot_step",): ("hotspot2d", "hotspot3d"),
    ("fdtd_h_step", "fdtd_e_step"): ("fdtd",),
}


def _check_program(program, state) -> str:
    names = tuple(getattr(s, "__name__", repr(s)) for s in getattr(program, "steps", ()))
    kinds = _PROGRAM_STEPS.get(names)
    if kinds is None:
        raise ValueError(
            f"program steps {names} have no device implementation (supported: "
            f"{sorted(_PROGRAM_STEPS)}); this package has no CPU fallback"
        )
    kind = _kind_of_state(state)
    if kind not in kinds:
        raise ValueError(f"program {names} does not apply to a {kind} state")
    return kind


# ================================================================================================
# Drivers
# ================================================================================================
def run_loop(program, state, total_iterations: int, workers=None, *, dtype="f64", devices=None,
             pdl: bool = False, fuse: bool = False, halo: str = "store"):
    """Apply the program total_iterations times, one launch at a time (Listing 1).

    Mirrors workloads.py:442-450: N = 0 returns the same state; N < 0 raises ValueError.
    """
    total = operator.index(total_iterations)
    if total < 0:
        raise ValueError("total_iterations must be >= 0")
    _check_program(program, state)
    if total == 0:
        return state
    with _solver(state, dtype, devices, fuse, halo) as s:
        s.run_stream(total, pdl=pdl)
        return s.download(state, fields=_written_fields(state))


def run_batched(program, state, batch_size: int, num_batches: int, workers=None, *, dtype="f64",
                devices=None, build: str = "manual", pdl: bool = False, while_loop: bool = False,
                fuse: bool = False, patch: bool = False, halo: str = "store"):
    """Apply the program in num_batches replays of a batch_size-iteration CUDA graph (Listing 3).

    Mirrors workloads.py:453-471 (batch_size < 1 or num_batches < 0 raise ValueError) and
    returns the state bit-identical to run_loop over batch_size * num_batches iterations.
    """
    size = operator.index(batch_size)
    num = operator.index(num_batches)
    if size < 1:
        raise ValueError("batch_size must be >= 1")
    if num < 0:
        raise ValueError("num_batches must be >= 0")
    _check_program(program, state)
    if num == 0:
        return state
    with _solver(state, dtype, devices, fuse, halo) as s:
        s.build_graph(size, build=build, pdl=pdl, while_loop=while_loop, patch=patch)
        s.run_graph(num)
        s.destroy_graph()
        return s.download(state, fields=_written_fields(state))


def run_peeled(program, state, total_iterations: int, batch_size: int, workers=None, *,
               dtype="f64", devices=None, build: str = "manual", pdl: bool = False, fuse: bool = False,
               halo: str = "store"):
    """Any total_iterations with any batch_size: floor(N/K) graph replays plus a remainder graph.

    Loop peeling, the paper's remedy for the divisibility restriction that the
    reference's BatchPlan enforces (model.py:104-108). Bit-identical to run_loop(N).
    """
    total = operator.index(total_iterations)
    size = operator.index(batch_size)
    if total < 0:
        raise ValueError("total_iterations must be >= 0")
    if size < 1:
        raise ValueError("batch_size must be >= 1")
    _check_program(program, state)
    if total == 0:
        return state
    with _solver(state, dtype, devices, fuse, halo) as s:
        s.run_peeled(total, size, build=build, pdl=pdl)
        return s.download(state, fields=_written_fields(state))


def _written_fields(state):
    kind = _kind_of_state(state)
    return (0,) if kind in ("hotspot2d", "hotspot3d") else None


class ExecutionOrder(Enum):
    LOOP = "loop"
    BATCHED = "batched"


def _order_value(order) -> str:
    return getattr(order, "value", order)


def time_workload(program, state, plan, order, repeats: int = 10, workers: int | None = None,
                  label: str = "", *, dtype="f64", devices=None, build: str = "manual",
                  pdl: bool = False, fuse: bool = False) -> MeasurementSeries:
    """Wall-clock the full plan `repeats` times from a fresh state (workloads.py:479-505).

    The upload of the fresh state happens outside the timed region (the reference's state.copy()
    does too). LOOP times the stream-mode run; BATCHED times graph creation + instantiation +
    upload + all launches to the final synchronisation, i.e. T = T_C + T_E (Eq. 1).
    """
    if operator.index(repeats) < 1:
        raise ValueError("repeats must be >= 1")
    _check_program(program, state)
    phases = time_workload_phases(program, state, plan, order, repeats, dtype=dtype,
                                  devices=devices, build=build, pdl=pdl, fuse=fuse)
    samples = phases["total"]
    return MeasurementSeries((MeasurementPoint(plan.batch_size, tuple(samples)),), label)


def time_workload_phases(program, state, plan, order, repeats: int = 10, *, dtype="f64",
                         devices=None, build: str = "manual", pdl: bool = False,
                         while_loop: bool = False, meminfo: bool = False, fuse: bool = False,
                         patch: bool = False) -> dict:
    """Per-repeat samples split into the paper's phases.

    Returns {"creation": [T_C...], "execution": [T_E...], "total": [...], "gpu": [device T_E...],
    "times": [Times...]} — host wall-clock seconds except "gpu" (CUDA events). For LOOP order
    creation is 0.
    """
    reps = operator.index(repeats)
    if reps < 1:
        raise ValueError("repeats must be >= 1")
    _check_program(program, state)
    with _solver(state, dtype, devices, fuse) as s:
        out = {"creation": [], "execution": [], "total": [], "gpu": [], "times": []}
        batched = _order_value(order) == ExecutionOrder.BATCHED.value
        for r in range(reps):
            if r:
                s.upload(state)
            if batched:
                t0 = time.perf_counter()
                tb = s.build_graph(plan.batch_size, build=build, pdl=pdl, while_loop=while_loop,
                                   meminfo=meminfo and r == 0, patch=patch)
                te = s.run_graph(plan.num_batches)
                total = time.perf_counter() - t0
                s.destroy_graph()
                out["creation"].append(tb.build_s)
                out["execution"].append(te.exec_s)
                out["times"].append((tb, te))
            else:
                t0 = time.perf_counter()
                te = s.run_stream(plan.total_kernel_executions, pdl=pdl)
                total = time.perf_counter() - t0
                out["creation"].append(0.0)
                out["execution"].append(te.exec_s)
                out["times"].append((None, te))
            out["total"].append(total)
            out["gpu"].append(te.gpu_s)
        return out


# ================================================================================================
# Checksum (workloads.py:508-525), native FNV-1a
# ================================================================================================
_FNV_OFFSET = _lib.FNV_OFFSET


def state_checksum(workload) -> int:
    """64-bit FNV-1a over the canonical little-endian bytes of the state arrays."""
    L = _lib.lib()
    h = _FNV_OFFSET
    for arr in workload.state_arrays():
        b = np.ascontiguousarray(arr, dtype="<f8")
        h = int(L.ib_fnv1a64(b.ctypes.data_as(ctypes.c_void_p), b.nbytes, h))
    return h

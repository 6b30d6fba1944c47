"""One process per GPU: axis-0 slabs of a hotspot grid, halo planes exchanged by NCCL in-graph.

SURVEY.md §8e: the large Hotspot3D grid (2048x2048x256) is partitioned along axis 0 with the
reference's row-slab bounds ``rows*g//P`` (workloads.py:60-69). Rank g owns rows [lo, hi) and one
halo plane per interior face. After every iteration's stencil kernel the runtime sends its first
owned plane to rank g-1 and its last to rank g+1 and receives theirs into its halos — one NCCL
group on the launch stream, captured into the iteration-batch graph together with the kernels
(``ib_create_dist`` in include/iterbatch_b200.h). The exchange plan is restated in pure Python
(``exchange_plan``) so the CPU tests can run the same protocol over gloo against the oracle.

Launch with torchrun (RANK / WORLD_SIZE / LOCAL_RANK); ``torch.distributed`` only carries the
128-byte NCCL id and the final gather — the data path is the runtime's own NCCL communicator.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .workloads import DeviceSolver, Times, _dims_scalars, _kind_of_state, _norm_dtype, _NP_DTYPE

__all__ = ["slab_bounds", "halo_window", "exchange_plan", "unique_id", "seeded_window",
           "DistributedSolver"]


def slab_bounds(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) of rank's slab — the reference's bounds formula (workloads.py:65)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    if world > rows:
        raise ValueError("more ranks than rows along axis 0")
    return rows * rank // world, rows * (rank + 1) // world


def halo_window(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Global rows a rank uploads: its slab plus one halo row per interior face."""
    lo, hi = slab_bounds(rows, world, rank)
    return lo - (1 if rank > 0 else 0), hi + (1 if rank < world - 1 else 0)


def exchange_plan(rows: int, world: int, rank: int) -> list[tuple[str, int, int, int]]:
    """(op, peer, local_row) of one iteration's halo exchange, in the runtime's order.

    local_row indexes the rank's slab buffer of (hi - lo + 2) planes: 0 = top halo,
    1..n = owned rows, n+1 = bottom halo (runtime.cu: nccl_exchange).
    """
    lo, hi = slab_bounds(rows, world, rank)
    n = hi - lo
    plan = []
    if rank > 0:
        plan += [("send", rank - 1, 1), ("recv", rank - 1, 0)]
    if rank < world - 1:
        plan += [("send", rank + 1, n), ("recv", rank + 1, n + 1)]
    return plan


def seeded_window(shape, rank: int, world: int, seed: int = 20240817):
    """This rank's (temperature window with halo rows, power rows) of the reference's seeded input.

    The reference builds T = rng.random(shape) then P = rng.random(shape) * 1e-3 from one
    default_rng(seed) stream (cli.py:173,182,192). PCG64 draws one 64-bit word per double, so a
    rank advances the bit generator to its first row and draws only its window — the values are
    identical to slicing the global arrays, without any rank materialising them.
    """
    shape = tuple(int(x) for x in shape)
    rows = shape[0]
    plane = int(np.prod(shape[1:]))
    lo, hi = slab_bounds(rows, world, rank)
    wlo, whi = halo_window(rows, world, rank)
    bg = np.random.PCG64(seed)
    bg.advance(wlo * plane)
    t = np.random.Generator(bg).random((whi - wlo,) + shape[1:])
    bg = np.random.PCG64(seed)
    bg.advance(rows * plane + lo * plane)
    p = np.random.Generator(bg).random((hi - lo,) + shape[1:]) * 1e-3
    return t, p


def unique_id() -> bytes:
    """A fresh NCCL unique id (call on rank 0, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _lib.check(_lib.lib().ib_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


class DistributedSolver(DeviceSolver):
    """This rank's slab of a global hotspot grid, resident on one GPU.

    ``state`` is the GLOBAL HotspotWorkload (each rank only uploads its window). Graph builds
    are stream-captured (the exchange is part of every iteration). Two exchanges:

    * ``exchange="nccl"`` (``uid`` = rank 0's NCCL id): one NCCL send/recv group per iteration;
    * ``exchange="peer"`` (``allgather`` = a callable gathering one bytes object per rank, e.g.
      over torch.distributed): the stencil kernel stores its boundary planes straight into the
      neighbours' halo planes through CUDA IPC mappings (NVLink peer stores), ordered across
      processes by device-side iteration counters (include/iterbatch_b200.h, ib_ipc_attach).
    """

    def __init__(self, state, dtype, rank: int, world: int, device: int, uid: bytes | None = None,
                 upload: bool = True, exchange: str = "nccl", allgather=None, fuse: bool = False,
                 timeout_ms: int | None = None):
        kind = _kind_of_state(state)
        if kind not in ("hotspot2d", "hotspot3d", "fdtd"):
            raise ValueError("distributed execution is defined for hotspot grids and FDTD")
        if fuse and kind != "fdtd":
            raise ValueError("fuse=True applies to FDTD (H and E half-steps in one kernel)")
        self.fused = bool(fuse)
        if kind == "fdtd" and world > 1 and exchange != "peer":
            raise ValueError("distributed FDTD uses exchange='peer'")
        self.kind = kind
        self.dtype = _norm_dtype(dtype)
        self.np_dtype = _NP_DTYPE[self.dtype]
        self.dims, self.scalars = _dims_scalars(kind, state)
        self.devices = (device,)
        self.rank, self.world = rank, world
        # axis-0 units: hotspot rows, FDTD lattice planes (nx + 1)
        self.rows = self.dims[0] + (1 if kind == "fdtd" else 0)
        self.lo, self.hi = slab_bounds(self.rows, world, rank)
        self.wlo, self.whi = halo_window(self.rows, world, rank)
        L = _lib.lib()
        ctx = ctypes.c_void_p()
        dims = (ctypes.c_int64 * len(self.dims))(*self.dims)
        sc = (ctypes.c_double * len(self.scalars))(*self.scalars)
        if exchange not in ("nccl", "peer"):
            raise ValueError(f"exchange must be 'nccl' or 'peer', got {exchange!r}")
        self.exchange = exchange
        idp = None
        if world > 1 and exchange == "nccl":
            if uid is None or len(uid) != 128:
                raise ValueError("world > 1 needs the 128-byte NCCL unique id from rank 0")
            self._uid = ctypes.create_string_buffer(uid, 128)
            idp = ctypes.cast(self._uid, ctypes.c_void_p)
        if world > 1 and exchange == "peer" and allgather is None:
            raise ValueError("exchange='peer' needs an allgather callable for the IPC handles")
        _lib.check(L.ib_create_dist(ctypes.byref(ctx), _lib.SOLVER["fdtd_fused" if self.fused else kind],
                                    _lib.DTYPE[self.dtype], dims,
                                    len(self.dims), sc, len(self.scalars), device, rank, world, idp))
        self._ctx = ctx
        if timeout_ms is not None:  # the in-graph wait kernel's trap deadline (ib_set_dist_timeout)
            _lib.check(L.ib_set_dist_timeout(ctx, int(timeout_ms)))
        self._allgather = allgather if (world > 1 and exchange == "peer") else None
        if self._allgather is not None:
            self._attach_peers(allgather)
        if kind == "fdtd":
            self.nfields = 6
            self.field_shapes = []
            for f in range(6):
                shp = (ctypes.c_int64 * 3)()
                nd = ctypes.c_int()
                _lib.check(L.ib_field_shape(ctx, f, shp, ctypes.byref(nd)))
                self.field_shapes.append(tuple(shp[:3]))
            # download: owned planes [lo, hi) of each field, clipped to its extent (the header)
            self.shapes = [(max(0, min(self.hi, fs[0]) - min(self.lo, fs[0])),) + fs[1:]
                           for fs in self.field_shapes]
        else:
            self.nfields = 2
            plane = tuple(self.dims[1:])
            self.shapes = [(self.hi - self.lo,) + plane, (self.hi - self.lo,) + plane]
        self.batch_size = 0
        if upload:
            self.upload(state)

    def _attach_peers(self, allgather) -> None:
        """Swap IPC handles with every rank and map the two neighbours' buffers."""
        L = _lib.lib()
        mine = ctypes.create_string_buffer(_lib.IPC_BYTES)
        _lib.check(L.ib_ipc_export(self.ctx, ctypes.cast(mine, ctypes.c_void_p), _lib.IPC_BYTES))
        handles = list(allgather(mine.raw))
        if len(handles) != self.world:
            raise RuntimeError(f"allgather returned {len(handles)} handle sets for world {self.world}")
        keep = []

        def ptr(blob):
            if blob is None:
                return None
            b = ctypes.create_string_buffer(bytes(blob), _lib.IPC_BYTES)
            keep.append(b)
            return ctypes.cast(b, ctypes.c_void_p)

        up = handles[self.rank - 1] if self.rank > 0 else None
        dn = handles[self.rank + 1] if self.rank + 1 < self.world else None
        _lib.check(L.ib_ipc_attach(self.ctx, ptr(up), ptr(dn)))

    @classmethod
    def from_seed(cls, shape, k: float, dtype, rank: int, world: int, device: int,
                  uid: bytes | None, seed: int = 20240817, exchange: str = "nccl",
                  allgather=None) -> "DistributedSolver":
        """Build this rank's slab of the reference generator's grid (cli.py:183-192) directly."""

        class _Shape:  # the global state's metadata only; the arrays come from seeded_window
            def __init__(self, shape, k):
                self.temperature = np.lib.stride_tricks.as_strided(np.zeros(1), shape, [0] * len(shape))
                self.power = self.temperature
                self.diffusion_coefficient = float(k)

        solver = cls(_Shape(shape, k), dtype, rank, world, device, uid, upload=False,
                     exchange=exchange, allgather=allgather)
        t, p = seeded_window(shape, rank, world, seed)
        solver.upload([t, p])
        return solver

    def host_arrays(self, state):
        if self.kind == "fdtd":  # every field's window: [lo - top, hi + bot) clipped to its extent
            out = []
            for a, fs in zip(state.state_arrays(), self.field_shapes):
                lo, hi = min(self.wlo, fs[0]), min(self.whi, fs[0])
                out.append(np.ascontiguousarray(a[lo:hi], dtype=self.np_dtype))
            return out
        t = np.ascontiguousarray(state.temperature[self.wlo:self.whi], dtype=self.np_dtype)
        p = np.ascontiguousarray(state.power[self.lo:self.hi], dtype=self.np_dtype)
        return [t, p]

    def upload(self, state, fields=None) -> None:
        arrs = state if isinstance(state, (list, tuple)) else self.host_arrays(state)
        L = _lib.lib()
        for f, a in enumerate(arrs):
            if fields is not None and f not in fields:
                continue
            a = np.ascontiguousarray(a, dtype=self.np_dtype)
            _lib.check(L.ib_upload(self.ctx, f, a.ctypes.data_as(ctypes.c_void_p), a.nbytes))
        if self._allgather is not None:
            # peer exchange: a neighbour's first kernel stores into this rank's halo planes, so
            # no rank may start running before every rank's upload has landed (host barrier)
            self._allgather(b"")

    def build_graph(self, batch_size: int, build: str = "capture", pdl: bool = False,
                    device_launch: bool = False, upload: bool = True,
                    while_loop: bool = False, meminfo: bool = False) -> Times:
        t = super().build_graph(batch_size, "capture", pdl, False, upload, False, meminfo)
        if self._allgather is not None:
            # peer exchange: a rank still capturing / instantiating would leave its neighbours'
            # in-graph wait kernels spinning towards their trap deadline — no rank launches
            # before every rank's graph exists (host barrier)
            self._allgather(b"")
        return t

    def run_batched(self, batch_size: int, num_batches: int, build: str = "capture",
                    pdl: bool = False, while_loop: bool = False) -> Times:
        """Build, (peer exchange: host barrier,) replay, destroy. ``gpu_s`` is T_C + T_E: the
        device time of the launches plus the host time of the build (NCCL: one device interval
        from before the build, as DeviceSolver.run_batched)."""
        if self._allgather is None:
            return super().run_batched(batch_size, num_batches, "capture", pdl, False)
        tb = self.build_graph(batch_size, pdl=pdl)
        te = self.run_graph(num_batches)
        self.destroy_graph()
        return Times(create_s=tb.create_s, instantiate_s=tb.instantiate_s, upload_s=tb.upload_s,
                     build_s=tb.build_s + te.build_s, exec_s=te.exec_s, gpu_s=tb.build_s + te.gpu_s,
                     kernels=te.kernels, launches=te.launches, nodes=tb.nodes)

    def local_temperature(self) -> np.ndarray:
        """This rank's owned rows [lo, hi) of the current temperature."""
        return self.download_field(0)

    def local_fields(self) -> list[np.ndarray]:
        """FDTD: this rank's owned planes [lo, hi) of every field (clipped to each extent)."""
        return [self.download_field(f) for f in range(self.nfields)]

    @property
    def iteration_bytes(self) -> int:
        if self.kind == "fdtd":  # this rank's share of the global H + E half-step bytes
            g = int(_lib.lib().ib_iteration_bytes(self.ctx))
            return g * (self.hi - self.lo) // self.rows
        return 3 * int(np.prod(self.shapes[0])) * np.dtype(self.np_dtype).itemsize

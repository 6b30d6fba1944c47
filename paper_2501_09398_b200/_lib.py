"""ctypes binding of libiterbatch_b200.so (declarations: include/iterbatch_b200.h).

The library is REQUIRED: there is no CPU fallback anywhere in this package. If the shared object
is missing, or no CUDA device is visible, calls fail loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IB_LIB_PATH") or os.path.join(PKG, "libiterbatch_b200.so")  # override: A/B tooling

IB_OK, IB_EINVAL, IB_ECUDA, IB_ENOMEM, IB_ESTATE, IB_ENODEV = 0, -1, -2, -3, -4, -5
SOLVER = {"vector": 0, "hotspot2d": 1, "hotspot3d": 2, "fdtd": 3, "fdtd_fused": 4}
DTYPE = {"f32": 0, "f64": 1}
BUILD = {"manual": 0, "capture": 1}
FLAG_PDL, FLAG_DEVICE_LAUNCH, FLAG_NO_UPLOAD, FLAG_WHILE, FLAG_MEMINFO, FLAG_PATCH = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20

FNV_OFFSET = 0xCBF29CE484222325


class IbTimes(ctypes.Structure):
    _fields_ = [
        ("create_s", ctypes.c_double),
        ("instantiate_s", ctypes.c_double),
        ("upload_s", ctypes.c_double),
        ("build_s", ctypes.c_double),
        ("exec_s", ctypes.c_double),
        ("gpu_s", ctypes.c_double),
        ("kernels", ctypes.c_int64),
        ("launches", ctypes.c_int64),
        ("nodes", ctypes.c_int64),
        ("graph_bytes", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lock = threading.Lock()

IPC_BYTES = 192  # IB_IPC_BYTES

# (name, restype, argtypes) — must match include/iterbatch_b200.h
_P, _I, _I64, _SZ, _U64, _D = (
    ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_double,
)
_T = ctypes.POINTER(IbTimes)
PROTOTYPES = [
    ("ib_abi_version", _I, []),
    ("ib_last_error", ctypes.c_char_p, []),
    ("ib_device_count", _I, [ctypes.POINTER(_I)]),
    ("ib_mem_info", _I, [_I, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("ib_create", _I, [ctypes.POINTER(_P), _I, _I, ctypes.POINTER(_I64), _I, ctypes.POINTER(_D), _I,
                       ctypes.POINTER(_I), _I]),
    ("ib_destroy", None, [_P]),
    ("ib_num_fields", _I, [_P]),
    ("ib_field_shape", _I, [_P, _I, ctypes.POINTER(_I64), ctypes.POINTER(_I)]),
    ("ib_field_bytes", _I64, [_P, _I]),
    ("ib_upload", _I, [_P, _I, _P, _SZ]),
    ("ib_download", _I, [_P, _I, _P, _SZ]),
    ("ib_iteration_bytes", _I64, [_P]),
    ("ib_run_stream", _I, [_P, _I64, _I, _T]),
    ("ib_run_step", _I, [_P, _I, _T]),
    ("ib_num_steps", _I, [_P]),
    ("ib_graph_build", _I, [_P, _I64, _I, _I, _T]),
    ("ib_graph_run", _I, [_P, _I64, _T]),
    ("ib_graph_destroy", _I, [_P]),
    ("ib_run_batched", _I, [_P, _I64, _I64, _I, _I, _T]),
    ("ib_run_peeled", _I, [_P, _I64, _I64, _I, _I, _T]),
    ("ib_graph_batch_size", _I64, [_P]),
    ("ib_sync", _I, [_P]),
    ("ib_host_alloc", _I, [ctypes.POINTER(_P), _SZ]),
    ("ib_host_free", _I, [_P]),
    ("ib_fnv1a64", _U64, [_P, _SZ, _U64]),
    ("ib_fnv1a64_f64", _U64, [_P, _SZ, _I, _U64]),
    ("ib_nccl_unique_id", _I, [_P]),
    ("ib_create_dist", _I, [ctypes.POINTER(_P), _I, _I, ctypes.POINTER(_I64), _I, ctypes.POINTER(_D), _I,
                            _I, _I, _I, _P]),
    ("ib_slab_info", _I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I),
                          ctypes.POINTER(_I)]),
    ("ib_describe", _I64, [_P, ctypes.c_char_p, _I64]),
    ("ib_set_halo_mode", _I, [_P, _I]),
    ("ib_ipc_export", _I, [_P, _P, _SZ]),
    ("ib_ipc_attach", _I, [_P, _P, _P]),
    ("ib_set_dist_timeout", _I, [_P, ctypes.c_int64]),
    ("ib_trace_enable", _I, [_P, _I64]),
    ("ib_trace_kernels", _I64, [_P, ctypes.POINTER(_I64), _I64]),
    ("ib_trace_host_events", _I64, [_P, ctypes.POINTER(_I64), _I64]),
    ("ib_flush_l2", _I, [_P]),
]


class LibraryMissingError(ImportError):
    pass


def _point_at_torch_nccl() -> None:
    """Let the runtime dlopen the NCCL wheel torch links against (not an older system copy)."""
    if os.environ.get("IB_NCCL_LIB"):
        return
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["IB_NCCL_LIB"] = cand
            return


def lib():
    """Load the runtime library (once). Raises LibraryMissingError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissingError(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2501_09398_b200.build` "
                    "(this package has no CPU fallback)"
                )
            _point_at_torch_nccl()
            L = ctypes.CDLL(LIB_PATH)
            for name, res, args in PROTOTYPES:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            if L.ib_abi_version() != 1:
                raise LibraryMissingError("libiterbatch_b200.so ABI version mismatch; rebuild it")
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().ib_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map an IB_* status to the reference's exception convention."""
    if rc == IB_OK:
        return
    msg = last_error()
    if rc == IB_EINVAL:
        raise ValueError(msg)
    if rc == IB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"iterbatch_b200 error {rc}: {msg}")


def device_count() -> int:
    n = ctypes.c_int(0)
    lib().ib_device_count(ctypes.byref(n))
    return n.value

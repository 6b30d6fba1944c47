"""Pageable vs register-in-place H2D of the headline's 8 MB fields (diagnostic): cudaMemcpy from
a numpy array as is, against cudaHostRegister + cudaMemcpy + cudaHostUnregister of the same array
(measured: 0.43-0.49 ms pageable vs 2.2-4.3 ms registering — the drop-in path keeps pageable
copies), and cudaMemcpyAsync on a non-blocking stream vs cudaMemcpy (equal).
    python tools/h2d_pin_probe.py"""
import ctypes
import statistics
import time

import numpy as np
import torch

import glob  # noqa: E402
import os  # noqa: E402

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
cr = ctypes.CDLL(cands[0] if cands else "libcudart.so")
dev = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
a = np.random.default_rng(1).random(1 << 20)
ptr, n = a.ctypes.data, a.nbytes
dptr = dev.data_ptr()
cr.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
cr.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
cr.cudaHostUnregister.argtypes = [ctypes.c_void_p]
for name in ("pageable", "register+copy+unregister", "pageable", "register+copy+unregister"):
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        if name.startswith("register"):
            assert cr.cudaHostRegister(ptr, n, 0) == 0
            assert cr.cudaMemcpy(dptr, ptr, n, 1) == 0
            assert cr.cudaHostUnregister(ptr) == 0
        else:
            assert cr.cudaMemcpy(dptr, ptr, n, 1) == 0
        ts.append(time.perf_counter() - t0)
    print(f"{name:28s} 8 MB H2D: median {1e3 * statistics.median(ts[2:]):.3f} ms")
# cudaMemcpyAsync on a non-blocking stream (the runtime's transfers) vs synchronous cudaMemcpy
cr.cudaStreamCreateWithFlags.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_uint]
cr.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
cr.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]
st = ctypes.c_void_p()
assert cr.cudaStreamCreateWithFlags(ctypes.byref(st), 1) == 0
b = np.random.default_rng(2).random(1 << 20)  # a second array, as T and P
for name in ("async non-blocking", "sync cudaMemcpy", "async, two arrays", "sync, two arrays", "D2H async", "D2H sync"):
    ts = []
    for _ in range(20):
        out = np.empty(1 << 20)
        t0 = time.perf_counter()
        if name == "async non-blocking":
            cr.cudaMemcpyAsync(dptr, ptr, n, 1, st); cr.cudaStreamSynchronize(st)
        elif name == "sync cudaMemcpy":
            cr.cudaMemcpy(dptr, ptr, n, 1)
        elif name == "async, two arrays":
            for q in (a, b):
                cr.cudaMemcpyAsync(dptr, q.ctypes.data, n, 1, st); cr.cudaStreamSynchronize(st)
        elif name == "sync, two arrays":
            for q in (a, b):
                cr.cudaMemcpy(dptr, q.ctypes.data, n, 1)
        elif name == "D2H async":
            cr.cudaMemcpyAsync(out.ctypes.data, dptr, n, 2, st); cr.cudaStreamSynchronize(st)
        else:
            cr.cudaMemcpy(out.ctypes.data, dptr, n, 2)
        ts.append(time.perf_counter() - t0)
    print(f"{name:28s} median {1e3 * statistics.median(ts[2:]):.3f} ms")

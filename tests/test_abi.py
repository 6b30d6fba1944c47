"""The C ABI library builds, loads, and exports every symbol include/iterbatch_b200.h declares.

CPU-only: no compute calls. On a machine without a CUDA device every entry point that needs one
must fail loudly (IB_ENODEV -> RuntimeError), never fall back to the CPU.
"""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2501_09398_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "iterbatch_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ib_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("ib_create", "ib_upload", "ib_download", "ib_run_stream", "ib_graph_build",
                 "ib_graph_run", "ib_destroy", "ib_last_error", "ib_fnv1a64"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode == 0:
        exported = set(line.split()[-1] for line in out.stdout.splitlines() if line.strip())
        for name in _declared():
            assert name in exported, name


def test_python_prototypes_cover_the_header():
    assert sorted(n for n, _, _ in _lib.PROTOTYPES) == _declared()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_fnv_native_matches_python():
    from tests.test_oracle import _fnv_py

    L = _lib.lib()
    b = np.random.default_rng(1).random(33)
    raw = b.astype("<f8").tobytes()
    buf = ctypes.create_string_buffer(raw, len(raw))
    assert L.ib_fnv1a64(ctypes.cast(buf, ctypes.c_void_p), len(raw), _lib.FNV_OFFSET) == _fnv_py(raw)
    f = b.astype(np.float32)
    h = L.ib_fnv1a64_f64(f.ctypes.data_as(ctypes.c_void_p), f.size, _lib.DTYPE["f32"], _lib.FNV_OFFSET)
    assert h == _fnv_py(f.astype("<f8").tobytes())


def test_no_device_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    from paper_2501_09398_b200 import workloads as wl

    w = wl.VectorWorkload(np.ones(8), 0.5)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        wl.run_loop(wl.vector_program(), w, 2)
    with pytest.raises(RuntimeError):
        wl.run_batched(wl.vector_program(), w, 2, 2)


def test_create_validates_arguments_before_touching_a_device():
    L = _lib.lib()
    ctx = ctypes.c_void_p()
    dims = (ctypes.c_int64 * 2)(4, 4)
    sc = (ctypes.c_double * 1)(0.1)
    assert L.ib_create(ctypes.byref(ctx), 9, 0, dims, 2, sc, 1, None, 0) == _lib.IB_EINVAL
    assert "unknown solver" in _lib.last_error()
    assert L.ib_create(ctypes.byref(ctx), 1, 7, dims, 2, sc, 1, None, 0) == _lib.IB_EINVAL
    assert L.ib_create(ctypes.byref(ctx), 1, 0, dims, 3, sc, 1, None, 0) == _lib.IB_EINVAL
    bad = (ctypes.c_int64 * 2)(0, 4)
    assert L.ib_create(ctypes.byref(ctx), 1, 0, bad, 2, sc, 1, None, 0) == _lib.IB_EINVAL
    assert L.ib_graph_run(None, 1, None) == _lib.IB_EINVAL


def test_plain_c_caller_compiles_and_links(tmp_path):
    """examples/hotspot_c.c: the C ABI is usable from C alone (gcc, the header, the .so)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib_dir = os.path.join(ROOT, "paper_2501_09398_b200")
    out = tmp_path / "hotspot_c"
    r = subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-o", str(out),
                        os.path.join(ROOT, "examples", "hotspot_c.c"), "-L", lib_dir, "-literbatch_b200",
                        f"-Wl,-rpath,{lib_dir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

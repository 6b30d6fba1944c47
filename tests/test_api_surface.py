"""The drop-in claim, checked against the reference itself where it is importable (this build
container; /root/reference does not exist on the GPU box, so these skip there): every public
name of iterbatch.workloads exists here with the reference's parameters in the reference's
order (extras may only follow, keyword-style), the same dataclass fields, the same constants,
and the same validation errors on bad input."""
import dataclasses
import importlib
import inspect
import os
import sys

import numpy as np
import pytest

from paper_2501_09398_b200 import workloads as ours

REF_SRC = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF_SRC)
    try:
        yield importlib.import_module("iterbatch.workloads")
    finally:
        sys.path.remove(REF_SRC)


def test_every_public_name_exists(ref):
    missing = [n for n in ref.__all__ if not hasattr(ours, n)]
    assert not missing


def test_function_parameters_are_a_prefix(ref):
    for name in ref.__all__:
        r = getattr(ref, name)
        if not inspect.isfunction(r):
            continue
        rp = list(inspect.signature(r).parameters.values())
        op = list(inspect.signature(getattr(ours, name)).parameters.values())
        assert [p.name for p in op[: len(rp)]] == [p.name for p in rp], name
        for a, b in zip(rp, op):
            assert a.kind == b.kind or b.kind == inspect.Parameter.POSITIONAL_OR_KEYWORD, (name, a.name)
            if a.default is not inspect.Parameter.empty:
                assert b.default == a.default, (name, a.name)
        for extra in op[len(rp):]:  # additions never displace a reference argument
            assert extra.default is not inspect.Parameter.empty, (name, extra.name)


def test_dataclass_fields_and_constants(ref):
    for name in ("VectorWorkload", "HotspotWorkload", "FdtdWorkload"):
        rf = [f.name for f in dataclasses.fields(getattr(ref, name))]
        of = [f.name for f in dataclasses.fields(getattr(ours, name))]
        assert of == rf, name
    for name in ("VACUUM_LIGHT_SPEED", "VACUUM_PERMEABILITY", "VACUUM_PERMITTIVITY"):
        assert getattr(ours, name) == getattr(ref, name)
    assert [m.name for m in ours.ExecutionOrder] == [m.name for m in ref.ExecutionOrder]


BAD_INPUTS = [
    ("VectorWorkload", (np.ones(0), 0.5)),
    ("HotspotWorkload", (np.ones((4, 4)), np.ones((4, 4)), 0.3)),
    ("HotspotWorkload", (np.ones((2, 2, 2, 2)), np.ones((2, 2, 2, 2)), 0.1)),
    ("VectorWorkload", (np.ones((2, 2)), 0.5)),
    ("HotspotWorkload", (np.ones((4, 4)), np.ones((4, 3)), 0.1)),
    ("HotspotWorkload", (np.ones(4), np.ones(4), 0.1)),
    ("HotspotWorkload", (np.ones((4, 4)), np.ones((4, 4)), -1.0)),
]


@pytest.mark.parametrize("name,args", BAD_INPUTS)
def test_validation_errors_match(ref, name, args):
    with pytest.raises(Exception) as er:
        getattr(ref, name)(*args)
    with pytest.raises(Exception) as eo:
        getattr(ours, name)(*args)
    assert type(eo.value) is type(er.value)
    assert str(eo.value) == str(er.value)


def test_run_driver_argument_errors_match(ref):
    rng = np.random.default_rng(0)
    st_ref = ref.HotspotWorkload(rng.random((8, 8)), rng.random((8, 8)), 0.1)
    st_our = ours.HotspotWorkload(st_ref.temperature, st_ref.power, 0.1)
    for call in (lambda m, s: m.run_loop(m.hotspot_program(), s, -1),
                 lambda m, s: m.run_batched(m.hotspot_program(), s, 0, 3),
                 lambda m, s: m.run_batched(m.hotspot_program(), s, 2, -1)):
        with pytest.raises(Exception) as er:
            call(ref, st_ref)
        with pytest.raises(Exception) as eo:
            call(ours, st_our)
        assert type(eo.value) is type(er.value) and str(eo.value) == str(er.value)


def test_fdtd_factories_match(ref):
    for args in ((4, 3, 5), (2, 2, 2, 0.5, 0.7)):
        a, b = ref.fdtd_cavity(*args), ours.fdtd_cavity(*args)
        assert a.time_step == b.time_step and a.cell_size == b.cell_size
        assert [x.shape for x in a.state_arrays()] == [x.shape for x in b.state_arrays()]
    a, b = ref.te101_cavity(6, 3, 5), ours.te101_cavity(6, 3, 5)
    assert all(np.array_equal(x, y) for x, y in zip(a.state_arrays(), b.state_arrays()))
    for bad in ((0, 2, 2), (2, 2, 2, 1.0, 1.5)):
        with pytest.raises(Exception) as er:
            ref.fdtd_cavity(*bad)
        with pytest.raises(Exception) as eo:
            ours.fdtd_cavity(*bad)
        assert type(eo.value) is type(er.value) and str(eo.value) == str(er.value)


def test_checksum_is_the_references(ref):
    rng = np.random.default_rng(1)
    st = ref.HotspotWorkload(rng.random((6, 5)), rng.random((6, 5)), 0.1)
    assert ours.state_checksum(st) == ref.state_checksum(st)

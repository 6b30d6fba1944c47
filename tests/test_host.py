"""Host-side logic of the drop-in API (no device needed): validation, plans, CLI, generators."""

import numpy as np
import pytest

from paper_2501_09398_b200 import cli
from paper_2501_09398_b200 import workloads as wl
from paper_2501_09398_b200.fitting import MeasurementPoint, MeasurementSeries, write_measurements_csv
from paper_2501_09398_b200.model import BatchPlan, feasible_batch_sizes


def test_batch_plan_mirrors_reference():
    p = BatchPlan.from_batch_size(10000, 100)
    assert (p.total_kernel_executions, p.batch_size, p.num_batches) == (10000, 100, 100)
    with pytest.raises(ValueError, match="does not divide"):
        BatchPlan.from_batch_size(10, 3)
    with pytest.raises(ValueError):
        BatchPlan(6, 2, 4)
    with pytest.raises(TypeError):
        BatchPlan.from_batch_size(10, 2.5)


def test_feasible_batch_sizes_match_survey_table():
    assert feasible_batch_sizes(1000) == (1, 2, 4, 5, 8, 10, 20, 25, 40, 50, 100, 125, 200, 250, 500, 1000)
    assert len([d for d in feasible_batch_sizes(10000) if d <= 2000]) == 22


def test_dataclass_validation_mirrors_reference():
    with pytest.raises(ValueError):
        wl.VectorWorkload(np.ones((2, 2)), 0.5)
    with pytest.raises(ValueError, match="must not be empty"):
        wl.VectorWorkload(np.ones(0), 0.5)
    with pytest.raises(ValueError, match="stable range"):
        wl.HotspotWorkload(np.zeros((4, 4)), np.zeros((4, 4)), 0.26)
    with pytest.raises(ValueError, match="stable range"):
        wl.HotspotWorkload(np.zeros((4, 4, 4)), np.zeros((4, 4, 4)), 0.18)
    with pytest.raises(ValueError, match="shape"):
        wl.HotspotWorkload(np.zeros((4, 4)), np.zeros((4, 5)), 0.2)
    with pytest.raises(ValueError, match="2-D or 3-D"):
        wl.HotspotWorkload(np.zeros(16), np.zeros(16), 0.2)
    w = wl.fdtd_cavity(4, 5, 6)
    assert w.dims == (4, 5, 6) and w.ex.shape == (4, 6, 7) and w.hz.shape == (4, 5, 7)
    with pytest.raises(ValueError, match="ey shape"):
        wl.FdtdWorkload(w.ex, np.zeros((4, 4, 4)), w.ez, w.hx, w.hy, w.hz, w.cell_size, w.time_step)
    with pytest.raises(ValueError, match="courant"):
        wl.fdtd_cavity(4, 4, 4, courant=1.01)
    with pytest.raises(ValueError):
        wl.FdtdWorkload(w.ex, w.ey, w.ez, w.hx, w.hy, w.hz, w.cell_size, 0.0)


def test_te101_matches_reference_profile():
    import math

    w = wl.te101_cavity(8, 4, 8)
    assert not w.ex.any() and not w.ez.any() and not w.hx.any()
    assert w.ey[4, 2, 4] == pytest.approx(math.sin(math.pi * 4 / 8) ** 2, rel=1e-12)
    assert not w.ey[0].any() and not w.ey[-1].any() and not w.ey[:, :, 0].any()


def test_program_dispatch_and_errors():
    v = wl.VectorWorkload(np.ones(4), 0.5)
    assert wl._check_program(wl.vector_program(), v) == "vector"
    h = wl.HotspotWorkload(np.zeros((3, 3, 3)), np.zeros((3, 3, 3)), 0.1)
    assert wl._check_program(wl.hotspot_program(), h) == "hotspot3d"
    with pytest.raises(ValueError, match="does not apply"):
        wl._check_program(wl.fdtd_program(), h)
    with pytest.raises(ValueError, match="no device implementation"):
        wl._check_program(wl.ChainProgram((lambda s, w=None: s,)), v)
    with pytest.raises(ValueError):
        wl.ChainProgram(())
    assert wl.fdtd_program().steps == (wl.fdtd_h_step, wl.fdtd_e_step)


def test_driver_argument_errors_precede_device_use():
    v = wl.VectorWorkload(np.ones(4), 0.5)
    with pytest.raises(ValueError):
        wl.run_loop(wl.vector_program(), v, -1)
    with pytest.raises(ValueError):
        wl.run_batched(wl.vector_program(), v, 0, 5)
    with pytest.raises(ValueError):
        wl.run_batched(wl.vector_program(), v, 2, -1)
    with pytest.raises(TypeError):
        wl.run_loop(wl.vector_program(), v, 2.0)
    assert wl.run_loop(wl.vector_program(), v, 0) is v
    assert wl.run_batched(wl.vector_program(), v, 3, 0) is v
    assert wl.ExecutionOrder.LOOP.value == "loop" and wl.ExecutionOrder.BATCHED.value == "batched"


def test_reference_generators_are_reproduced():
    v = cli.build_workload("vector", [16])
    assert np.array_equal(v.values, np.random.default_rng(20240817).random(16))
    h = cli.build_workload("hotspot3d", [4, 2])
    assert h.temperature.shape == (4, 4, 2) and h.diffusion_coefficient == 0.1
    f = cli.build_workload("fdtd", [3, 2, 4])
    assert f.dims == (3, 2, 4)
    with pytest.raises(cli.UsageError):
        cli.build_workload("vector", [8, 8])


def test_cli_usage_errors(capsys):
    code = cli.main(["run-workload", "--workload", "vector", "--size", "64", "--iterations", "4",
                     "--batch-size", "2", "--mode", "loop"])
    assert code == 2 and "usage error" in capsys.readouterr().err
    code = cli.main(["run-workload", "--workload", "vector", "--size", "64", "--iterations", "5",
                     "--batch-size", "2", "--mode", "batched", "--checksum"])
    assert code == 1 and "does not divide" in capsys.readouterr().err


def test_measurement_csv_schema(tmp_path):
    s = MeasurementSeries((MeasurementPoint(2, (0.1, 0.2)), MeasurementPoint(4, (0.05,))), "x")
    p = tmp_path / "m.csv"
    write_measurements_csv(s, p)
    lines = p.read_text().splitlines()
    assert lines[0] == "# schema=1" and lines[1] == "batch_size,run_index,seconds"
    assert lines[2] == "2,0,0.100000000" and lines[4] == "4,0,0.050000000"


def test_reference_dataclasses_are_accepted_duck_typed():
    """A reference-style state object (any class with the same fields) is dispatched by shape."""

    class RefVector:
        def __init__(self, values, c):
            self.values, self.scale_constant = np.asarray(values, float), float(c)

        def state_arrays(self):
            return (self.values,)

    r = RefVector(np.ones(5), 0.5)
    assert wl._kind_of_state(r) == "vector"
    assert wl._dims_scalars("vector", r) == ((5,), (0.5,))
    out = wl._rebuild(r, [np.zeros(5)])
    assert isinstance(out, RefVector) and out.scale_constant == 0.5

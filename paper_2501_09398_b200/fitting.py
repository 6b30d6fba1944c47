"""Measurement containers emitted by the timing harness.

Mirror of the reference's ``MeasurementPoint`` / ``MeasurementSeries``
(pkg/src/iterbatch/fitting.py:28-64) and of its measurement-CSV writer
(pkg/src/iterbatch/fileio.py:184-190, header ``batch_size,run_index,seconds`` under
``# schema=1``, seconds with 9 decimals) so that the reference's ``iterbatch fit`` /
``optimize`` / ``speedup`` commands read this package's B200 measurements unchanged.
"""

from __future__ import annotations

import operator
import statistics
from dataclasses import dataclass

__all__ = ["MeasurementPoint", "MeasurementSeries", "write_measurements_csv", "MEASUREMENT_HEADER"]

MEASUREMENT_HEADER = "batch_size,run_index,seconds"


@dataclass(frozen=True)
class MeasurementPoint:
    """Repeated wall-clock samples for one batch size."""

    batch_size: int
    samples: tuple[float, ...]

    def __post_init__(self):
        size = operator.index(self.batch_size)
        if size < 1:
            raise ValueError(f"batch_size must be positive, got {size}")
        object.__setattr__(self, "batch_size", size)
        samples = tuple(float(s) for s in self.samples)
        if not samples:
            raise ValueError("a measurement point needs at least one sample")
        for s in samples:
            if not s > 0.0:
                raise ValueError(f"samples must be positive, got {s!r}")
        object.__setattr__(self, "samples", samples)

    def mean(self) -> float:
        return statistics.fmean(self.samples)


@dataclass(frozen=True)
class MeasurementSeries:
    points: tuple[MeasurementPoint, ...]
    label: str = ""

    def __post_init__(self):
        points = tuple(self.points)
        if not points:
            raise ValueError("a measurement series needs at least one point")
        object.__setattr__(self, "points", points)

    def batch_sizes(self) -> tuple[int, ...]:
        return tuple(p.batch_size for p in self.points)


def write_measurements_csv(series: MeasurementSeries, path) -> None:
    with open(path, "w") as fh:
        fh.write("# schema=1\n")
        fh.write(MEASUREMENT_HEADER + "\n")
        for point in series.points:
            for run, seconds in enumerate(point.samples):
                fh.write(f"{point.batch_size},{run},{seconds:.9f}\n")

"""BatchPlan: the factorisation I_k = S x I of the total kernel count (Eq. 4).

Mirrors the reference's ``iterbatch.model.BatchPlan`` (pkg/src/iterbatch/model.py:77-109) field for
field and error for error, so plans built by either package are interchangeable (the drivers here
only read ``total_kernel_executions``, ``batch_size`` and ``num_batches``). The rest of the
reference's analytic model (Eqs. 1-6, model.py:37-75,112-269) is host arithmetic that consumes
this package's measurements unchanged and is not restated here.
"""

from __future__ import annotations

import operator
from dataclasses import dataclass

__all__ = ["BatchPlan", "feasible_batch_sizes"]


@dataclass(frozen=True)
class BatchPlan:
    """A factorization of the total kernel count into equal launch batches."""

    total_kernel_executions: int
    batch_size: int
    num_batches: int

    def __post_init__(self):
        for name in ("total_kernel_executions", "batch_size", "num_batches"):
            value = operator.index(getattr(self, name))
            if value < 1:
                raise ValueError(f"{name} must be a positive integer, got {value}")
            object.__setattr__(self, name, value)
        if self.batch_size * self.num_batches != self.total_kernel_executions:
            raise ValueError(
                f"batch_size ({self.batch_size}) * num_batches ({self.num_batches}) "
                f"!= total_kernel_executions ({self.total_kernel_executions})"
            )

    @classmethod
    def from_batch_size(cls, total_kernel_executions: int, batch_size: int) -> "BatchPlan":
        """Plan for a batch size that must divide the total kernel count (model.py:98-109)."""
        total = operator.index(total_kernel_executions)
        size = operator.index(batch_size)
        if total < 1 or size < 1:
            raise ValueError("total_kernel_executions and batch_size must be positive")
        num, rem = divmod(total, size)
        if rem:
            raise ValueError(f"batch size {size} does not divide total kernel count {total}")
        return cls(total, size, num)


def feasible_batch_sizes(total_kernel_executions: int) -> tuple[int, ...]:
    """All divisors of the kernel count, ascending (reference optimize.py:39-53)."""
    total = operator.index(total_kernel_executions)
    if total < 1:
        raise ValueError("total_kernel_executions must be >= 1")
    small: list[int] = []
    large: list[int] = []
    d = 1
    while d * d <= total:
        if total % d == 0:
            small.append(d)
            if d != total // d:
                large.append(total // d)
        d += 1
    return tuple(small + large[::-1])

"""paper_2501_09398_b200 — B200-native iteration-batched CUDA-Graph execution of solver kernels.

Drop-in for the hot path of arXiv 2501.09398 (Ekelund, Markidis, Peng: "Boosting Performance of
Iterative Applications on GPUs: Kernel Batching with CUDA Graphs"): the reference's solver API
``iterbatch.workloads`` (pkg/src/iterbatch/workloads.py) re-implemented over a C++/CUDA runtime
for sm_100a (``libiterbatch_b200.so``, C ABI in include/iterbatch_b200.h).

    from paper_2501_09398_b200 import workloads as wl
    state = wl.HotspotWorkload(T, P, 0.1)
    out = wl.run_batched(wl.hotspot_program(), state, batch_size=100, num_batches=100)

See DESIGN.md for the architecture and INTEGRATION.md for the reference-side binding.
"""

__version__ = "0.1.0"

from .model import BatchPlan, feasible_batch_sizes  # noqa: F401
from .fitting import MeasurementPoint, MeasurementSeries  # noqa: F401

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as fh:
        return json.load(fh)["kats"]


@pytest.fixture(scope="session")
def fixtures():
    with np.load(os.path.join(GOLDEN, "fixtures.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def gpu():
    """The runtime library on a visible CUDA device (tests marked gpu only)."""
    from paper_2501_09398_b200 import _lib

    _lib.lib()
    n = _lib.device_count()
    if n < 1:
        pytest.fail("no CUDA device visible for a -m gpu test (no CPU fallback exists)")
    return n


def spread(n: int) -> list:
    """Device list for n axis-0 slabs: distinct GPUs when the box has them (peer access, cross-
    device graph edges, NVLink halo stores), else all on GPU 0 — the same code path either way."""
    from paper_2501_09398_b200 import _lib

    count = max(1, _lib.device_count())
    return [g % count for g in range(n)]

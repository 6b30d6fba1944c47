"""Static checks of the shipped sm_100a SASS (CPU: cuobjdump on the built library, no GPU).

* Exactness: no fused multiply-add anywhere in the solver kernels (every numpy op is one
  correctly rounded __f*_rn / __d*_rn; an FFMA / FFMA2 / DFMA would round once where the
  reference rounds twice — kernels.cuh header). The only exception is IEEE division
  (the FDTD variants with cell size d != 1, template UNIT_D = false), whose correctly rounded
  __ddiv_rn / __fdiv_rn is itself an FMA-based Newton sequence.
* The design's hardware paths are really in the binary: every per-iteration solver kernel waits
  on the previous grid with griddepcontrol.wait (ACQBULK — PDL edges); the TMA hotspot kernel and
  the staged FDTD kernel stream through cp.async.bulk (UBLKCP) with mbarrier completion (SYNCS).
* No register spills (local-memory stack beyond a call frame) in the d == 1 kernels.
"""

import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2501_09398_b200", "libiterbatch_b200.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

pytestmark = pytest.mark.skipif(not (os.path.exists(LIB) and os.path.exists(CUOBJDUMP)),
                                reason="built library or cuobjdump not present")

SOLVER = re.compile(r"^_ZN2ib\d+(k_vector_f(32|64)|k_hotspot(_vec|_tma)?|k_fdtd_(lf|h2|e2))I")
DIVISION = re.compile(r"^_ZN2ib\d+k_fdtd_(lf|h2|e2)I[fd]Lb0E")  # UNIT_D = false: d != 1


@pytest.fixture(scope="module")
def sass():
    out = subprocess.run([CUOBJDUMP, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    parts = re.split(r"\n\s*Function : (\S+)\n", out)
    return {parts[i]: parts[i + 1] for i in range(1, len(parts) - 1, 2)}


@pytest.fixture(scope="module")
def usage():
    out = subprocess.run([CUOBJDUMP, "-res-usage", LIB], capture_output=True, text=True, check=True).stdout
    return {m.group(1): (int(m.group(2)), int(m.group(3)))
            for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", out)}


def _solvers(sass):
    names = [n for n in sass if SOLVER.match(n)]
    assert len(names) > 50, "solver kernels not found in the SASS"
    return names


def test_no_fused_multiply_add_outside_division(sass):
    bad = {}
    for name in _solvers(sass):
        if DIVISION.match(name):
            continue
        # (HFMA2 with zero operands is ptxas's move-immediate idiom, not arithmetic: the kernels
        # have no half-precision math, so it is not counted)
        n = len(re.findall(r"\b(FFMA2?|DFMA)\b", sass[name]))
        if n:
            bad[name] = n
    assert not bad, f"FMA contraction in exact kernels: {bad}"


def test_every_solver_kernel_waits_on_the_previous_grid(sass):
    missing = [n for n in _solvers(sass) if "ACQBULK" not in sass[n]]
    assert not missing, f"no griddepcontrol.wait (PDL) in {missing[:5]}"


def test_tma_kernels_use_bulk_copies_and_mbarriers(sass):
    names = [n for n in _solvers(sass) if re.match(r"^_ZN2ib\d+(k_hotspot_tma|k_fdtd_lf)I", n)]
    assert len(names) >= 20
    for n in names:
        assert "UBLKCP" in sass[n], n
        assert "SYNCS" in sass[n], n


def test_no_spills_in_unit_cell_kernels(usage):
    # <= 8 bytes is a call frame (a 64-bit division helper's return address), not a register spill
    spills = {n: s for n, (r, s) in usage.items() if SOLVER.match(n) and not DIVISION.match(n) and s > 8}
    assert not spills, f"local-memory stack in {spills}"

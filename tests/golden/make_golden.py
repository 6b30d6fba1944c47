"""Generate golden vectors for the hot path by running the REFERENCE itself.

Run in the build container only (the reference is not present on the GPU box):

    python tests/golden/make_golden.py [--long]

It imports the reference package read-only from /root/reference/pkg/src and writes
  tests/golden/kats.json       final-state checksums (the reference's state_checksum,
                               workloads.py:520-525) for run-workload configurations built by
                               the reference CLI's own generator (cli.py:172-199, seed 20240817)
  tests/golden/fixtures.npz    small input/output states (binary64) of the reference steps
Checksums are computed by the reference's own _fnv1a64 ("hash": "reference") except for states
above 64 MiB, where the pure-Python byte loop (~7 MB/s) is replaced by the C FNV-1a of
oracle/ib_oracle.c over the reference-computed arrays ("hash": "oracle-fnv"); that C hash is
itself checked against the reference's _fnv1a64 in tests/test_oracle.py.
"""

from __future__ import annotations

import argparse
import io
import json
import os
import sys
import time
from contextlib import redirect_stdout

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from iterbatch import cli as rcli  # noqa: E402
from iterbatch import workloads as rw  # noqa: E402

from oracle import cpu as ocpu  # noqa: E402

SHORT = [
    # (workload, size, iterations, batch_size)  — SURVEY.md App. B.4 plus edge shapes
    ("vector", "16384", 100, 10),
    ("vector", "16384", 10000, 100),
    ("vector", "1", 12, 4),
    ("vector", "3", 12, 3),
    ("vector", "5", 25, 5),
    ("vector", "7", 10, 2),
    ("vector", "1000", 60, 6),
    ("hotspot2d", "1024", 100, 10),
    ("hotspot2d", "64,48", 1000, 100),
    ("hotspot2d", "16,12", 12, 4),
    ("hotspot2d", "1", 10, 5),
    ("hotspot2d", "1,17", 9, 3),
    ("hotspot2d", "17,1", 9, 9),
    ("hotspot2d", "5,3", 15, 5),
    ("hotspot3d", "512,8", 10, 5),
    ("hotspot3d", "32,24,8", 200, 20),
    ("hotspot3d", "7,5,3", 13, 13),
    ("hotspot3d", "1,1,1", 4, 2),
    ("hotspot3d", "2,1,5", 6, 3),
    ("hotspot3d", "9,1,1", 5, 5),
    ("hotspot3d", "64,64,64", 20, 5),
    ("fdtd", "16,8,16", 120, 12),
    ("fdtd", "32", 50, 10),
    ("fdtd", "9,5,7", 300, 30),
    ("fdtd", "8,4,8", 6, 3),
    ("fdtd", "1,1,1", 5, 5),
    ("fdtd", "1,2,3", 7, 7),
    ("fdtd", "2,3,1", 4, 2),
]

LONG = [
    ("hotspot2d", "1024", 10000, 100),  # BASELINE config 2 at its full horizon (~4 min CPU)
    ("hotspot3d", "512,8", 1000, 100),  # BASELINE config 3 at its full horizon (~1.5 min)
    ("fdtd", "64", 2000, 100),          # long-horizon FDTD (~1 min)
    ("fdtd", "256", 20, 10),            # BASELINE config 4 grid, 20 steps (~1 min, 8 workers)
    ("hotspot3d", "256,256,64", 10, 5), # proxy for the 2048x2048x256 grid
]

HASH_LIMIT = 64 << 20


def reference_checksum(state) -> tuple[str, str]:
    nbytes = sum(a.size * 8 for a in state.state_arrays())
    if nbytes <= HASH_LIMIT:
        return f"{rw.state_checksum(state):016x}", "reference"
    return f"{ocpu.checksum(state.state_arrays()):016x}", "oracle-fnv"


def kat(workload, size, iterations, batch_size, workers):
    sizes = [int(s) for s in size.split(",")]
    t0 = time.perf_counter()
    state = rcli._build_workload(workload, sizes)
    program = rcli._PROGRAMS[workload]()
    plan = rcli.BatchPlan.from_batch_size(iterations, batch_size)
    final = rw.run_batched(program, state.copy(), plan.batch_size, plan.num_batches, workers)
    digest, how = reference_checksum(final)
    if how == "reference" and iterations <= 1000 and nbytes_small(final):
        # cross-check the batched checksum against the reference CLI in loop mode
        buf = io.StringIO()
        with redirect_stdout(buf):
            code = rcli.main(
                ["run-workload", "--workload", workload, "--size", size, "--iterations",
                 str(iterations), "--batch-size", str(batch_size), "--mode", "loop", "--checksum"]
            )
        assert code == 0 and buf.getvalue().strip() == digest, (workload, size, buf.getvalue())
    return {
        "workload": workload,
        "size": size,
        "iterations": iterations,
        "batch_size": batch_size,
        "checksum": digest,
        "hash": how,
        "seconds": round(time.perf_counter() - t0, 2),
    }


def nbytes_small(state) -> bool:
    return sum(a.size * 8 for a in state.state_arrays()) <= (4 << 20)


def fixtures() -> dict:
    out = {}
    rng = np.random.default_rng(3)
    v = rw.VectorWorkload(rng.random(1000), 0.9999)
    out["vector_in"] = v.values
    out["vector_out60"] = rw.run_loop(rw.vector_program(), v, 60).values
    rng = np.random.default_rng(7)
    h2 = rw.HotspotWorkload(rng.random((12, 9)), rng.random((12, 9)) * 1e-3, 0.2)
    out["hot2_T"], out["hot2_P"] = h2.temperature, h2.power
    out["hot2_out12"] = rw.run_loop(rw.hotspot_program(), h2, 12).temperature
    rng = np.random.default_rng(11)
    h3 = rw.HotspotWorkload(rng.random((6, 5, 4)), rng.random((6, 5, 4)) * 1e-3, 0.125)
    out["hot3_T"], out["hot3_P"] = h3.temperature, h3.power
    out["hot3_out5"] = rw.run_loop(rw.hotspot_program(), h3, 5).temperature
    f = rw.te101_cavity(8, 4, 8)
    for name, a in zip(("ex", "ey", "ez", "hx", "hy", "hz"), f.state_arrays()):
        out["fdtd_in_" + name] = a
    after_h = rw.fdtd_h_step(f)
    for name, a in zip(("hx", "hy", "hz"), after_h.state_arrays()[3:]):
        out["fdtd_h1_" + name] = a
    g = rw.run_loop(rw.fdtd_program(), f, 12)
    for name, a in zip(("ex", "ey", "ez", "hx", "hy", "hz"), g.state_arrays()):
        out["fdtd_out12_" + name] = a
    out["fdtd_scalars"] = np.array([f.cell_size, f.time_step])
    # unphysical dirty state: E step must ground every tangential wall component
    base = rw.fdtd_cavity(6, 5, 4)
    rng = np.random.default_rng(5)
    dirty = rw.FdtdWorkload(
        rng.random(base.ex.shape), rng.random(base.ey.shape), rng.random(base.ez.shape),
        rng.random(base.hx.shape), rng.random(base.hy.shape), rng.random(base.hz.shape),
        base.cell_size, base.time_step,
    )
    for name, a in zip(("ex", "ey", "ez", "hx", "hy", "hz"), dirty.state_arrays()):
        out["dirty_in_" + name] = a
    de = rw.run_loop(rw.fdtd_program(), dirty, 3)
    for name, a in zip(("ex", "ey", "ez", "hx", "hy", "hz"), de.state_arrays()):
        out["dirty_out3_" + name] = a
    out["dirty_scalars"] = np.array([base.cell_size, base.time_step])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--long", action="store_true", help="also run the full-horizon configs")
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    path = os.path.join(HERE, "kats.json")
    old = []
    if os.path.exists(path):
        with open(path) as fh:
            old = json.load(fh)["kats"]
    table = {(k["workload"], k["size"], k["iterations"], k["batch_size"]): k for k in old}
    for spec in SHORT + (LONG if args.long else []):
        if spec in table:
            continue
        entry = kat(*spec, workers=args.workers)
        table[spec] = entry
        print(json.dumps(entry), flush=True)
        with open(path, "w") as fh:
            json.dump({"generator": "tests/golden/make_golden.py", "reference": REF,
                       "seed": rcli._WORKLOAD_SEED, "kats": list(table.values())}, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "fixtures.npz"), **fixtures())
    print("fixtures written")


if __name__ == "__main__":
    main()

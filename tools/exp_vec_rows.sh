#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for R in 1 2 4; do
  for cfg in "hotspot3d 512,8 1000" "hotspot2d 1024 2000"; do
    set -- $cfg
    IB_HOTSPOT_VEC_ROWS=$R W=$1 S=$2 N=$3 K=50 python - <<'PY'
import os, sys, statistics
sys.path.insert(0, ".")
from paper_2501_09398_b200 import cli
from paper_2501_09398_b200 import workloads as wl
w, size, n, k = os.environ["W"], os.environ["S"], int(os.environ["N"]), int(os.environ["K"])
st = cli.build_workload(w, [int(x) for x in size.split(",")])
s = wl.DeviceSolver(st, "f32")
s.run_batched(k, n // k, pdl=True)
xs, ys = [], []
for _ in range(7):
    s.flush_l2(); s.upload(st)
    xs.append(s.run_batched(k, n // k, pdl=True).gpu_s)
    s.flush_l2(); s.upload(st)
    ys.append(s.run_stream(n).gpu_s)
print("R=" + os.environ["IB_HOTSPOT_VEC_ROWS"], w, size, f"graph {1e6*statistics.median(xs)/n:.3f} us/iter  stream {1e6*statistics.median(ys)/n:.3f}")
PY
  done
done

#!/bin/bash
# Kernel-variant experiment: graph-mode us/iter for forced variants (run under gpurun).
cd "${GRAFT_REPO_ROOT:-.}"
run() {  # label env... -- workload size iters K
  local label=$1; shift
  env "$@" python - <<'PY'
import os, sys, json, statistics
sys.path.insert(0, ".")
from paper_2501_09398_b200 import cli
from paper_2501_09398_b200 import workloads as wl
w, size, n, k = os.environ["W"], os.environ["S"], int(os.environ["N"]), int(os.environ["K"])
st = cli.build_workload(w, [int(x) for x in size.split(",")])
s = wl.DeviceSolver(st, "f32")
s.run_batched(k, n // k, pdl=True)
xs = []
for _ in range(5):
    s.flush_l2(); s.upload(st)
    xs.append(s.run_batched(k, n // k, pdl=True).gpu_s)
print(os.environ.get("LABEL"), w, size, f"{1e6*statistics.median(xs)/n:.3f} us/iter")
PY
}
for rpc in 2 4 8 16; do
  run x LABEL=tma_rpc$rpc IB_HOTSPOT_KERNEL=tma IB_HOTSPOT_RPC=$rpc W=hotspot3d S=512,8 N=1000 K=50
  run x LABEL=tma_rpc$rpc IB_HOTSPOT_KERNEL=tma IB_HOTSPOT_RPC=$rpc W=hotspot2d S=1024 N=2000 K=50
done
run x LABEL=vec IB_HOTSPOT_KERNEL=vec W=hotspot3d S=512,8 N=1000 K=50
run x LABEL=vec IB_HOTSPOT_KERNEL=vec W=hotspot2d S=1024 N=2000 K=50
for st in 3 6; do
  run x LABEL=tma_rpc4_st$st IB_HOTSPOT_KERNEL=tma IB_HOTSPOT_RPC=4 IB_TMA_STAGES=$st W=hotspot3d S=512,8 N=1000 K=50
done

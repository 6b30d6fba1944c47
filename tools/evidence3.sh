#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/evidence
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/evidence/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/evidence/pytest_gpu.log | tail -3; grep -E "^FAILED|Error" gpurun_out/evidence/pytest_gpu.log | head -5
trace() { timeout 600 python -m paper_2501_09398_b200 trace --workload $1 --size $2 --iterations $3 \
  --batch-size $4 --dtype f32 --out gpurun_out/evidence/trace_$5 > gpurun_out/evidence/trace_$5.json 2>&1; echo "trace $5 rc=$?"; }
trace vector 16384 10000 100 skeleton
trace hotspot2d 1024 10000 100 hotspot2d
trace hotspot3d 512,8 1000 100 hotspot3d
trace fdtd 256 2000 100 fdtd
python - <<'PY'
import sys, statistics, os; sys.path.insert(0, ".")
from paper_2501_09398_b200 import cli, workloads as wl
st = cli.build_workload("fdtd", [256])
for fuse, ppc in ((False, 0), (True, 0), (True, 32), (True, 64), (True, 129)):
    os.environ["IB_FDTD_PPC"] = str(ppc)
    s = wl.DeviceSolver(st, "f32", fuse=fuse)
    s.run_batched(50, 40, pdl=True)
    xs = []
    for _ in range(3):
        s.flush_l2(); s.upload(st); xs.append(s.run_batched(50, 40, pdl=True).gpu_s)
    it = s.iteration_bytes
    t = statistics.median(xs) / 2000
    print(f"fdtd fuse={fuse} ppc={ppc}: {1e6*t:.1f} us/iter, {it/t/1e9:.0f} GB/s of {it} B/iter", flush=True)
    s.close()
PY

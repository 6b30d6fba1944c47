#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/evidence
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/evidence/pytest_gpu.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/evidence/pytest_gpu.log | tail -3; grep -E "^FAILED" gpurun_out/evidence/pytest_gpu.log | head
trace() { timeout 600 python -m paper_2501_09398_b200 trace --workload $1 --size $2 --iterations $3 \
  --batch-size $4 --dtype f32 --out gpurun_out/evidence/trace_$5 > gpurun_out/evidence/trace_$5.json 2>&1; echo "trace $5 rc=$?"; }
trace vector 16384 10000 100 skeleton
trace hotspot2d 1024 10000 100 hotspot2d
trace hotspot3d 512,8 1000 100 hotspot3d
trace fdtd 256 2000 100 fdtd
san() {  # tool workload size dtype
  timeout 600 compute-sanitizer --tool $1 --error-exitcode 7 python tools/profile_run.py --workload $2 --size $3 --iters 4 --dtype $4 --graph 3 > gpurun_out/evidence/san_$1_$2_$4.log 2>&1; echo "sanitizer $1 $2 $4 rc=$?"; }
for tool in memcheck racecheck; do
  san $tool hotspot2d 64,48 f32; san $tool hotspot3d 24,20,8 f64; san $tool fdtd 9,5,7 f32; san $tool vector 1001 f32
  IB_HOTSPOT_KERNEL=tma san $tool hotspot3d 40,16,256 f32
done
IB_HOTSPOT_KERNEL=tma san synccheck hotspot3d 40,16,256 f32
for kv in 1 2; do IB_FDTD_PPC=$kv timeout 300 python -m paper_2501_09398_b200 sweep --workload fdtd --size 256 --iterations 2000 --batch-sizes 100 --repeats 3 --dtype f32 --pdl --out gpurun_out/evidence/fused_tmp > /dev/null 2>&1; done
python - <<'PY'
import sys, statistics; sys.path.insert(0, ".")
from paper_2501_09398_b200 import cli, workloads as wl
st = cli.build_workload("fdtd", [256])
for fuse in (False, True):
    s = wl.DeviceSolver(st, "f32", fuse=fuse)
    s.run_batched(50, 40, pdl=True)
    xs = []
    for _ in range(3):
        s.flush_l2(); s.upload(st); xs.append(s.run_batched(50, 40, pdl=True).gpu_s)
    it = s.iteration_bytes
    t = statistics.median(xs) / 2000
    print(f"fdtd fuse={fuse}: {1e6*t:.1f} us/iter, {it/t/1e9:.0f} GB/s of {it} B/iter")
    s.close()
PY

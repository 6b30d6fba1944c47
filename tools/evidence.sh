#!/bin/bash
# Round evidence (run under gpurun): tests, K sweeps + traces for the model fit, sanitizers.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/evidence
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/evidence/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/evidence/pytest_gpu.log
python __graft_entry__.py > gpurun_out/evidence/smoke.log 2>&1; echo "smoke rc=$?"
# K sweeps (paper Sec. III-C: creation / execution / stream per feasible K, 5 repeats)
sweep() { timeout 900 python -m paper_2501_09398_b200 sweep --workload $1 --size $2 --iterations $3 \
  --batch-sizes $4 --repeats 5 --dtype f32 $5 --out gpurun_out/evidence/sweep_$6 > gpurun_out/evidence/sweep_$6.log 2>&1; echo "sweep $6 rc=$?"; }
sweep vector 16384 10000 all "" skeleton
sweep vector 16384 10000 all "--pdl" skeleton_pdl
sweep hotspot2d 1024 10000 1,2,4,5,8,10,16,20,25,40,50,80,100,125,200,250,400,500,625,1000,1250,2000 "" hotspot2d
sweep hotspot3d 512,8 1000 all "" hotspot3d
sweep fdtd 256 2000 1,2,4,5,8,10,16,20,25,40,50,80,100,125,200,250,400,500 "" fdtd
sweep fdtd 256 2000 1,2,4,5,8,10,16,20,25,40,50,80,100,125,200,250,400,500 "--fuse" fdtd_fused
# real traces -> measured model constants (params file for `iterbatch optimize`)
trace() { timeout 600 python -m paper_2501_09398_b200 trace --workload $1 --size $2 --iterations $3 \
  --batch-size $4 --dtype f32 --out gpurun_out/evidence/trace_$5 > gpurun_out/evidence/trace_$5.json 2>&1; echo "trace $5 rc=$?"; }
trace vector 16384 10000 100 skeleton
trace hotspot2d 1024 10000 100 hotspot2d
trace hotspot3d 512,8 1000 100 hotspot3d
trace fdtd 256 2000 100 fdtd
timeout 600 python -m paper_2501_09398_b200 trace --workload fdtd --size 256 --iterations 2000 --batch-size 100 \
  --dtype f32 --fuse --out gpurun_out/evidence/trace_fdtd_fused > gpurun_out/evidence/trace_fdtd_fused.json 2>&1; echo "trace fdtd_fused rc=$?"
# sanitizers on small configs (every kernel variant)
san() {  # tool workload size dtype [extra profile_run args]
  timeout 600 compute-sanitizer --tool $1 --error-exitcode 7 python tools/profile_run.py --workload $2 --size $3 --iters 4 --dtype $4 --graph 3 $5 > gpurun_out/evidence/san_$1_$2_$4$5.log 2>&1; echo "sanitizer $1 $2 $4 $5 rc=$?"; }
for tool in memcheck racecheck; do
  san $tool hotspot2d 64,48 f32; san $tool hotspot3d 24,20,8 f64; san $tool fdtd 9,5,7 f32; san $tool vector 1001 f32
  san $tool fdtd 9,5,7 f32 --fuse; san $tool fdtd 20,17,40 f64 --fuse; IB_FDTD_KERNEL=lean san $tool fdtd 9,5,7 f32
  san $tool hotspot2d 40,128 f32; san $tool hotspot3d 24,16,8 f32; san $tool hotspot3d 24,16,8 f64  # shuffle paths
  IB_HOTSPOT_KERNEL=tma san $tool hotspot3d 40,16,256 f32
done
IB_HOTSPOT_KERNEL=tma san synccheck hotspot3d 40,16,256 f32
san synccheck fdtd 20,17,40 f32 --fuse; san synccheck fdtd 20,17,40 f32

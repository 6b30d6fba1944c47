#!/bin/bash
# The model-fit evidence (K sweeps + real traces) on the GPU box; then, in the build container:
#   python tools/model_fit.py gpurun_out/evidence --round r02
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/evidence
# K sweeps (paper Sec. III-C: creation / execution / stream per feasible K, 5 repeats)
sweep() { timeout 900 python -m paper_2501_09398_b200 sweep --workload $1 --size $2 --iterations $3 \
  --batch-sizes $4 --repeats 5 --dtype $5 $6 --out gpurun_out/evidence/sweep_$7 > gpurun_out/evidence/sweep_$7.log 2>&1; echo "sweep $7 rc=$?"; }
[ "${TRACE_ONLY:-0}" = 1 ] && sweep() { :; }
H=1,2,4,5,8,10,16,20,25,40,50,80,100,125,200,250,400,500,625,1000,1250,2000
F=1,2,4,5,8,10,16,20,25,40,50,80,100,125,200,250,400,500
sweep vector 16384 10000 all f32 "" skeleton
sweep hotspot2d 1024 10000 $H f64 "" hotspot2d_f64
sweep hotspot2d 1024 10000 $H f32 "" hotspot2d
sweep hotspot3d 512,8 1000 all f32 "" hotspot3d
sweep fdtd 256 2000 $F f32 "" fdtd
sweep fdtd 256 2000 $F f32 "--fuse" fdtd_fused
# real traces -> measured model constants (params file for `iterbatch optimize`)
trace() { timeout 600 python -m paper_2501_09398_b200 trace --workload $1 --size $2 --iterations $3 \
  --batch-size $4 --dtype $5 $6 --out gpurun_out/evidence/trace_$7 > gpurun_out/evidence/trace_$7.json 2>&1; echo "trace $7 rc=$?"; }
trace vector 16384 10000 100 f32 "" skeleton
trace hotspot2d 1024 10000 100 f64 "" hotspot2d_f64
trace hotspot2d 1024 10000 100 f32 "" hotspot2d
trace hotspot3d 512,8 1000 100 f32 "" hotspot3d
trace fdtd 256 2000 100 f32 "" fdtd
trace fdtd 256 2000 100 f32 "--fuse" fdtd_fused
# a small canned trace + sweep for the CPU round-trip test (tests/golden/b200_fit/)
trace hotspot2d 1024 200 20 f64 "" canned
sweep hotspot2d 1024 200 2,4,10,20,50 f64 "" canned

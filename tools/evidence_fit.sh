#!/bin/bash
# The model-fit evidence alone (K sweeps + real traces), without the tests / sanitizers of
# tools/evidence.sh; then, in the build container: python tools/model_fit.py gpurun_out/evidence --round r01
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/evidence
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

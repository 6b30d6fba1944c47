#!/bin/bash
# compute-sanitizer over every kernel variant the runtime can pick (small shapes), stream launches
# then a graph, plus axis-0 slabs on one device (halo stores / peer-copy nodes). Writes the logs
# and a summary table to gpurun_out/evidence/ (profiles/r01_sanitizers.md is that table).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/evidence
san() {  # tool workload size dtype [extra profile_run args]
  local tag; tag=$(echo "$5" | tr -d '-' | tr ' ' '_')
  timeout 600 compute-sanitizer --tool $1 --error-exitcode 7 python tools/profile_run.py --workload $2 \
    --size $3 --iters 4 --dtype $4 --graph 3 $5 > "gpurun_out/evidence/san_$1_$2_${3//,/x}_$4${tag:+_$tag}${KTAG:+_$KTAG}.log" 2>&1
  echo "sanitizer $1 $2 $3 $4 $5 $KTAG rc=$?"; }
for tool in memcheck racecheck; do
  san $tool vector 1001 f32
  san $tool hotspot2d 64,48 f32; san $tool hotspot2d 40,128 f32; san $tool hotspot3d 24,20,8 f64
  san $tool hotspot3d 24,16,8 f32; san $tool hotspot3d 24,16,8 f64  # warp-shuffle paths
  KTAG=tma IB_HOTSPOT_KERNEL=tma san $tool hotspot3d 40,16,256 f32
  KTAG=tma IB_HOTSPOT_KERNEL=tma san $tool hotspot3d 40,16,256 f64; san $tool hotspot3d 24,64,8 f64
  KTAG=scalar IB_HOTSPOT_KERNEL=scalar san $tool hotspot2d 40,128 f32
  san $tool fdtd 9,5,7 f32; san $tool fdtd 20,17,40 f64; KTAG=lean IB_FDTD_KERNEL=lean san $tool fdtd 9,5,7 f32
  KTAG=lean_scalar IB_FDTD_LEANV=0 IB_FDTD_KERNEL=lean san $tool fdtd 9,5,7 f32; KTAG=leanv IB_FDTD_LEANV=1 IB_FDTD_KERNEL=lean san $tool fdtd 20,17,40 f64
  san $tool fdtd 9,5,7 f32 --fuse; san $tool fdtd 20,17,40 f64 --fuse
  san $tool hotspot3d 30,16,8 f32 "--slabs 3"; san $tool hotspot2d 41,128 f64 "--slabs 2 --halo copy"
  KTAG=tma IB_HOTSPOT_KERNEL=tma san $tool hotspot3d 40,16,256 f32 "--slabs 2"
  san $tool fdtd 20,17,40 f32 "--slabs 3"; san $tool fdtd 20,17,40 f64 "--slabs 3 --fuse"
  san $tool fdtd 20,17,40 f32 "--slabs 2 --halo copy"; san $tool fdtd 20,17,40 f32 "--slabs 2 --fuse --halo copy"
done
san synccheck hotspot2d 40,128 f32; san synccheck fdtd 20,17,40 f32 --fuse; san synccheck fdtd 20,17,40 f32
KTAG=tma IB_HOTSPOT_KERNEL=tma san synccheck hotspot3d 40,16,256 f32
KTAG=tma IB_HOTSPOT_KERNEL=tma san synccheck hotspot3d 40,16,256 f64; san synccheck fdtd 20,17,40 f64 --fuse
{
  echo "| run (tool_workload_size_dtype[_flags][_kernel]) | summary |"
  echo "|---|---|"
  for f in gpurun_out/evidence/san_*.log; do
    n=$(basename "$f" .log); n=${n#san_}
    echo "| $n | $(grep -hE "ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK SUMMARY" "$f" | tail -1) |"
  done
} > gpurun_out/evidence/sanitizers.md
cat gpurun_out/evidence/sanitizers.md

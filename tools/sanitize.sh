cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/evidence
san() {
  timeout 600 compute-sanitizer --tool $1 --error-exitcode 7 python tools/profile_run.py --workload $2 --size $3 --iters 4 --dtype $4 --graph 3 $5 > gpurun_out/evidence/san_$1_$2_$4$5.log 2>&1; echo "sanitizer $1 $2 $3 $4 $5 rc=$?"; }
for tool in memcheck racecheck; do
  san $tool hotspot2d 40,128 f32; san $tool hotspot3d 24,16,8 f32; san $tool hotspot3d 24,16,8 f64
  san $tool fdtd 20,17,40 f64; san $tool fdtd 20,17,40 f64 --fuse
done
san synccheck hotspot2d 40,128 f32

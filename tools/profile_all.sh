#!/bin/bash
# ncu evidence for the committed kernels (run under gpurun; one GPU; never multi-rank).
# Writes gpurun_out/ncu_<name>_raw.csv (every metric of the --set full capture; the .ncu-rep is
# kept only with KEEP_REPS=1) and gpurun_out/launches_bench.csv.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
full() {  # name regex skip -- profile_run.py args
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s "$skip" -c 2 \
    -o "gpurun_out/ncu_$name" python tools/profile_run.py "$@" > "gpurun_out/ncu_$name.log" 2>&1
  echo "ncu full $name rc=$?"
  # keep gpurun_out small enough to come back (64 MiB): every raw metric as CSV, the report only
  # with KEEP_REPS=1
  ncu -i "gpurun_out/ncu_$name.ncu-rep" --page raw --csv > "gpurun_out/ncu_${name}_raw.csv" 2>/dev/null
  [ "${KEEP_REPS:-0}" = 1 ] || rm -f "gpurun_out/ncu_$name.ncu-rep"
}
for dt in f64 f32; do
  full hotspot2d_$dt k_hotspot 2 --workload hotspot2d --size 1024 --iters 4 --dtype $dt
  full hotspot3d_512_$dt k_hotspot 2 --workload hotspot3d --size 512,8 --iters 4 --dtype $dt
  full hotspot3d_large_$dt k_hotspot 2 --workload hotspot3d --size 2048,2048,256 --iters 4 --dtype $dt
  full fdtd_$dt k_fdtd 2 --workload fdtd --size 256 --iters 3 --dtype $dt
  full fdtd_fused_$dt k_fdtd_lf 2 --workload fdtd --size 256 --iters 4 --fuse --dtype $dt
  full skeleton_$dt k_vector 2 --workload vector --size 16384 --iters 4 --dtype $dt
done
# launch list of a short bench run (cold-cache, serialised; compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --quick \
  --cpu-budget 1 --no-extra > gpurun_out/launches_bench.log 2>&1
echo "ncu launches rc=$?"

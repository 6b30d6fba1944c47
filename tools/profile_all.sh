#!/bin/bash
# ncu evidence for the committed kernels (run under gpurun; one GPU; never multi-rank).
# Writes gpurun_out/ncu_<name>.ncu-rep (--set full) and gpurun_out/launches_<name>.csv.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
full() {  # name workload size regex
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$4" -s 2 -c 2 \
    -o "gpurun_out/ncu_$1" python tools/profile_run.py --workload "$2" --size "$3" --iters 3 \
    > "gpurun_out/ncu_$1.log" 2>&1
  echo "ncu full $1 rc=$?"
}
full hotspot2d hotspot2d 1024 k_hotspot
full hotspot3d_512 hotspot3d 512,8 k_hotspot
full hotspot3d_large hotspot3d 2048,2048,256 k_hotspot
full fdtd fdtd 256 k_fdtd
full skeleton vector 16384 k_vector
# launch list of a short bench run (cold-cache, serialised; compare shares, not absolutes)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --quick \
  --cpu-budget 1 --no-extra > gpurun_out/launches_bench.log 2>&1
echo "ncu launches rc=$?"

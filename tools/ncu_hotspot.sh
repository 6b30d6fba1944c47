cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/hs
timeout 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_hotspot -s 5 -c 2 -o gpurun_out/hs/h3 python tools/profile_run.py --workload hotspot3d --size 512,8 --iters 10 > gpurun_out/hs/h3.log 2>&1; echo "rc=$?"
timeout 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_hotspot -s 5 -c 2 -o gpurun_out/hs/h2 python tools/profile_run.py --workload hotspot2d --size 1024 --iters 10 > gpurun_out/hs/h2.log 2>&1; echo "rc=$?"

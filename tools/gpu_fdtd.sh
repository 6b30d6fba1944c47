cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r7
timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -q -m gpu -x -k fused -p no:cacheprovider > gpurun_out/r7/fused.log 2>&1; echo "fused rc=$?"; tail -15 gpurun_out/r7/fused.log
timeout 600 python tools/fdtd_tune.py > gpurun_out/r7/tune.log 2>&1; echo "tune rc=$?"; cat gpurun_out/r7/tune.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fdtd_lf -s 2 -c 1 -o gpurun_out/r7/lf python tools/profile_run.py --workload fdtd --size 256 --iters 3 --fuse > gpurun_out/r7/lf.log 2>&1; echo "ncu rc=$?"

cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/fd
timeout 900 python -m pytest tests/ -q -m gpu -x -k "fdtd or fused or smoke or parity" -p no:cacheprovider > gpurun_out/fd/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fd/tests.log; grep -E "^(FAILED|E  )" gpurun_out/fd/tests.log | head
timeout 600 python tools/fdtd_tune.py > gpurun_out/fd/tune.log 2>&1; echo "tune rc=$?"; cat gpurun_out/fd/tune.log

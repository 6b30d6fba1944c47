cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/suite
timeout 600 python -m pytest tests/test_gpu_physics.py -q -m gpu -p no:cacheprovider > gpurun_out/suite/physics.log 2>&1
echo "physics rc=$?"; tail -3 gpurun_out/suite/physics.log; grep "^E  " gpurun_out/suite/physics.log | head -5
timeout 600 python -m pytest tests/test_gpu_physics.py -q -m gpu -p no:cacheprovider -k trace > gpurun_out/suite/trace.log 2>&1
echo "trace only rc=$?"; tail -3 gpurun_out/suite/trace.log; grep "^E  " gpurun_out/suite/trace.log | head -5

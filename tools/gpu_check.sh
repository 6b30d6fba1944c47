#!/bin/bash
# One gpurun call: GPU parity tests, smoke(), the default bench line and the reference arm.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/check
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/check/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/check/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/check/pytest_gpu.log; grep -E "^FAILED" gpurun_out/check/pytest_gpu.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check/smoke.log 2>&1
echo "smoke rc=$?"; tail -5 gpurun_out/check/smoke.log
timeout 900 python bench.py > gpurun_out/check/bench.json 2> gpurun_out/check/bench.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/check/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/check/bench_ref.json 2> gpurun_out/check/bench_ref.err
echo "ref rc=$?"; cat gpurun_out/check/bench_ref.json

cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k "fused" -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/fdtd_tune.py

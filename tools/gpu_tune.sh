cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k "hotspot or fdtd" -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/hotspot_tune.py
timeout 600 python tools/fdtd_tune.py
timeout 300 python -m paper_2501_09398_b200 trace --workload hotspot2d --size 1024 --iterations 10000 --batch-size 100 --dtype f32 --out /tmp/tr 2>&1 | tail -1

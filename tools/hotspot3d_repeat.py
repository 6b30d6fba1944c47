"""Hotspot3D 512^2x8 vectorised-kernel CTA shapes in interleaved repeats (diagnostic): R = 4 in
128 x 8 CTAs against the alternatives, binary32, graph us/iter.
    python tools/hotspot3d_repeat.py"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl
st = cli.build_workload("hotspot3d", [512, 8])
cfgs = {"default": {}, "R4 128x8": {"IB_HOTSPOT_VEC_ROWS": "4", "IB_HOTSPOT_BX": "128", "IB_HOTSPOT_BLOCK": "1024"},
        "R4 256x4": {"IB_HOTSPOT_VEC_ROWS": "4", "IB_HOTSPOT_BX": "256", "IB_HOTSPOT_BLOCK": "1024"},
        "R2 64x4": {"IB_HOTSPOT_VEC_ROWS": "2", "IB_HOTSPOT_BX": "64", "IB_HOTSPOT_BLOCK": "256"},
        "R4 256x2": {"IB_HOTSPOT_VEC_ROWS": "4", "IB_HOTSPOT_BX": "256", "IB_HOTSPOT_BLOCK": "512"}}
res = {k: [] for k in cfgs}
for rep in range(4):
    for name, env in cfgs.items():
        for k in ("IB_HOTSPOT_VEC_ROWS", "IB_HOTSPOT_BX", "IB_HOTSPOT_BLOCK"):
            os.environ.pop(k, None)
        os.environ.update(env)
        s = wl.DeviceSolver(st, "f32")
        s.run_batched(40, 25, pdl=True)
        for _ in range(3):
            s.flush_l2(); s.upload(st)
            res[name].append(s.run_batched(40, 25, pdl=True).gpu_s / 1000)
        s.close()
for name, v in res.items():
    print(f"{name:10s} median {1e6*statistics.median(v):.3f}  min {1e6*min(v):.3f}  max {1e6*max(v):.3f}")

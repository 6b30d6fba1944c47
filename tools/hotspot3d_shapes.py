"""Hotspot3D vectorised-kernel defaults vs the previous ones (R=2, 256 x 1 CTAs) over L2-resident
shapes (diagnostic): graph + PDL, interleaved repeats, median."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import workloads as wl
import numpy as np

OLD = {"IB_HOTSPOT_VEC_ROWS": "2", "IB_HOTSPOT_BX": "256", "IB_HOTSPOT_BLOCK": "256"}
rng = np.random.default_rng(3)
for shape in ((512, 512, 8), (256, 256, 32), (384, 384, 16), (128, 128, 64), (768, 512, 8), (1024, 256, 16), (576, 512, 8), (640, 384, 8),
              (256, 512, 8), (64, 64, 8)):
    t = rng.random(shape)
    st = wl.HotspotWorkload(t, t * 1e-3, 0.1)
    res = {"new": [], "old": []}
    for rep in range(3):
        for name in ("new", "old"):
            for k in OLD:
                os.environ.pop(k, None)
            if name == "old":
                os.environ.update(OLD)
            s = wl.DeviceSolver(st, "f32")
            s.run_batched(40, 10, pdl=True)
            for _ in range(3):
                s.flush_l2(); s.upload(st)
                res[name].append(s.run_batched(40, 10, pdl=True).gpu_s / 400)
            if name == "new":
                d = s.describe()[0]
            s.close()
    print(f"{'x'.join(map(str, shape)):14s} new {1e6*statistics.median(res['new']):7.3f}  old {1e6*statistics.median(res['old']):7.3f}  "
          f"({d['kernel'][:34]} grid {d['grid'][:2]} block {d['block'][:2]})", flush=True)

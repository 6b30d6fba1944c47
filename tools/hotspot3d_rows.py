import os, sys, statistics
sys.path.insert(0, '/root/repo')
from paper_2501_09398_b200 import workloads as wl
import numpy as np
rng = np.random.default_rng(5)
for shape in ((768, 512, 8), (1024, 256, 16), (640, 384, 8), (896, 512, 8), (512, 1024, 16)):
    t = rng.random(shape); st = wl.HotspotWorkload(t, t * 1e-3, 0.1)
    out = []
    for name, env in (("default", {}), ("R1 256", {"IB_HOTSPOT_VEC_ROWS": "1"}), ("R1 512", {"IB_HOTSPOT_VEC_ROWS": "1", "IB_HOTSPOT_BLOCK": "512"}),
                      ("R4 256", {"IB_HOTSPOT_VEC_ROWS": "4"})):
        for k in ("IB_HOTSPOT_VEC_ROWS", "IB_HOTSPOT_BLOCK"): os.environ.pop(k, None)
        os.environ.update(env)
        s = wl.DeviceSolver(st, "f32")
        s.run_batched(50, 4, pdl=True)
        g = []
        for _ in range(5):
            s.flush_l2(); s.upload(st)
            g.append(s.run_batched(50, 4, pdl=True).gpu_s / 200)
        s.close()
        out.append(f"{name} {1e6*statistics.median(g):6.2f}")
    print("x".join(map(str, shape)), " | ".join(out), flush=True)

import os, sys, statistics
sys.path.insert(0, os.getcwd())
from paper_2501_09398_b200 import cli, workloads as wl
import json
cases = json.loads(os.environ.get("CASES", "null")) or [
    ("hotspot2d", [1024], 2000, [(2, 256), (2, 512), (1, 512)]),
    ("hotspot3d", [512, 8], 1000, [(2, 128), (2, 256), (4, 512), (4, 256)])]
cases = [(w, size, n, [tuple(v) for v in vs]) for w, size, n, vs in cases]
for w, size, n, vs in cases:
    st = cli.build_workload(w, size)
    res = {v: [] for v in vs}
    for rep in range(4):
        for (r, bs) in vs:
            os.environ.update(IB_HOTSPOT_KERNEL="vec", IB_HOTSPOT_VEC_ROWS=str(r), IB_HOTSPOT_SHUFFLE="1",
                              IB_HOTSPOT_BLOCK=str(bs))
            s = wl.DeviceSolver(st, "f32")
            s.run_batched(50, n // 50, pdl=True)
            xs = []
            for _ in range(5):
                s.flush_l2(); s.upload(st)
                xs.append(s.run_batched(50, n // 50, pdl=os.environ.get("PDL", "1") == "1").gpu_s / n)
            res[(r, bs)].append(1e6 * statistics.median(xs))
            s.close()
    for v, xs in res.items():
        print(w, v, " ".join(f"{x:.3f}" for x in xs), "median", round(statistics.median(xs), 3), flush=True)

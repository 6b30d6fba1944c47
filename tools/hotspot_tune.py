"""Hotspot launch-bound configs: graph-mode (PDL, K=50) and stream us/iter per kernel variant."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

KEYS = ("IB_HOTSPOT_KERNEL", "IB_HOTSPOT_VEC_ROWS", "IB_HOTSPOT_RPC", "IB_TMA_STAGES", "IB_HOTSPOT_BLOCK",
        "IB_VECTOR_BLOCK", "IB_HOTSPOT_SHUFFLE")
cfgs = [("hotspot3d", [512, 8], 1000), ("hotspot2d", [1024], 2000)]
if os.environ.get("CFGS"):  # e.g. CFGS=hotspot2d
    cfgs = [c for c in cfgs if c[0] in os.environ["CFGS"].split(",")]
DTYPE = os.environ.get("DTYPE", "f32")
variants = [("auto", {})]
for r in (1, 2, 4):
    for bs in (128, 256, 512, 1024):
        variants.append((f"vec R={r} sh=1 block={bs}", {"IB_HOTSPOT_KERNEL": "vec", "IB_HOTSPOT_VEC_ROWS": r,
                                                        "IB_HOTSPOT_SHUFFLE": 1, "IB_HOTSPOT_BLOCK": bs}))

if os.environ.get("ALL"):
    for rpc in (2, 4, 8, 16):
        variants.append((f"tma rpc={rpc}", {"IB_HOTSPOT_KERNEL": "tma", "IB_HOTSPOT_RPC": rpc}))
    for rpc in (2, 4, 8):
        variants.append((f"scalar rpc={rpc}", {"IB_HOTSPOT_KERNEL": "scalar", "IB_HOTSPOT_RPC": rpc}))
if os.environ.get("AUTO_ONLY"):
    variants = variants[:1]
vec_variants = [(f"block={bs}", {"IB_VECTOR_BLOCK": bs}) for bs in (128, 256, 512, 1024)]
for w, size, n in cfgs:
    st = cli.build_workload(w, size)
    for name, env in (vec_variants if w == "vector" else variants):
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update({k: str(v) for k, v in env.items()})
        s = wl.DeviceSolver(st, DTYPE)
        s.run_batched(50, n // 50, pdl=True)
        g, gp, sp = [], [], []
        for _ in range(5):
            s.flush_l2(); s.upload(st)
            g.append(s.run_batched(50, n // 50, pdl=False).gpu_s / n)
            s.flush_l2(); s.upload(st)
            gp.append(s.run_batched(50, n // 50, pdl=True).gpu_s / n)
            s.flush_l2(); s.upload(st)
            sp.append(s.run_stream(n).gpu_s / n)
        m = lambda x: 1e6 * statistics.median(x)
        print(f"{DTYPE} {w:9s} {name:24s} graph {m(g):6.3f}  graph+pdl {m(gp):6.3f}  stream {m(sp):6.3f}  "
              f"ratio {statistics.median(sp)/min(statistics.median(g), statistics.median(gp)):.3f}", flush=True)
        s.close()

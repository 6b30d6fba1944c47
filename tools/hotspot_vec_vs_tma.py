"""Vectorised vs TMA hotspot kernel around the L2 size (diagnostic): auto / vec / tma per shape,
binary32, graph us/iter — the 104 MB crossover in hotspot_variant.
    python tools/hotspot_vec_vs_tma.py [shape ...]   # shapes as N or R,C,L"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl
for size in ([int(x) for x in a.split(",")] for a in sys.argv[1:]) if sys.argv[1:] else ([1024, 8], [768, 8], [1024, 1024, 12], [1536, 1024, 8], [1024], [2048], [3072], [4096]):
    w = "hotspot3d" if len(size) != 1 else "hotspot2d"
    st = cli.build_workload(w, size)
    row = []
    for kern in ("auto", "vec", "tma"):
        os.environ.pop("IB_HOTSPOT_KERNEL", None)
        if kern != "auto": os.environ["IB_HOTSPOT_KERNEL"] = kern
        s = wl.DeviceSolver(st, "f32")
        s.run_batched(20, 5, pdl=True)
        g = []
        for pdl in (False, True):
            for _ in range(3):
                s.flush_l2()
                g.append(s.run_batched(20, 5, pdl=pdl).gpu_s / 100)
        d = s.describe()[0]["kernel"][12:24]
        s.close()
        row.append(f"{kern}:{1e6*min(g):8.2f} ({d})")
    print(w, size, "  ".join(row), flush=True)

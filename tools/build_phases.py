"""Graph build phases (create / instantiate / upload, us) per batch size over three rounds of the
bench's own sweep order (build + run + destroy), to tell one-time costs and host hiccups from
per-build costs (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl

st = cli.build_workload("hotspot2d", [1024])
s = wl.DeviceSolver(st, "f32")
n = 10000
for rnd in range(3):
    for k in (10, 20, 25, 40, 50, 80, 100, 125, 200, 250, 400, 500, 1000, 2000):
        for pdl in (False, True):
            t = s.build_graph(k, pdl=pdl)
            r = s.run_graph(n // k)
            s.destroy_graph()
            print(f"round {rnd} K={k:4d} pdl={int(pdl)} create {1e6*t.create_s:8.1f} instantiate {1e6*t.instantiate_s:8.1f} "
                  f"upload {1e6*t.upload_s:8.1f} total {1e6*t.build_s:8.1f} nodes {t.nodes} exec_us/iter {1e6*r.gpu_s/n:6.3f}",
                  flush=True)

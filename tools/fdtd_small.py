import os, sys, statistics
sys.path.insert(0, os.getcwd())
from paper_2501_09398_b200 import cli, workloads as wl
for n in (16, 32, 48, 64, 96, 128, 160):
    st = cli.build_workload("fdtd", [n])
    res = []
    for kern in ("staged", "lean"):
        os.environ["IB_FDTD_KERNEL"] = kern
        s = wl.DeviceSolver(st, "f32")
        s.run_batched(10, 5, pdl=True)
        best = None
        for pdl in (False, True):
            xs = []
            for _ in range(3):
                s.flush_l2()
                xs.append(s.run_batched(20, 10, pdl=pdl).gpu_s / 200)
            t = statistics.median(xs)
            best = t if best is None else min(best, t)
        res.append(1e6 * best)
        s.close()
    print(f"fdtd {n}^3: staged {res[0]:.2f} us/iter  lean {res[1]:.2f}", flush=True)

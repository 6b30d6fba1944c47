"""A/B of two runtime builds on FDTD 256^3 (diagnostic): run once per library (IB_LIB_PATH), two
half-steps and fused, graph at K=20 with plain and programmatic (PDL) edges, device us/iter, median
of 5; the SM clock and board power are sampled (NVML, 20 ms) while the runs execute, because an
issue-bound kernel's time follows the clock and sw_power_cap moves it.
  python tools/ab_fdtd.py ; IB_LIB_PATH=ab/lib_old.so DTYPE=f64 N=2000 python tools/ab_fdtd.py"""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

tag = os.environ.get("IB_LIB_PATH", "in-tree")
n = int(os.environ.get("N", "200"))
dtype = os.environ.get("DTYPE", "f32")
st = cli.build_workload("fdtd", [int(os.environ.get("SIZE", "256"))])


class Sampler:
    def __init__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
            self.nv = pynvml
        except Exception:  # noqa: BLE001
            self.nv = None
        self.clk, self.pw, self.stop = [], [], False

    def __enter__(self):
        self.clk, self.pw, self.stop = [], [], False
        if self.nv:
            self.t = threading.Thread(target=self.loop, daemon=True)
            self.t.start()
        return self

    def loop(self):
        while not self.stop:
            self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000)
            time.sleep(0.02)

    def __exit__(self, *a):
        self.stop = True
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.clk:
            return "clk n/a"
        return f"sm {statistics.median(self.clk):.0f} MHz (min {min(self.clk)}) power {statistics.median(self.pw):.0f} W"


smp = Sampler()
for fuse in (False, True):
    s = wl.DeviceSolver(st, dtype, fuse=fuse)
    s.run_batched(20, n // 20)
    for pdl in (False, True):
        g = []
        with smp:
            for _ in range(5):
                s.flush_l2()
                g.append(s.run_batched(20, n // 20, pdl=pdl).gpu_s / n)
        print(f"{tag:24s} {dtype} {'fused' if fuse else 'H+E  '} {'pdl  ' if pdl else 'plain'} "
              f"{1e6 * statistics.median(g):8.2f} us/iter  {smp.summary()}", flush=True)
    s.close()

"""Where the headline's end-to-end time goes (diagnostic): 20 drop-in calls
workloads.run_batched(hotspot_program(), HotspotWorkload(binary64 1024^2), K=100, I=100) with the
host wall clock of each call, then the same steps timed one by one (pageable H2D of T and P,
graph build + launches, D2H of T, the result dataclass).
    python tools/e2e_breakdown.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli, workloads as wl  # noqa: E402

dtype = os.environ.get("DTYPE", "f64")
st = cli.build_workload("hotspot2d", [1024])
prog = wl.hotspot_program()
k, num, n = 100, 100, 10000
calls = []
for _ in range(23):
    t0 = time.perf_counter()
    wl.run_batched(prog, st, k, num, dtype=dtype, pdl=True)
    calls.append(time.perf_counter() - t0)
calls = calls[3:]
print(f"drop-in call: median {1e6 * statistics.median(calls) / n:.3f} us/iter, mean "
      f"{1e6 * statistics.fmean(calls) / n:.3f}, min {1e6 * min(calls) / n:.3f}, max {1e6 * max(calls) / n:.3f}")
parts = {"upload (pageable H2D, T and P)": [], "build + launches + wait": [], "download T (pageable D2H)": [],
         "result dataclass": []}
with wl.DeviceSolver(st, dtype) as s:
    for _ in range(13):
        t0 = time.perf_counter()
        s.upload(st)
        t1 = time.perf_counter()
        s.build_graph(k, pdl=True)
        s.run_graph(num)
        s.destroy_graph()
        t2 = time.perf_counter()
        a = s.download_field(0)
        t3 = time.perf_counter()
        wl.HotspotWorkload(a, st.power, st.diffusion_coefficient)
        t4 = time.perf_counter()
        for key, v in zip(parts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
            parts[key].append(v)
for key, v in parts.items():
    print(f"{key:34s} median {1e3 * statistics.median(v[3:]):8.3f} ms  max {1e3 * max(v[3:]):8.3f} ms")

"""Does sampling nvidia-smi during a timed region perturb short graph runs? (diagnostic)"""
import os, statistics, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_09398_b200 import cli
from paper_2501_09398_b200 import workloads as wl

def run(s, label, n=10):
    xs = []
    for _ in range(n):
        s.flush_l2()
        xs.append(s.run_batched(100, 100, pdl=True).gpu_s)
    print(f"{label:40s} {1e6*statistics.fmean(xs)/10000:.3f} us/iter  (min {1e6*min(xs)/10000:.3f}, max {1e6*max(xs)/10000:.3f})", flush=True)

st = cli.build_workload("hotspot2d", [1024])
s = wl.DeviceSolver(st, "f32")
run(s, "warm")
run(s, "plain")
for ms in (100, 500):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap", "--format=csv,noheader", "-lms", str(ms)], stdout=subprocess.DEVNULL)
    time.sleep(0.3)
    run(s, f"nvidia-smi -lms {ms} (full query)")
    p.terminate(); p.wait()
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"], stdout=subprocess.DEVNULL)
time.sleep(0.3); run(s, "nvidia-smi -lms 100 (clocks.sm only)"); p.terminate(); p.wait()
try:
    import pynvml, threading
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    stop = False; samples = []
    def loop():
        while not stop:
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            time.sleep(0.1)
    th = threading.Thread(target=loop); th.start()
    run(s, "pynvml clocks+reasons @100ms")
    stop = True; th.join()
    print("pynvml samples", samples[:5])
except Exception as e:
    print("pynvml failed", e)
run(s, "plain again")

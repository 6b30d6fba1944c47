"""Render gpurun_out/graph_modes.json (tools/graph_modes.py) as profiles/<round>_graph_modes.md."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for dt in ("f64", "f32"):
    path = os.path.join(ROOT, "gpurun_out", f"graph_modes_{dt}.json")
    if os.path.exists(path):
        rows += [dict(r, config=f"{r['config']} {dt}") for r in json.load(open(path))]
cfgs, modes = [], []
for r in rows:
    if r["config"] not in cfgs:
        cfgs.append(r["config"])
    if r["mode"] not in modes:
        modes.append(r["mode"])
out = [f"# Graph-mode variants on one B200 ({rnd})", "",
       "`python tools/graph_modes.py` under gpurun (DTYPE=f64 and f32): device time (CUDA events) per iteration, "
       "L2 flushed before every run, median of 5 runs; T_C = host build time (create + instantiate + "
       "upload), µs. `stream` is Listing 1 (the paper's baseline); `manual` / `capture` are Listing 3 "
       "built with explicit nodes or stream capture; `+pdl` adds programmatic dependent-launch edges "
       "(launch attribute in stream mode); `device-launch` instantiates with "
       "`cudaGraphInstantiateFlagDeviceLaunch` as the paper; `while` wraps the K-chain in a conditional "
       "WHILE node so ONE host launch runs every batch; `peeled N+7` runs N+7 iterations (not divisible "
       "by K) as floor(N/K) replays plus a remainder graph; `odd K=25 baked / patched` runs an odd batch "
       "on the ping-pong solvers with two executables (buffer parity baked in) or one executable "
       "re-pointed by `cudaGraphExecKernelNodeSetParams` (`IB_FLAG_PATCH`).", "",
       "| config | K | " + " | ".join(modes) + " |", "|---|---|" + "---|" * len(modes)]
for c in cfgs:
    rr = {r["mode"]: r for r in rows if r["config"] == c}
    k = next(iter(rr.values()))["K"]
    out.append(f"| {c} | {k} | " + " | ".join(f"{rr[m]['us_per_iter']:.3f}" for m in modes) + " |")
gm = [m for m in modes if not m.startswith("stream")]
out += ["", "T_C (µs) of the graph modes:", "", "| config | " + " | ".join(gm) + " |", "|---|" + "---|" * len(gm)]
for c in cfgs:
    rr = {r["mode"]: r for r in rows if r["config"] == c}
    out.append(f"| {c} | " + " | ".join(f"{rr[m]['T_C_us']:.0f}" for m in gm) + " |")
out += ["", "Reading:", "",
        "* Batching into a graph removes the host launch cost; programmatic edges then overlap each "
        "kernel's launch with its predecessor's tail.",
        "* PDL in plain stream mode recovers part of the gap, which makes the graph's advantage on a "
        "~4 µs kernel small once both use it; the bench reports both stream numbers.",
        "* FDTD: the staged kernels hold one CTA per SM (206 KB ring), so an early-launched successor "
        "cannot co-reside; the bench's K/PDL sweep picks whichever edge type is faster.",
        "* The WHILE node and device-launch instantiation cost slightly more T_C and a few percent per "
        "iteration; loop peeling costs one extra graph build (the remainder graph); re-pointing one "
        "executable for odd K halves T_C at an unchanged per-iteration time (the host patches while "
        "the previous batch runs).", ""]
open(os.path.join(ROOT, "profiles", f"{rnd}_graph_modes.md"), "w").write("\n".join(out))
print("\n".join(out[6:12]))

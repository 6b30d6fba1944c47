"""SASS evidence for the shipped kernels (run in the build container): per kernel of the built
library, the count of the instructions that prove the design — UBLKCP (cp.async.bulk, the TMA
engine), SYNCS (mbarrier), ACQBULK / PREEXIT (griddepcontrol.wait / launch_dependents, PDL),
SHFL (warp shuffles), LDG/STG.E.128 (16-byte global accesses), LDS/STS (shared memory), MEMBAR
(the cross-process fence), FMA/FFMA (must be 0: every op is a correctly rounded __f*_rn) — and
the register / stack use.
    python tools/sass_evidence.py > profiles/r01_sass_evidence.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2501_09398_b200", "libiterbatch_b200.so")
KEYS = ["UBLKCP", "SYNCS", "ACQBULK", "PREEXIT", "SHFL", "LDG.E.128", "STG.E.128", "LDS", "STS",
        "MEMBAR", "FFMA", "DFMA", "FMUL", "DMUL"]
# the kernels the bench configs run (f32) and their f64 twins
WANT = [r"k_vector_f32ILb0E", r"k_hotspot_vecIfLb0ELi2ELi1ELb0E", r"k_hotspot_vecIfLb1ELi4ELi1ELb0E",
        r"k_hotspot_vecIfLb1ELi2ELi1ELb1E", r"k_hotspot_tmaIfLb1ELi2E", r"k_fdtd_lfIfLb1ELi4ELi1ELb0E",
        r"k_fdtd_lfIfLb1ELi4ELi2ELb0E", r"k_fdtd_lfIfLb1ELi4ELi0ELb0E", r"k_fdtd_lfIfLb1ELi4ELi3ELb0E",
        r"k_hotspot_vecIdLb0ELi2ELi1ELb0E", r"k_fdtd_lfIdLb1ELi2ELi0ELb0E", r"k_dist_wait", r"k_dist_signal"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
usage = {}
for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", res):
    usage[m.group(1)] = (int(m.group(2)), int(m.group(3)))
funcs = {}
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4}\*/", line):
        op = line.split("*/", 1)[1].strip().split(";")[0]
        op = re.sub(r"^@!?U?P\w+\s+", "", op)
        for k in KEYS:
            if op.startswith(k):
                funcs[cur][k] += 1
        funcs[cur]["total"] += 1

print("# SASS evidence (r01)\n")
print("`python tools/sass_evidence.py` over the built `libiterbatch_b200.so` (sm_100a, nvcc 12.9): "
      "static instruction counts per kernel. UBLKCP = `cp.async.bulk` on the TMA engine, SYNCS = "
      "mbarrier ops, ACQBULK / PREEXIT = `griddepcontrol.wait` / `launch_dependents` (programmatic "
      "dependent launch), MEMBAR = the cross-process system fence; FFMA / DFMA must be 0 (every "
      "numpy op is one correctly rounded `__f*_rn`, no contraction).\n")
print("| kernel | regs | stack | total | " + " | ".join(KEYS) + " |")
print("|---|---|---|---|" + "---|" * len(KEYS))
for w in WANT:
    for name, c in funcs.items():
        if re.search(w, name):
            demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            demangled = re.sub(r"\(.*\)$", "", demangled).replace("ib::", "")
            reg, stack = usage.get(name, ("?", "?"))
            print(f"| `{demangled}` | {reg} | {stack} | {c['total']} | " + " | ".join(str(c[k]) for k in KEYS) + " |")
            break

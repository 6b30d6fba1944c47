"""GPU: the bench contract line end to end (a short `python bench.py` run): every key the driver
reads, with the types and invariants it checks — value / ms_per_step / steps consistent, warmup
>= 3, the roofline (bound, achieved = bytes / time, peak, frac = achieved / peak, traffic),
cpu_baseline (kind, cores, sample), e2e (value, H2D / D2H bytes per step = the fields copied),
gpu_launches = steps x N x kernels per iteration, clocks sampled during the timed region."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_keeps_the_contract(gpu):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3",
                        "--quick", "--no-extra", "--no-f32", "--cpu-budget", "0.5"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # ONE JSON line
    d = json.loads(lines[0])
    assert d["metric"].startswith("µs/iteration") and d["unit"] == "µs/iteration"
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["higher_is_better"] is False and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert d["dtype"] == "f64" and d["data"].startswith("synthetic")
    assert d["config"]["workload"].startswith("Rodinia Hotspot 2-D 1024x1024") and "model" not in d["config"]
    n = d["config"]["iterations"]
    assert d["value"] > 0 and abs(d["ms_per_step"] - d["value"] * n / 1e3) < 1e-3 * d["ms_per_step"] + 1e-3
    roof = d["roofline"]
    assert roof["bound"] in ("hbm", "tensor") and roof["unit"] == "GB/s" and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-3
    assert roof["bytes_per_iter"] == 3 * 1024 * 1024 * 8  # read T, P; write T' (binary64)
    assert "traffic" in roof
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 2 * 1024 * 1024 * 8 and e2e["d2h_bytes_per_step"] == 1024 * 1024 * 8
    assert d["gpu_launches"] == d["steps"] * n
    clk = d["clocks"]
    assert clk["samples"] >= 1 and clk["sm_mhz"] > 0 and isinstance(clk["reasons"], list)

"""bench.py contract checks that need no GPU: the reference arm's JSON line, its torchrun
behaviour (rank 0 alone prints), and our arm failing loudly without a device."""
import json
import os
import subprocess
import sys

from .conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None, timeout=240):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH] + args, cwd=ROOT, env=e, capture_output=True,
                          text=True, timeout=timeout)


def test_reference_arm_line():
    p = _run(["--impl", "reference", "--only", "skeleton", "--steps", "2", "--warmup", "3"])
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["higher_is_better"] is False and d["unit"] == "µs/iteration"
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_warmup_floor():
    p = _run(["--impl", "reference", "--only", "skeleton", "--steps", "1", "--warmup", "1"])
    assert p.returncode == 0, p.stderr
    d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert d["warmup"] == 3  # timing rules: W >= 3


def test_reference_arm_under_torchrun():
    # launched like the driver's N>1 reference run: rank 0 alone runs and prints, the others exit 0
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29613", BENCH, "--impl", "reference",
           "--gpus", "2", "--only", "skeleton", "--steps", "1", "--warmup", "3"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_our_arm_fails_loudly_without_gpu():  # GPUs hidden: no CPU fallback, no line
    p = _run(["--steps", "1", "--warmup", "3", "--no-extra"], env={"CUDA_VISIBLE_DEVICES": ""})
    assert p.returncode != 0
    assert not [ln for ln in p.stdout.splitlines() if ln.startswith("{")]

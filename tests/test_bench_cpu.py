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
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["dtype"] == "f64"  # the reference computes in binary64 only
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


# ---- the line shapes of our arm (pure functions; no GPU) -------------------------------------------
def _bench():
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_under_test", BENCH)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class _Args:
    steps, warmup = 4, 3


def _dist_result(dtype):
    return {"name": "hotspot3d_large", "dtype": dtype, "workload": "w", "exchange": "peer stores",
            "iterations": 100, "batch_size": 20, "us_per_iter": 260.0, "ms_per_step": 26.0,
            "gpu_launches": 1200, "roofline": {"bound": "hbm", "achieved": 6000.0, "peak": 6448.4,
                                               "unit": "GB/s", "frac": 0.93, "traffic": None},
            "e2e": {"value": 300.0, "unit": "µs/iteration", "h2d_bytes_per_step": 1, "d2h_bytes_per_step": 1},
            "clocks": {"sm_mhz": 1900, "sm_max_mhz": 1965, "reasons": []}}


def test_scale_line_is_the_sharded_config_strong_scaling():
    """--gpus N > 1: the headline is Hotspot3D 2048^2x256 strong scaling — value is the max-over-
    ranks step time per iteration of the WHOLE grid (never a replica time divided by N), n_gpus == N,
    the config object equals the reference arm's, the 1-GPU base point rides along."""
    b = _bench()
    single = {"value": 2000.0, "n_gpus": 1}
    line = b.scale_line(_dist_result("f64"), _dist_result("f32"), single, _Args, 8, False)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 8 and line["scaling"] == "strong" and line["value"] == 260.0
    assert line["config"] == b.config_of("hotspot3d_large", "f64", 8)
    assert line["config"]["size"] == [2048, 2048, 256]
    assert line["single_gpu"]["value"] == 2000.0 and line["f32"]["value"] == 260.0
    assert line["gpu_launches"] == 1200 * 8
    shared = b.scale_line(_dist_result("f64"), None, None, _Args, 2, True)
    assert "protocol check" in shared["impl_detail"]["parallelism"]


def test_reference_arm_config_equals_ours():
    """same_config: the reference arm's `config` object is built by the same function, same dtype."""
    b = _bench()
    p = _run(["--impl", "reference", "--only", "skeleton", "--steps", "1", "--warmup", "3"])
    d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"] == b.config_of("skeleton", "f64", 1)


def test_gpus_n_spawns_n_ranks(monkeypatch):
    """`bench.py --gpus N` without WORLD_SIZE starts N ranks itself (torchrun on 127.0.0.1)."""
    b = _bench()
    seen = {}
    monkeypatch.setattr(b.subprocess, "call", lambda cmd, cwd=None: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(b.sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    assert b.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]

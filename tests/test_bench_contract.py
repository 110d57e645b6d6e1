"""bench.py's driver contract: one JSON line with the required keys (GPU), and --gpus N failing loudly when fewer
than N GPUs are visible (CPU)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_more_than_visible_fails_loudly():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2
    assert "needs 2 visible GPUs" in r.stderr


def test_reference_arm_line():
    """--impl reference: the CPU port on a tiny sample, with the reference arm's keys."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg4",
                        "--steps", "1", "--warmup", "0", "--cpu-sample", "512"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "voxels/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["cfg1", "cfg4"])
def test_bench_line_keys(config):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    args = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", "3", "--warmup", "3",
            "--no-cpu", "--no-clocks"]
    if config == "cfg4":
        args += ["--grid", "64", "64", "64", "--no-e2e"]
    r = subprocess.run(args, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches"):
        assert k in line, k
    assert line["value"] > 0 and line["gpu_launches"] > 0 and "workload" in line["config"]
    roof = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof, k
    if config == "cfg4":
        assert line["kernel_ms"]["fwd_ms"] > 0 and line["reconcile"]["ok"]

"""bench.py's output contract (one JSON line with the driver's keys), for the
reference arm on CPU and for our arm on the B200."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_reference_arm_contract():
    rec = _run(["--impl", "reference", "--steps", "2", "--warmup", "3"], 600)
    assert BASE_KEYS <= set(rec)
    assert rec["impl"] == "reference" and rec["value"] > 0 and rec["warmup"] >= 3
    cb = rec["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == rec["value"]
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["e2e"]["d2h_bytes_per_step"] == 0
    assert rec["config"]["workload"].startswith("c2")
    assert rec["config"]["same_config"] is True and rec["config"]["n"] == 1_000_000


def test_multi_rank_harness_over_gloo():
    """`bench.py --gpus 2` launches its own ranks (torch.distributed.run on
    127.0.0.1) when no torchrun environment is present; rank 0 prints one line
    with the world size."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--cpu-harness", "--steps", "3", "--warmup", "3"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=300, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["steps"] == 3 and rec["value"] > 0


@pytest.mark.gpu
def test_our_arm_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rec = _run(["--steps", "3", "--warmup", "3", "--no-solve", "--no-cpu"], 900)
    assert BASE_KEYS <= set(rec)
    assert rec["n_gpus"] == 1 and rec["steps"] == 3 and rec["higher_is_better"] is True
    rf = rec["roofline"]
    assert rf["bound"] == "hbm" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    assert rec["e2e"]["h2d_bytes_per_step"] > 0 and rec["e2e"]["d2h_bytes_per_step"] > 0
    assert rec["gpu_launches"] > 0 and "sm_mhz" in rec["clocks"]
    assert rec["sketch_precond_build"]["s1"]["ms"] > 0

"""bench.py's driver contract, checked on CPU through the reference arm (the oracle port on host
cores): one JSON line with the contract keys; under torchrun only rank 0 prints."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None):
    env = dict(os.environ, **(extra_env or {}))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--n", "32",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout


def test_reference_arm_prints_one_contract_line():
    lines = [ln for ln in _run().splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("config2")
    # like-for-like: the m = 40 factorisation, iterations sampled across j in [0, 40)
    assert d["config"]["m_sampled"] == 40 and d["config"]["j_sampled"] == [20]
    assert d["full_build"]["iterations_per_s"] > 0 and len(d["full_build"]["per_iteration_s"]) == 40
    assert "Gram-Schmidt" in d["config"]["orthogonalisation"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    assert _run({"WORLD_SIZE": "2", "RANK": "1"}).strip() == ""


@pytest.mark.gpu
def test_our_arm_contract_line_on_gpu():
    """Our arm on a small grid: roofline, cpu_baseline, e2e, clocks and launch count present
    and consistent (the full-size line is what the driver runs)."""
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    r = subprocess.run([sys.executable, "bench.py", "--n", "128", "--steps", "3", "--warmup", "3",
                        "--jv", "5", "--no-trajectory", "--no-secondary"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert len(d["cpu_baseline"]["j_sampled"]) == 5
    tp = d["two_pass"]
    assert tp["value"] > 0 and tp["iteration_roofline"]["frac"] > 0

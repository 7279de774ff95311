"""bench.py keeps the driver's contract: one JSON line with the required keys, for our
arm (GPU) and for the reference arm (the oracle on the host; runs here on CPU), also
under torchrun with 2 ranks (rank 0 alone prints)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _run(args, timeout=600, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=e)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout


def test_reference_arm_contract():
    lines = _json_lines(_run(["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"]))
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_torchrun_two_ranks():
    out = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                "--master-port", "29561", "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                "--warmup", "0"], env={"OMP_NUM_THREADS": "1"})
    lines = _json_lines(out)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


@pytest.mark.gpu
def test_our_arm_contract():
    lines = _json_lines(_run(["bench.py", "--steps", "3", "--warmup", "3", "--no-extra", "--cpu-seconds", "1",
                              "--e2e-steps", "1"]))
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0 and d["warmup"] >= 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # one fused codec launch per step (or codec + finalize, or decode group + encode group + finalize)
    assert d["gpu_launches"] in (d["steps"], 2 * d["steps"], 3 * d["steps"])
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["cpu_baseline"]["kind"] == "oracle"


def test_reference_arm_gpus_flag_without_torchrun():
    """`bench.py --impl reference --gpus 2` (no torchrun) reports the N asked for."""
    lines = _json_lines(_run(["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"]))
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


@pytest.mark.gpu
def test_our_arm_spawns_ranks():
    """`bench.py --gpus 2` started without torchrun spawns 2 ranks itself and prints ONE line
    with n_gpus 2 (on a 1-GPU box the ranks share it over gloo and the line says so)."""
    lines = _json_lines(_run(["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-extra",
                              "--cpu-seconds", "1", "--e2e-steps", "1"], timeout=900))
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["ranks"] == 2 and d["cpu_baseline"]["kind"] == "oracle"
    assert "error_combine" in d["config"]
    import torch

    if torch.cuda.device_count() < 2:
        assert "shared_gpus" in d["config"]


@pytest.mark.gpu
def test_multi_gpu_rows_real_ranks():
    """With >= 2 visible GPUs: the strong-scaling rows over 2 real ranks (NCCL and the peer
    combine side by side), first error found across ranks."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    lines = _json_lines(_run(["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1",
                              "--e2e-steps", "1"], timeout=1800))
    d = lines[0]
    r = d["rows"]["configs[4]"]
    assert r["first_error"] == r["first_error"] and r["injected"] == 1000
    assert r["decode_ms_with_combine_peer"] is not None

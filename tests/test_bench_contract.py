"""bench.py keeps the driver's contract: one JSON line with the required keys
(task statement).  The reference arm (the oracle on the host
cores) runs on CPU; the GPU arm needs a device."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config")


def run_bench(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         cwd=ROOT, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench(["--impl", "reference", "--config", "c0", "--steps", "2", "--warmup", "1"])
    for k in BASE_KEYS:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "c0"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench(["--config", "c0", "--steps", "5", "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline"])
    for k in BASE_KEYS + ("roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 5 and d["warmup"] == 3 and d["n_gpus"] == 1
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and r["achieved"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 5 * d["steps"]
    assert d["clocks"]["samples"] >= 1 and d["clocks"]["sm_mhz"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["c0", "c2"])
def test_gpu_arm_two_ranks(cfg):
    """The N > 1 path of bench.py (torchrun, one process per rank, k-d decomposition,
    first step with host-side counts, then the asynchronous all-to-all step, max-over-ranks
    timing, e2e per rank) with gloo as the transport so that both ranks can share the one
    GPU of the test box; its observables match the single-process run of the same steps."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    common = ["--config", cfg, "--steps", "4", "--warmup", "3", "--e2e-steps", "1", "--no-cpu-baseline"]
    one = run_bench(common)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo"] + common
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    two = json.loads(lines[0])
    assert two["n_gpus"] == 2 and two["value"] > 0 and two["steps"] == 4
    assert "gloo" in two["config"]["parallelism"]
    assert "error" not in two["e2e"], two["e2e"]
    a, b = one["observables"], two["observables"]
    assert a["step"] == b["step"]
    assert abs(a["U_pot"] - b["U_pot"]) <= 1e-5 * abs(a["U_pot"])
    assert abs(a["virial"] - b["virial"]) <= 1e-5 * abs(a["virial"])
    assert abs(a["T"] - b["T"]) <= 1e-5 * a["T"]
    assert abs(a["n_pairs"] - b["n_pairs"]) <= 2

"""bench.py keeps the driver's contract (-m gpu): one JSON line with the required keys, a positive value, the roofline
and e2e objects, device-timed steps; the reference arm prints its own line.  Run on config 0 with one timed step so
that it takes seconds."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "clocks", "e2e"]


def run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = run("--config", "0", "--steps", "2", "--warmup", "3", "--no-cpu-baseline")
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2
    assert d["unit"] == "MDoF*iter/s" and d["dtype"] == "f64" and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("cfg0")
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] <= 1.0 and r["peak"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0


def test_reference_arm_line():
    d = run("--impl", "reference", "--config", "0", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"


def test_two_rank_shm_bench():
    """The N > 1 flow of bench.py (barriers, max-over-ranks timing, decomposition, halo exchange inside every V-cycle
    and FGMRES dot) on the one GPU of the test box: two ranks over torchrun share cuda:0 through the host
    shared-memory transport (STGMG_COMM_SHM).  Config 1 (64 x 64 cells, split 32 + 32)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29631", os.path.join(ROOT, "bench.py"), "--gpus", "2", "--transport", "shm",
           "--config", "1", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "shared-memory" in d["config"]["parallelism"]

"""bench.py's JSON contract on small workloads (the driver runs the full
sizes): the single-GPU line, the emulated partitioned (C4-style) line and
the reference arm print one JSON line each with the keys the driver reads."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"}


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_single_gpu_line():
    d = _run("--nx", "200", "--ny", "150", "--seeds", "64", "--steps", "8", "--warmup", "3", "--cpu-seconds", "2")
    assert KEYS <= set(d)
    assert d["metric"] == "time-steps/sec (fused Euler step)" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"]
    assert d["parity"]["bitwise"] is True
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_emulated_partitioned_icosphere_line():
    d = _run("--emulate-ranks", "2", "--mesh", "ico7", "--seeds", "256", "--steps", "4", "--warmup", "3",
             "--no-e2e")
    assert d["scaling"] == "strong" and d["value"] > 0 and d.get("emulated") is True
    assert "icosphere-7" in d["config"]["workload"]


def test_reference_arm_line():
    d = _run("--impl", "reference", "--nx", "60", "--ny", "50", "--seeds", "16", "--steps", "2", "--warmup", "3")
    assert d["impl"] == "reference" and d["metric"] == "time-steps/sec (fused Euler step)"
    assert d["cpu_baseline"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


def test_torchrun_two_processes_line():
    """The driver's N>1 launch (torchrun, one process per rank) end to end,
    both ranks on cuda:0 with the host-staged gloo transport."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, FT_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(REPO, "bench.py"), "--gpus", "2", "--mesh", "ico7", "--seeds", "256",
                          "--steps", "4", "--warmup", "3"],
                         capture_output=True, text=True, timeout=900, cwd=REPO, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                       # rank 0 alone prints
    d = json.loads(lines[0])
    assert KEYS <= set(d)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0 and d["backend"] == "gloo"
    assert d["e2e"]["d2h_bytes_per_step"] > 0

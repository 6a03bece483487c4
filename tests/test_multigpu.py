"""Multi-GPU parity (one process per GPU over CUDA-IPC windows); runs
tests/mp_worker.py under torchrun on every visible GPU (>= 2)."""

import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_multigpu_parity_torchrun():
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={n}", "--master-addr=127.0.0.1",
           f"--master-port={_port()}", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("[PASS]") >= 6


def test_multigpu_stress_with_random_delays():
    """10,000 LL rounds (64 tokens), 5,000 LL rounds (2 tokens) and 500 HT
    rounds across real GPUs with random
    __nanosleep before payload stores and releases in every kernel
    (EPB_CHAOS_NS), bit-exact every round (the reference's flush-ordering
    property test, test_acceptance.py:286-292, on hardware)."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    env = dict(os.environ, EPB_MP_STRESS=os.environ.get("EPB_MP_STRESS", "10000"),
               EPB_CHAOS_NS=os.environ.get("EPB_CHAOS_NS", "3000"))
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={n}", "--master-addr=127.0.0.1",
           f"--master-port={_port()}", os.path.join(ROOT, "tests", "mp_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=ROOT, env=env)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("[PASS]") == 3

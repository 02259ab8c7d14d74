"""Multi-GPU parity (skipped on a one-GPU box): tools/dist_parity.py under
torchrun -- the distributed round loop with the NVLink peer-memory and the
NCCL transports reproduces the oracle's run_parallel bit for bit."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_distributed_round_loop_matches_oracle():
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + os.getpid() % 300),
           str(ROOT / "tools" / "dist_parity.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in out.stdout.splitlines() if l.startswith(("OK", "BAD"))]
    assert out.returncode == 0 and lines and all(l.startswith("OK") for l in lines), out.stdout + out.stderr

"""Multi-GPU parity (P2P and NCCL transports, direct and two-level) via torchrun.

Skipped unless at least 2 GPUs are visible; run with `gpurun --gpus 2|4`.
"""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _gpus() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("n", [2, 4])
def test_multirank_parity(n):
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29531", str(ROOT / "tests" / "workers" / "dist_parity.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:], out.stderr[-4000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]


@pytest.mark.parametrize("n", [2, 4])
def test_multirank_sharded_aggregate(n):
    """K5 over an edge list split across ranks (limbs all-reduced) == single-GPU aggregate, bit for bit."""
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29532", str(ROOT / "tests" / "workers" / "dist_aggregate.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:], out.stderr[-4000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]

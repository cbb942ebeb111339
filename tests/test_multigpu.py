"""Multi-GPU parity (N ranks = N GPUs over NCCL): runs tests/mp_worker.py
under torchrun on every visible GPU (2, 4 or 8)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpus():
    import torch
    n = torch.cuda.device_count()
    p = 1
    while p * 2 <= n:
        p *= 2
    return p


def test_multi_rank_parity():
    n = _ngpus()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(HERE, "mp_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-6000:]
    assert "CASE train_e8: PASS" in out
    assert "CASE train_adagrad: PASS" in out

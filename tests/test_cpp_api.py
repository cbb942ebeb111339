"""GPU: the C++ host-side mirror of the reference API (include/hps_gpu/hbm_tier.hpp)
driven by a compiled C++ test (tests/cpp/test_hbm_tier.cpp)."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_hbm_tier")

pytestmark = pytest.mark.gpu


def test_cpp_hbm_tier_parity():
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/test_hbm_tier not built (run __graft_entry__.build())")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert " 0 failed" in p.stdout


COMPAT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_hps_compat")


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("G", [1, 2])
def test_cpp_reference_api_device_worker_loop(G):
    """include/hps_gpu/hbm_ps.hpp (namespace hps, the reference signatures)
    driven by the reference's device-worker loop, one thread per device; at
    G = 2 both handles live in one process (same-process NVLink peer path)."""
    if G > _gpus():
        pytest.skip(f"needs {G} GPUs")
    if not os.path.exists(COMPAT):
        pytest.fail("tests/cpp/test_hps_compat not built (run __graft_entry__.build())")
    p = subprocess.run([COMPAT, str(G)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert " 0 failed" in p.stdout

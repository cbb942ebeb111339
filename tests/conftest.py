import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def _gpu_count() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def pytest_collection_modifyitems(config, items):
    n = _gpu_count()
    for it in items:
        if "gpu" in it.keywords and n == 0:
            it.add_marker(pytest.mark.skip(reason="no CUDA GPU"))
        if "multigpu" in it.keywords and n < 2:
            it.add_marker(pytest.mark.skip(reason="needs >= 2 GPUs"))


@pytest.fixture(scope="session")
def oracle():
    from native import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def pkg():
    import paper_2003_05622_b200 as p
    p.lib()
    return p

"""CPU: the drop-in boundary. libhps_gpu.so loads without a GPU, exports every
function include/hps_gpu.h declares, and the host-only entry points work;
compute entry points fail cleanly (an hps_status, no crash) when no GPU is
present — there is no CPU fallback."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hps_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hps_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_reference_boundary():
    names = declared_functions()
    for must in ["hps_create", "hps_destroy", "hps_build", "hps_pull", "hps_push", "hps_drain",
                 "hps_dump", "hps_table_info", "hps_table_slots", "hps_dense_sync",
                 "hps_train_batch", "hps_attach_store", "hps_gen_dataset", "hps_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(pkg):
    lib = ctypes.CDLL(pkg.hps.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding knows every one of them
    assert set(declared_functions()) <= set(pkg.hps._SIGS)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2003_05622_b200", "libhps_gpu.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_and_generator_need_no_gpu(pkg):
    assert b"sm_100a" in pkg.lib().hps_version()
    off, keys, lab = pkg.gen_dataset(1000, 10, 5, seed=2)
    assert off.tolist() == list(range(0, 55, 5))
    for e in range(10):
        ex = keys[off[e]:off[e + 1]]
        assert (np.diff(ex.astype(np.int64)) > 0).all()  # sorted unique features
    with pytest.raises(pkg.Error) as ei:
        pkg.gen_dataset(3, 1, 5)
    assert "nnz <= dims" in str(ei.value)


def test_config_validation_errors(pkg):
    with pytest.raises(pkg.Error) as ei:
        pkg.Tier(nodes=3)
    assert "power of two" in str(ei.value)
    with pytest.raises(pkg.Error) as ei:
        pkg.Tier(layer_dims=(8, 2))
    assert "end in 1" in str(ei.value)


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and
                    __import__("torch").cuda.is_available(), reason="GPU present")
def test_create_without_gpu_fails_cleanly(pkg):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pkg.Error) as ei:
        pkg.Tier(width=8)
    assert ei.value.code in ("HPS_ERR_CUDA",)

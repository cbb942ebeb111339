"""B200-native HBM-PS tier of the hierarchical GPU parameter server
(arXiv 2003.05622): sm_100a kernels behind the C ABI in include/hps_gpu.h.

The product is ``libhps_gpu.so`` (built in-tree from ``csrc/``); ``hps`` is its
ctypes binding plus a host-side mirror of the reference ``hps::HbmTier`` API.
"""
from . import hps  # noqa: F401
from .hps import (DeviceTable, Error, HbmTier, Tier, Topology, canonical_order,  # noqa: F401
                  gen_dataset, gen_multislot, lib, synchronize, unique_id)

__all__ = ["hps", "Tier", "HbmTier", "DeviceTable", "Topology", "Error", "gen_dataset", "gen_multislot",
           "synchronize", "canonical_order", "unique_id", "lib"]

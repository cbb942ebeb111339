"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libhps_ref.so, built from /root/reference/proj/include
by `make -C oracle ref`). Run in the build container:

    python tests/golden/make_golden.py

Fixtures (numpy .npz, compressed):
  dataset.npz       gen_dataset outputs for small specs + sha256 of the c1/c2
                    first batches (dataset.hpp:180-227)
  table.npz         DeviceTable slot order + capacity for key sets
                    (device_table.hpp:38-101, ascending insert hbm_ps.hpp:89-98)
  partition.npz     HbmTier::build_all ownership for Appendix-A keys and a
                    generated batch; extract_working_set (mem_ps.hpp:101-108)
  model.npz         init_dense + forward/backward on small shards (model.hpp)
  sync.npz          canonical_sum / synchronize (hbm_ps.hpp:258-408)
  train.npz         train_reference final parameters (oracle.hpp:55-122) and
                    the threaded HBM-PS hot path (pipeline.hpp:502-566)
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from native import RefHotPath, RefLib, make_cfg  # noqa: E402

DATASET_SPECS = [  # dims, n, nnz, zipf, s, seed, scale, clusters
    (1000, 200, 10, False, 1.0, 1, 6.0, 0),
    (1000, 200, 10, True, 1.0, 3, 6.0, 0),
    (10000, 100, 20, False, 1.0, 5, 6.0, 50),
    (10000, 100, 20, True, 1.2, 5, 6.0, 50),
    (500, 60, 5, False, 1.0, 7, 4.0, 0),
]
BIG_SPECS = {  # the first batch of BASELINE configs 1 and 2
    "c1": (10**6, 4096, 100, False, 1.0, 1, 6.0, 0),
    "c2": (10**7, 16384, 100, True, 1.0, 1, 6.0, 0),
}
TRAIN_CASES = [  # name, nodes, devices, E, layers, J, dims, B, nbatch_examples, nnz, zipf
    ("n1d1_e8", 1, 1, 8, (8, 16, 1), 4, 5000, 256, 3 * 256, 20, False),
    ("n1d2_e4", 1, 2, 4, (4, 1), 2, 500, 60, 3 * 60 + 7, 5, False),
    ("n1d8_e8_zipf", 1, 8, 8, (8, 16, 1), 4, 5000, 256, 3 * 256, 20, True),
    ("n2d2_e8", 2, 2, 8, (8, 16, 1), 4, 5000, 256, 4 * 256 + 3, 20, False),
    ("n1d4_e16_zipf", 1, 4, 16, (8, 16, 1), 4, 100000, 1024, 2 * 1024, 50, True),
]


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    ref = RefLib()
    out = {}
    # ---- dataset
    d = {}
    for i, spec in enumerate(DATASET_SPECS):
        off, keys, lab = ref.gen_dataset(*spec)
        d[f"spec{i}"] = np.array(spec, dtype=np.float64)
        d[f"off{i}"], d[f"keys{i}"], d[f"lab{i}"] = off, keys, lab
    for name, spec in BIG_SPECS.items():
        off, keys, lab = ref.gen_dataset(*spec)
        d[f"big_{name}_spec"] = np.array(spec, dtype=np.float64)
        d[f"big_{name}_sha256"] = np.array(digest(off, keys, lab))
        ws = ref.working_set(off, keys)
        d[f"big_{name}_ws_size"] = np.array(ws.size)
        d[f"big_{name}_ws_sha256"] = np.array(digest(ws))
    out["dataset"] = d
    # ---- table layouts
    t = {}
    rng = np.random.default_rng(2026)
    for i, n in enumerate([0, 1, 6, 7, 100, 5000, 20000]):
        ks = np.unique(rng.integers(0, 1 << 40, size=n, dtype=np.uint64))
        order, cap = ref.table_slot_order(ks)
        t[f"keys{i}"], t[f"order{i}"], t[f"cap{i}"] = ks, order, np.array(cap)
    out["table"] = t
    # ---- partition / working set
    p = {}
    appendix_a = np.array([4, 5, 11, 50, 53, 56, 61, 87, 98], dtype=np.uint64)
    for (nn, dd) in [(1, 2), (1, 4), (2, 2), (1, 8), (4, 2)]:
        u, g = ref.partition(nn, dd, appendix_a)
        p[f"appA_{nn}x{dd}_keys"], p[f"appA_{nn}x{dd}_owner"] = u, g
    off, keys, lab = ref.gen_dataset(*DATASET_SPECS[1])
    ws = ref.working_set(off[:65], keys[: off[64]])
    p["ws_keys_in_off"], p["ws_keys_in"], p["ws"] = off[:65], keys[: off[64]], ws
    u, g = ref.partition(1, 4, keys)
    p["gen_1x4_keys"], p["gen_1x4_owner"] = u, g
    out["partition"] = p
    # ---- model
    mdl = {}
    for i, (E, layers, seed) in enumerate([(8, (8, 16, 1), 42), (4, (4, 1), 7), (16, (8, 16, 1), 3),
                                          (1, (1,), 11), (3, (5, 2, 1), 9)]):
        cfg = make_cfg(1, 1, E, layers, seed=seed)
        dense = ref.init_dense(cfg)
        off, keys, lab = ref.gen_dataset(300, 40, 6, False, 1.0, seed, 6.0, 0)
        ek = np.unique(keys)
        r2 = np.random.default_rng(seed)
        er = (r2.random((ek.size, E)) - 0.5).astype(np.float32)
        preds, dg, sg = ref.forward_backward(E, layers, dense, off, keys, lab, ek, er)
        mdl[f"E{i}"] = np.array(E)
        mdl[f"layers{i}"] = np.array(layers, dtype=np.uint64)
        mdl[f"seed{i}"] = np.array(seed)
        mdl[f"dense{i}"], mdl[f"off{i}"], mdl[f"keys{i}"], mdl[f"lab{i}"] = dense, off, keys, lab
        mdl[f"ek{i}"], mdl[f"er{i}"] = ek, er
        mdl[f"preds{i}"], mdl[f"dgrad{i}"], mdl[f"sgrad{i}"] = preds, dg, sg
    out["model"] = mdl
    # ---- sync
    s = {}
    rng = np.random.default_rng(9)
    for (nn, dd) in [(1, 4), (2, 2), (4, 8), (1, 1), (2, 4)]:
        bufs = (rng.random((nn * dd, 33)) - 0.5).astype(np.float32)
        s[f"bufs_{nn}x{dd}"] = bufs
        s[f"canon_{nn}x{dd}"] = ref.canonical_sum(nn, dd, bufs)
        s[f"det_{nn}x{dd}"] = ref.synchronize(nn, dd, True, bufs)
        s[f"fast_{nn}x{dd}"] = ref.synchronize(nn, dd, False, bufs)
    out["sync"] = s
    # ---- training
    tr = {}
    for (name, nn, dd, E, layers, J, dims, B, n, nnz, zipf) in TRAIN_CASES:
        off, keys, lab = ref.gen_dataset(dims, n, nnz, zipf, 1.0, 1, 6.0, 0)
        cfg = make_cfg(nn, dd, E, layers, J=J)
        dense, sk, sr = ref.train_reference(cfg, B, off, keys, lab)
        tr[f"{name}_spec"] = np.array([nn, dd, E, J, dims, B, n, nnz, int(zipf)], dtype=np.int64)
        tr[f"{name}_layers"] = np.array(layers, dtype=np.int64)
        tr[f"{name}_dense"], tr[f"{name}_keys"], tr[f"{name}_rows"] = dense, sk, sr
        if nn == 1:  # the threaded reference hot path agrees bit-for-bit
            hp = RefHotPath(ref, cfg, B, off, keys, lab)
            hp.run(0, (n + B - 1) // B)
            hd, hk, hr = hp.export(dims)
            hp.close()
            assert np.array_equal(hd, dense) and np.array_equal(hk, sk) and np.array_equal(hr, sr), name
    out["train"] = tr
    for name, arrays in out.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **arrays)
        print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(arrays)} arrays)")


if __name__ == "__main__":
    main()

"""CPU: the oracle restatement (oracle/hps_oracle.c) and the package's input
generator against golden fixtures produced by the UNMODIFIED reference
(tests/golden/make_golden.py). This pins the oracle before the GPU parity
tests trust it."""
import hashlib
import os

import numpy as np
import pytest

from native import dense_count, make_cfg

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ------------------------------------------------------------- generator --

def test_generator_matches_reference_small_specs(pkg):
    d = load("dataset")
    i = 0
    while f"spec{i}" in d:
        dims, n, nnz, zipf, s, seed, scale, clusters = d[f"spec{i}"].tolist()
        off, keys, lab = pkg.gen_dataset(int(dims), int(n), int(nnz), bool(zipf), s, int(seed),
                                         scale, int(clusters))
        assert np.array_equal(off, d[f"off{i}"])
        assert np.array_equal(keys, d[f"keys{i}"])
        assert np.array_equal(lab, d[f"lab{i}"])
        i += 1
    assert i >= 5


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_generator_matches_reference_baseline_batches(pkg, oracle, name):
    d = load("dataset")
    dims, n, nnz, zipf, s, seed, scale, clusters = d[f"big_{name}_spec"].tolist()
    off, keys, lab = pkg.gen_dataset(int(dims), int(n), int(nnz), bool(zipf), s, int(seed), scale,
                                     int(clusters))
    assert digest(off, keys, lab) == str(d[f"big_{name}_sha256"])
    ws = oracle.sort_unique(keys)  # mem_ps.hpp:101-108
    assert ws.size == int(d[f"big_{name}_ws_size"])
    assert digest(ws) == str(d[f"big_{name}_ws_sha256"])


# ----------------------------------------------------------------- table --

def test_table_layout_matches_reference(oracle):
    t = load("table")
    i = 0
    while f"keys{i}" in t:
        ks = t[f"keys{i}"]
        slots = oracle.table_build(ks)
        assert slots.size == int(t[f"cap{i}"])
        assert np.array_equal(slots[slots != np.uint64(2**64 - 1)], t[f"order{i}"])
        for k in ks[:50]:
            assert slots[oracle.L.or_table_find(slots.ctypes.data, slots.size, int(k))] == k
        i += 1


def test_capacity_rule(oracle):
    """test_device_table.cpp:33-47 and device_table.hpp:38-45."""
    assert oracle.capacity(6) == 8
    assert oracle.capacity(0) == 1
    assert oracle.capacity(7) == 16
    assert oracle.capacity(335830) == 524288  # config-1 working set


def test_table_overflow_and_duplicate_are_errors(oracle):
    import ctypes
    slots = np.empty(8, np.uint64)
    ks = np.arange(7, dtype=np.uint64)  # 7 > 0.75 * 8
    assert oracle.L.or_table_build(ks.ctypes.data, 7, 8, slots.ctypes.data) == 1
    assert "capacity overflow" in oracle.err()
    dup = np.array([3, 3], np.uint64)
    assert oracle.L.or_table_build(dup.ctypes.data, 2, 4, slots.ctypes.data) == 1
    assert "duplicate insert of key 3" in oracle.err()
    del ctypes


# ------------------------------------------------------ partition / dedup --

def test_partition_matches_reference(oracle):
    p = load("partition")
    for (nn, dd) in [(1, 2), (1, 4), (2, 2), (1, 8), (4, 2)]:
        keys = p[f"appA_{nn}x{dd}_keys"]
        assert np.array_equal(oracle.owner(keys, nn, dd), p[f"appA_{nn}x{dd}_owner"])
    keys = p["gen_1x4_keys"]
    assert np.array_equal(oracle.owner(keys, 1, 4), p["gen_1x4_owner"])
    assert np.array_equal(oracle.sort_unique(p["ws_keys_in"]), p["ws"])


def test_appendix_a_working_set(oracle):
    """test_mem_ps.cpp:63-75 / test_hbm_ps.cpp:42-60 worked example."""
    ks = np.array([98, 4, 53, 5, 11, 87, 50, 56, 61, 4, 53], np.uint64)
    assert oracle.sort_unique(ks).tolist() == [4, 5, 11, 50, 53, 56, 61, 87, 98]


def test_shard_batch(oracle):
    """test_pipeline.cpp:116-156."""
    dv, mb = oracle.shard(8, 2, 2)
    counts = np.zeros((2, 2), int)
    for d, j in zip(dv, mb):
        counts[d, j] += 1
    assert (counts == 2).all()
    dv, mb = oracle.shard(5, 2, 2)
    sizes = sorted(np.bincount(dv * 2 + mb, minlength=4).tolist())
    assert sizes == [1, 1, 1, 2]


# ----------------------------------------------------------------- model --

def test_init_dense_and_forward_backward_match_reference(oracle):
    m = load("model")
    i = 0
    while f"E{i}" in m:
        E, layers, seed = int(m[f"E{i}"]), m[f"layers{i}"].tolist(), int(m[f"seed{i}"])
        cfg = make_cfg(1, 1, E, layers, seed=seed)
        assert np.array_equal(oracle.init_dense(cfg), m[f"dense{i}"])
        preds, dg, sg = oracle.forward_backward(E, layers, m[f"dense{i}"], m[f"off{i}"],
                                                m[f"keys{i}"], m[f"lab{i}"], m[f"ek{i}"],
                                                m[f"er{i}"])
        assert np.array_equal(preds, m[f"preds{i}"])
        assert np.array_equal(dg, m[f"dgrad{i}"])
        assert np.array_equal(sg, m[f"sgrad{i}"])
        i += 1
    assert i == 5


def test_sigmoid_known_answer(oracle):
    """test_model.cpp:83-89: E=1, w=1, b=0, x=2 -> sigmoid(2)."""
    preds, _, _ = oracle.forward_backward(1, [1], np.array([1.0, 0.0], np.float32),
                                          np.array([0, 1]), np.array([7], np.uint64),
                                          np.array([1], np.uint8), np.array([7], np.uint64),
                                          np.array([[2.0]], np.float32))
    assert abs(preds[0] - 0.8807970779778823) < 1e-12


def test_closed_form_gradients(oracle):
    """test_model.cpp:122-134: E=1 linear model."""
    w, b, x = 1.3, 0.2, 0.7
    preds, dg, sg = oracle.forward_backward(1, [1], np.array([w, b], np.float32),
                                            np.array([0, 1]), np.array([5], np.uint64),
                                            np.array([1], np.uint8), np.array([5], np.uint64),
                                            np.array([[x]], np.float32))
    p = preds[0]
    assert abs(dg[0] - (p - 1.0) * np.float32(x)) < 1e-6
    assert abs(dg[1] - (p - 1.0)) < 1e-6
    assert abs(sg[0, 0] - (p - 1.0) * np.float32(w)) < 1e-6


def test_sgd_delta_accumulate_equals_apply_update(oracle):
    """test_model.cpp:228-235: bitwise."""
    import ctypes
    w1 = np.array([0.37], np.float32)
    g = np.array([0.113], np.float32)
    w2 = w1.copy()
    s = g.copy()
    oracle.L.or_average_apply(w1.ctypes.data, s.ctypes.data, 1, 1, ctypes.c_float(0.05))
    oracle.L.or_sgd_accumulate(w2.ctypes.data, g.ctypes.data, 1, ctypes.c_float(0.05))
    assert w1.tobytes() == w2.tobytes()


# ------------------------------------------------------------------ sync --

def test_canonical_sum_matches_reference(oracle):
    s = load("sync")
    for (nn, dd) in [(1, 4), (2, 2), (4, 8), (1, 1), (2, 4)]:
        bufs = s[f"bufs_{nn}x{dd}"]
        got = oracle.canonical_sum(nn, dd, bufs)
        assert np.array_equal(got, s[f"canon_{nn}x{dd}"])
        # the reference's deterministic synchronize == canonical_sum on every replica
        for r in s[f"det_{nn}x{dd}"]:
            assert np.array_equal(r, got)
        # default mode (f32 partial sums): within 1e-6 of the summands' scale
        # (test_hbm_ps.cpp:242-265 states it relative to the sum for its data)
        scale = np.maximum(np.abs(bufs).sum(axis=0), 1e-9)
        assert (np.abs(s[f"fast_{nn}x{dd}"] - got) / scale).max() < 1e-6


def test_sync_one_to_four_sums_to_ten(oracle):
    """test_hbm_ps.cpp:179-192."""
    for nn, dd in [(1, 4), (2, 2)]:
        bufs = np.array([[1.0], [2.0], [3.0], [4.0]], np.float32)
        assert oracle.canonical_sum(nn, dd, bufs).tolist() == [10.0]


# -------------------------------------------------------------- training --

def test_train_reference_matches_reference(oracle, pkg):
    tr = load("train")
    names = sorted({k.rsplit("_", 1)[0] for k in tr.files if k.endswith("_spec")})
    assert len(names) == 5
    for name in names:
        nn, dd, E, J, dims, B, n, nnz, zipf = tr[f"{name}_spec"].tolist()
        layers = tr[f"{name}_layers"].tolist()
        off, keys, lab = pkg.gen_dataset(dims, n, nnz, bool(zipf), seed=1)
        cfg = make_cfg(nn, dd, E, layers, J=J)
        dense, sk, sr = oracle.train_reference(cfg, B, off, keys, lab)
        assert dense.size == dense_count(E, layers)
        assert np.array_equal(dense, tr[f"{name}_dense"]), name
        assert np.array_equal(sk, tr[f"{name}_keys"]), name
        assert np.array_equal(sr, tr[f"{name}_rows"]), name


def test_multi_topology_determinism(oracle, pkg):
    """deterministic mode at 1x2, 1x4, 1x8 equals the canonical
    single-site update; different device counts shard differently, so only
    the 1x1 vs itself and per-topology reproducibility are asserted here."""
    off, keys, lab = pkg.gen_dataset(500, 130, 5, seed=3)
    for dd in (1, 2, 4, 8):
        a = oracle.train_reference(make_cfg(1, dd, 4, (4, 1), J=2), 60, off, keys, lab)
        b = oracle.train_reference(make_cfg(1, dd, 4, (4, 1), J=2), 60, off, keys, lab)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_auc_known_answers(oracle):
    """test_model.cpp:245-258."""
    assert oracle.auc([0, 0, 1, 1], [0.1, 0.2, 0.8, 0.9]) == 1.0
    assert oracle.auc([1, 1, 0, 0], [0.1, 0.2, 0.8, 0.9]) == 0.0
    assert oracle.auc([0, 1, 0, 1], [0.5, 0.5, 0.5, 0.5]) == 0.5

"""GPU parity of the Adagrad extension (BASELINE config 3: "emb dim 64 with
Adagrad state"). The optimizer state lives in the
HBM table row beside the embedding (rows of 2E floats) and travels with it
through build, carry-over, the store proxies, the value store, write-back,
dump and export; the owner applies the fused Adagrad step in place
(common.cuh Optim). Checked bit for bit against the oracle's self-pinned
restatement (oracle/hps_oracle.c or_adagrad_apply, pinned by
tests/test_oracle_adagrad.py)."""
import numpy as np
import pytest

from native import make_cfg

pytestmark = pytest.mark.gpu


def run(pkg, off, keys, lab, B, *, E, J, dims, store_kind="host", pipelined=False,
        layers=(8, 16, 1), eps=1e-8):
    import torch
    nb = (len(off) - 1 + B - 1) // B
    mk = int(max(off[min((b + 1) * B, len(off) - 1)] - off[b * B] for b in range(nb)))
    tier = pkg.Tier(width=E, layer_dims=layers, minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=mk, optimizer="adagrad",
                    adagrad_eps=eps)
    assert tier.row_width == 2 * E
    if store_kind == "host":
        store = np.zeros((dims, 2 * E), np.float32)
        tier.attach_store(store)
    else:
        dstore = torch.zeros((dims, 2 * E), dtype=torch.float32, device="cuda")
        tier.attach_store(dstore.data_ptr(), on_device=True, num_keys=dims)
    for b in range(nb):
        e0, e1 = b * B, min((b + 1) * B, len(off) - 1)
        args = (off[e0:e1 + 1] - off[e0], keys[off[e0]:off[e1]], lab[e0:e1])
        if pipelined:
            tier.submit_batch(*args)
            if b >= 2:
                tier.wait_batch()
        else:
            tier.train_batch(*args)
    if pipelined:
        for _ in range(min(nb, 2)):
            tier.wait_batch()
    tier.flush()
    dense = tier.get_dense()
    dk, dr = tier.dump()
    tier.close()
    if store_kind != "host":
        torch.cuda.synchronize()
        store = dstore.cpu().numpy()
    return dense, store, (dk, dr)


@pytest.mark.parametrize("E,J,zipf,store_kind,pipelined", [
    (8, 4, True, "host", False),
    (16, 4, True, "host", True),
    (16, 4, True, "device", True),
    (64, 4, False, "device", True),
    (12, 3, True, "host", False),
    (1, 1, False, "host", False),
])
def test_adagrad_train_bit_exact(pkg, oracle, E, J, zipf, store_kind, pipelined):
    dims, B, nnz = 30000, 512, 20
    off, keys, lab = pkg.gen_dataset(dims, 5 * B, nnz, zipf=zipf, seed=23)
    dense, store, (dk, dr) = run(pkg, off, keys, lab, B, E=E, J=J, dims=dims,
                                 store_kind=store_kind, pipelined=pipelined)
    wd, wk, wr = oracle.train_reference(
        make_cfg(1, 1, E, (8, 16, 1), J=J, optimizer="adagrad"), B, off, keys, lab)
    assert np.array_equal(dense, wd)
    got = store[wk.astype(np.int64)]
    bad = np.nonzero((got != wr).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, e.g. key {wk[bad[0]]}: {got[bad[0]]} vs {wr[bad[0]]}"
    assert (wr[:, E:] > 0).any()  # the state really accumulated
    # dump_node of the last table: the same rows (embedding + state)
    idx = np.searchsorted(wk, dk)
    assert np.array_equal(dr, wr[idx])


def test_adagrad_big_segments_and_forced_fallback(pkg, oracle, monkeypatch):
    """Hot keys (chunked big_fused path, its fused Adagrad apply), with every
    certificate forced to fail (the exact fallbacks feed the same apply)."""
    monkeypatch.setenv("HPS_MID_SEG", "32")  # the long segments on the certified path
    for force in ("0", "1"):
        monkeypatch.setenv("HPS_CERT_FORCE_FAIL", force)
        dims, B, E = 20000, 4096, 16
        off, keys, lab = pkg.gen_dataset(dims, 2 * B, 20, zipf=True, seed=31)
        dense, store, _ = run(pkg, off, keys, lab, B, E=E, J=4, dims=dims)
        wd, wk, wr = oracle.train_reference(
            make_cfg(1, 1, E, (8, 16, 1), J=4, optimizer="adagrad"), B, off, keys, lab)
        assert np.array_equal(dense, wd)
        assert np.array_equal(store[wk.astype(np.int64)], wr)


def test_adagrad_sort_dedup_path(pkg, oracle, monkeypatch):
    """HPS_DEDUP=sort: deltas go through the push rows and table_apply_kernel
    (the G > 1 style apply) instead of the fused in-place apply."""
    monkeypatch.setenv("HPS_DEDUP", "sort")
    dims, B, E = 20000, 512, 16
    off, keys, lab = pkg.gen_dataset(dims, 3 * B, 20, zipf=True, seed=8)
    dense, store, _ = run(pkg, off, keys, lab, B, E=E, J=4, dims=dims)
    wd, wk, wr = oracle.train_reference(
        make_cfg(1, 1, E, (8, 16, 1), J=4, optimizer="adagrad"), B, off, keys, lab)
    assert np.array_equal(dense, wd)
    assert np.array_equal(store[wk.astype(np.int64)], wr)


def test_adagrad_parity_api_push_drain(pkg, oracle):
    """build (host rows carry embedding + state), push gradients, drain applies
    the Adagrad step per sender; pull returns the embeddings only."""
    E = 8
    tier = pkg.Tier(width=E, key_space=1000, max_batch_keys=64, optimizer="adagrad",
                    adagrad_eps=1e-6)
    keys = np.array([3, 17, 40, 999], np.uint64)
    rows = np.random.default_rng(1).standard_normal((4, 2 * E)).astype(np.float32)
    rows[:, E:] = np.abs(rows[:, E:])
    tier.build(keys, rows)
    assert np.array_equal(tier.pull(keys), rows[:, :E])
    g = np.random.default_rng(2).standard_normal((4, E)).astype(np.float32)
    tier.push(keys, g)
    tier.drain()
    dk, dr = tier.dump()
    tier.close()
    want_v, want_s = oracle.adagrad_apply(rows[:, :E].ravel(), rows[:, E:].ravel(), g.ravel(),
                                          0.05, 1e-6)
    assert np.array_equal(dk, keys)
    assert dr[:, :E].tobytes() == want_v.tobytes()
    assert dr[:, E:].tobytes() == want_s.tobytes()


def test_adagrad_export_writes_opt_state(pkg, oracle, tmp_path):
    """hps_export: opt_state of every record = the Adagrad accumulator; the
    unmodified reference SsdStore loads and fscks the files."""
    from native import RefLib
    ref = RefLib()
    dims, B, E = 20000, 512, 16
    off, keys, lab = pkg.gen_dataset(dims, 2 * B, 20, zipf=True, seed=12)
    tier = pkg.Tier(width=E, key_space=dims, max_batch_examples=B,
                    max_batch_keys=int(off[B] - off[0]) + int(off[2 * B] - off[B]),
                    optimizer="adagrad")
    store = np.zeros((dims, 2 * E), np.float32)
    tier.attach_store(store)
    for b in range(2):
        tier.train_batch(off[b * B:(b + 1) * B + 1] - off[b * B],
                         keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
    nf = tier.export(str(tmp_path), file_capacity=500)
    tier.close()
    want = np.unique(keys[off[B]:off[2 * B]])
    k, e, o, info = ref.store_load_all(str(tmp_path), E, want.size)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, (8, 16, 1), J=4, optimizer="adagrad"),
                                        B, off, keys, lab)
    rows = dict(zip(wk.tolist(), wr))
    assert np.array_equal(k, want)
    assert e.tobytes() == np.stack([rows[int(x)][:E] for x in k]).tobytes()
    assert o.tobytes() == np.stack([rows[int(x)][E:] for x in k]).tobytes()
    assert info["fsck_ok"] == 1 and info["files"] == nf

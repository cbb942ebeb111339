"""GPU parity of the fused per-batch hot path (hps_train_batch) against the
oracle's train_reference restatement (oracle.hpp:55-122).

Deterministic mode must be bit-exact for every parameter (the reference's own
1x1 contract, test_pipeline.cpp:167-183; SURVEY §8c holds the GPU to the same
bar). Fast mode is held to the reference verify tolerance (max relative
parameter difference < 1e-5, hps_main.cpp:164-223).
"""
import numpy as np
import pytest

from native import make_cfg

pytestmark = pytest.mark.gpu


def run_gpu(pkg, off, keys, lab, B, *, E, layers, J, dims, det=True, skip=-1,
            device_store=False):
    nb = (len(off) - 1 + B - 1) // B
    tier = pkg.Tier(width=E, layer_dims=layers, minibatches=J, key_space=dims,
                    deterministic=det, inject_skip_sync=skip, max_batch_examples=B,
                    max_batch_keys=int(max(off[min((b + 1) * B, len(off) - 1)] - off[b * B]
                                           for b in range(nb))))
    store = np.zeros((dims, E), dtype=np.float32)
    tier.attach_store(store)
    losses = []
    for b in range(nb):
        e0, e1 = b * B, min((b + 1) * B, len(off) - 1)
        o = off[e0:e1 + 1] - off[e0]
        st = tier.train_batch(o, keys[off[e0]:off[e1]], lab[e0:e1])
        losses.append(st.loss_sum / max(1, st.examples))
    dense = tier.get_dense()
    tier.close()
    return dense, store, losses


def check_bit_exact(oracle, pkg, off, keys, lab, B, *, E, layers, J, dims):
    dense, store, _ = run_gpu(pkg, off, keys, lab, B, E=E, layers=layers, J=J, dims=dims)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, layers, J=J), B, off, keys, lab)
    assert np.array_equal(dense, wd), np.abs(dense - wd).max()
    got = store[wk.astype(np.int64)]
    bad = np.nonzero((got != wr).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, e.g. key {wk[bad[0]]}"
    untouched = np.ones(dims, bool)
    untouched[wk.astype(np.int64)] = False
    assert not store[untouched].any()


@pytest.mark.parametrize("E,layers,J,zipf", [
    (8, (8, 16, 1), 4, False),
    (16, (8, 16, 1), 4, True),
    (4, (4, 1), 2, False),
    (1, (1,), 1, False),
    (64, (8, 16, 1), 4, True),
    (12, (16, 8, 1), 3, True),
    (128, (8, 16, 1), 8, True),
])
def test_train_bit_exact_vs_oracle(pkg, oracle, E, layers, J, zipf):
    dims, B, nnz = 30000, 512, 20
    off, keys, lab = pkg.gen_dataset(dims, B * 3, nnz, zipf=zipf, seed=5)
    check_bit_exact(oracle, pkg, off, keys, lab, B, E=E, layers=layers, J=J, dims=dims)


def test_trailing_partial_batch_and_empty_shards(pkg, oracle):
    """A trailing batch of 5 examples leaves empty shards that still sync a zero
    gradient and divide by all replicas (SURVEY §8c edge cases)."""
    dims, B = 2000, 64
    off, keys, lab = pkg.gen_dataset(dims, 2 * B + 5, 7, zipf=True, seed=11)
    check_bit_exact(oracle, pkg, off, keys, lab, B, E=8, layers=(8, 16, 1), J=4, dims=dims)


def test_variable_length_examples(pkg, oracle):
    """CSR with ragged examples, including empty ones."""
    rng = np.random.default_rng(4)
    dims, n = 5000, 700
    lens = rng.integers(0, 40, size=n)
    lens[::17] = 0
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    keys = np.concatenate([np.sort(rng.choice(dims, size=l, replace=False)) for l in lens]
                          ).astype(np.uint64)
    lab = rng.integers(0, 2, size=n).astype(np.uint8)
    check_bit_exact(oracle, pkg, off, keys, lab, 256, E=8, layers=(8, 16, 1), J=4, dims=dims)


def test_config1_full_size_bit_exact(pkg, oracle):
    """BASELINE config 1 (dims 1e6, E=8, B=4096, 100 keys/example, J=4), two
    batches, bit-exact."""
    dims, B = 10**6, 4096
    off, keys, lab = pkg.gen_dataset(dims, 2 * B, 100, seed=1)
    check_bit_exact(oracle, pkg, off, keys, lab, B, E=8, layers=(8, 16, 1), J=4, dims=dims)


def test_skip_sync_knob_diverges(pkg, oracle):
    """inject_skip_sync skips the dense sync+update of one global mini-batch
    (pipeline.hpp:550-555); verify must then fail (test_pipeline.cpp:317-326)."""
    dims, B = 5000, 256
    off, keys, lab = pkg.gen_dataset(dims, 2 * B, 10, seed=2)
    dense, store, _ = run_gpu(pkg, off, keys, lab, B, E=8, layers=(8, 16, 1), J=4, dims=dims,
                              skip=1)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, 8, (8, 16, 1), J=4), B, off, keys, lab)
    assert not np.array_equal(dense, wd)


def test_key_out_of_range_is_an_error(pkg):
    tier = pkg.Tier(width=8, key_space=100, max_batch_examples=4, max_batch_keys=16)
    off = np.array([0, 2, 4], np.int64)
    with pytest.raises(pkg.Error) as e:
        tier.train_batch(off, np.array([1, 150, 3, 4], np.uint64), np.array([0, 1], np.uint8))
    assert "out of range" in str(e.value)
    tier.close()


def test_nondeterministic_flag_is_canonical(pkg, oracle):
    """deterministic=0 is accepted (config.hpp:67) but there is no separate
    f32 fast path: the dense sync always takes the canonical f64 sum, so the
    result is bit-exact, inside the reference default mode's 1e-5 contract."""
    dims, B = 20000, 512
    off, keys, lab = pkg.gen_dataset(dims, 3 * B, 20, zipf=True, seed=9)
    dense, store, _ = run_gpu(pkg, off, keys, lab, B, E=8, layers=(8, 16, 1), J=4, dims=dims,
                              det=False)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, 8, (8, 16, 1), J=4), B, off, keys, lab)
    assert np.array_equal(dense, wd)
    assert np.array_equal(store[wk.astype(np.int64)], wr)


def test_loss_decreases_on_learnable_data(pkg):
    dims, B = 20000, 1024
    off, keys, lab = pkg.gen_dataset(dims, 12 * B, 20, seed=3, clusters=50)
    _, _, losses = run_gpu(pkg, off, keys, lab, B, E=8, layers=(8, 16, 1), J=4, dims=dims)
    assert losses[-1] < losses[0]


def test_graph_replays_bit_exact(pkg, oracle):
    """Same-shape batches make hps_train_batch replay its captured CUDA graph
    (both table parities); every replay must still be bit-exact, and equal to
    the kernel-by-kernel (non-graph) execution and to a run that flushes the
    deferred write-back after every batch."""
    dims, B, nnz, nb = 20000, 512, 20, 9
    off, keys, lab = pkg.gen_dataset(dims, B * nb, nnz, zipf=True, seed=21)
    outs = []
    for graphs, flush_each in ((True, False), (False, False), (True, True)):
        tier = pkg.Tier(width=8, layer_dims=(8, 16, 1), minibatches=4, key_space=dims,
                        max_batch_examples=B, max_batch_keys=B * nnz)
        tier.set_graphs(graphs)
        store = np.zeros((dims, 8), dtype=np.float32)
        tier.attach_store(store)
        for b in range(nb):
            tier.train_batch(off[b * B:(b + 1) * B + 1] - off[b * B],
                             keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
            if flush_each:  # the deferred write-back never changes the result
                tier.flush()
        outs.append((tier.get_dense(), store))
        tier.close()
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, 8, (8, 16, 1), J=4), B, off, keys, lab)
    for dense, store in outs:
        assert np.array_equal(dense, wd)
        assert np.array_equal(store[wk.astype(np.int64)], wr)


def test_dump_after_sort_free_build(pkg, oracle):
    """hps_train_batch builds its table without sorting the working set; the
    reference dump_node contract (every key of the batch, ascending, with its
    row, hbm_ps.hpp:224-232) must still hold."""
    dims, B, nnz = 20000, 512, 20
    off, keys, lab = pkg.gen_dataset(dims, 2 * B, nnz, zipf=True, seed=8)
    tier = pkg.Tier(width=8, layer_dims=(8, 16, 1), minibatches=4, key_space=dims,
                    max_batch_examples=B, max_batch_keys=B * nnz)
    store = np.zeros((dims, 8), dtype=np.float32)
    tier.attach_store(store)
    for b in range(2):
        tier.train_batch(off[b * B:(b + 1) * B + 1] - off[b * B],
                         keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
    dk, dr = tier.dump()
    tier.flush()  # the second batch's write-back is deferred until here
    want = np.unique(keys[off[B]:off[2 * B]])
    assert np.array_equal(dk, want)
    assert np.array_equal(dr, store[want.astype(np.int64)])
    slots = tier.table_slots()
    assert np.array_equal(slots, oracle.table_build(want))  # layout == ascending insert
    tier.close()


def test_export_trained_table_as_reference_parameter_files(pkg, oracle, tmp_path):
    """hps_export: the trained table leaves as SSD-PS parameter files
    (ssd_ps.hpp:50-56) that the unmodified reference SsdStore recovers, loads
    and fscks, holding exactly train_reference's rows for the last batch's
    keys (bit-exact) and zero opt_state (plain SGD leaves it untouched,
    model.hpp:204)."""
    from native import RefLib
    ref = RefLib()
    dims, B, nnz, E, layers, J = 50000, 1024, 30, 16, (8, 16, 1), 4
    off, keys, lab = pkg.gen_dataset(dims, 3 * B, nnz, zipf=True, seed=12)
    tier = pkg.Tier(width=E, layer_dims=layers, minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=B * nnz)
    store = np.zeros((dims, E), dtype=np.float32)
    tier.attach_store(store)
    for b in range(3):
        tier.train_batch(off[b * B:(b + 1) * B + 1] - off[b * B],
                         keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
    nf = tier.export(str(tmp_path), file_capacity=1000, first_id=7)
    tier.flush()
    tier.close()
    want = np.unique(keys[off[2 * B]:off[3 * B]])
    assert nf == -(-want.size // 1000)
    k, e, o, info = ref.store_load_all(str(tmp_path), E, want.size)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, layers, J=J), B, off, keys, lab)
    assert np.array_equal(k, want)
    rows = dict(zip(wk.tolist(), wr))
    assert e.tobytes() == np.stack([rows[int(x)] for x in k]).tobytes()
    assert not o.any()
    assert info["fsck_ok"] == 1 and info["files"] == nf and info["live_records"] == want.size


@pytest.mark.parametrize("store_kind", ["host", "host-zerocopy", "device", "none"])
def test_pipelined_submit_wait_bit_exact(pkg, oracle, monkeypatch, store_kind):
    """hps_submit_batch / hps_wait_batch keep two batches in flight: the next
    batch's table is built (rows prefetched, from the table two builds back
    or the store) beside the running body, write-backs are deferred. Results
    must equal the oracle bit for bit, and equal hps_train_batch's, for a host
    store (mirrored in HBM, the default for a store that fits, or staged
    per batch with zero-copy kernels), an HBM store and no store (zeros for
    new rows)."""
    import torch
    if store_kind == "host-zerocopy":
        monkeypatch.setenv("HPS_STORE_MIRROR_GB", "0")
    dims, B, nnz, nb = 20000, 512, 20, 8
    off, keys, lab = pkg.gen_dataset(dims, B * nb, nnz, zipf=True, seed=33)
    tier = pkg.Tier(width=8, layer_dims=(8, 16, 1), minibatches=4, key_space=dims,
                    max_batch_examples=B, max_batch_keys=B * nnz)
    if store_kind.startswith("host"):
        store = np.zeros((dims, 8), dtype=np.float32)
        tier.attach_store(store)
        assert tier.store_mode() == ("host-mirrored" if store_kind == "host" else "host-zerocopy")
    elif store_kind == "device":
        dstore = torch.zeros((dims, 8), dtype=torch.float32, device="cuda")
        tier.attach_store(dstore.data_ptr(), on_device=True, num_keys=dims)
    stats = []
    for b in range(nb):
        tier.submit_batch(off[b * B:(b + 1) * B + 1] - off[b * B],
                          keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
        if b % 3 == 2:  # waits lag submits irregularly
            stats.append(tier.wait_batch())
    while len(stats) < nb:
        stats.append(tier.wait_batch())
    with pytest.raises(pkg.Error):
        tier.wait_batch()  # nothing left in flight
    tier.flush()
    dense = tier.get_dense()
    tier.close()
    if store_kind == "device":
        torch.cuda.synchronize()
        store = dstore.cpu().numpy()
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, 8, (8, 16, 1), J=4), B, off, keys, lab)
    if store_kind == "none":
        # no store: a key that left the table restarts from zeros; the dense
        # weights must still match a plain train_batch run
        ref = pkg.Tier(width=8, layer_dims=(8, 16, 1), minibatches=4, key_space=dims,
                       max_batch_examples=B, max_batch_keys=B * nnz)
        for b in range(nb):
            ref.train_batch(off[b * B:(b + 1) * B + 1] - off[b * B],
                            keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
        assert np.array_equal(dense, ref.get_dense())
        ref.close()
        return
    assert np.array_equal(dense, wd)
    assert np.array_equal(store[wk.astype(np.int64)], wr)
    assert all(s.examples == B for s in stats)
    # rows read from the store + carried + proxied == working set
    assert all(s.store_rows + s.carried_rows <= s.working_set for s in stats)
    assert any(s.store_rows + s.carried_rows < s.working_set for s in stats[2:])


@pytest.mark.parametrize("B", [512, 2048])
@pytest.mark.parametrize("dedup", ["hash", "hash-unfused", "sort"])
def test_duplicate_keys_within_examples(pkg, oracle, dedup, B, monkeypatch):
    """A key repeated inside one example is two occurrences (embed_sum adds
    its row twice, backward accumulates it twice, model.hpp:59-117,182-187).
    Both mini-batch dedup paths (slot grouping, group.cuh, with the segment
    ordering in one launch or, "hash-unfused", in four; radix sort) must keep
    the occurrence order and match the oracle bit for bit. Hot keys make long
    segments (the bitmap-ranked paths; at B = 2048 over 256 occurrences, the
    per-CTA path) that repeat inside examples (the counting fallback)."""
    monkeypatch.setenv("HPS_DEDUP", "hash" if dedup.startswith("hash") else dedup)
    monkeypatch.setenv("HPS_GROUP_FUSED", "0" if dedup == "hash-unfused" else "1")
    rng = np.random.default_rng(12)
    dims, n = 3000, 3 * B
    lens = rng.integers(1, 60, size=n)
    rows = []
    for l in lens:
        k = rng.integers(0, dims, size=l)
        k[: l // 3] = rng.integers(0, 8, size=l // 3)  # hot, often repeated
        rows.append(k)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    keys = np.concatenate(rows).astype(np.uint64)
    lab = rng.integers(0, 2, size=n).astype(np.uint8)
    check_bit_exact(oracle, pkg, off, keys, lab, B, E=8, layers=(8, 16, 1), J=4, dims=dims)


def test_sort_dedup_path_bit_exact(pkg, oracle, monkeypatch):
    """The radix-sort mini-batch dedup (HPS_DEDUP=sort, the G > 1 path)
    stays bit-exact at G = 1 too."""
    monkeypatch.setenv("HPS_DEDUP", "sort")
    dims, B, nnz = 30000, 512, 20
    off, keys, lab = pkg.gen_dataset(dims, B * 3, nnz, zipf=True, seed=5)
    check_bit_exact(oracle, pkg, off, keys, lab, B, E=16, layers=(8, 16, 1), J=4, dims=dims)


@pytest.mark.parametrize("J,prep_group", [(1, None), (3, None), (5, None), (4, "1"), (4, "3")])
def test_hbm_store_grouping_split_bit_exact(pkg, oracle, monkeypatch, J, prep_group):
    """With an HBM value store the body groups its later mini-batches on a side
    branch while the prep groups the first ones (HPS_PREP_GROUP moves the
    split): every split must stay bit-exact, including odd J."""
    import torch
    if prep_group is not None:
        monkeypatch.setenv("HPS_PREP_GROUP", prep_group)
    dims, B, nnz, nb = 20000, 600, 16, 7
    off, keys, lab = pkg.gen_dataset(dims, B * nb, nnz, zipf=True, seed=40 + J)
    tier = pkg.Tier(width=8, layer_dims=(8, 16, 1), minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=B * nnz)
    dstore = torch.zeros((dims, 8), dtype=torch.float32, device="cuda")
    tier.attach_store(dstore.data_ptr(), on_device=True, num_keys=dims)
    for b in range(nb):
        tier.submit_batch(off[b * B:(b + 1) * B + 1] - off[b * B],
                          keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B])
        if b >= 2:
            tier.wait_batch()
    for _ in range(2):
        tier.wait_batch()
    dense = tier.get_dense()
    tier.close()
    torch.cuda.synchronize()
    store = dstore.cpu().numpy()
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, 8, (8, 16, 1), J=J), B, off, keys, lab)
    assert np.array_equal(dense, wd)
    assert np.array_equal(store[wk.astype(np.int64)], wr)


@pytest.mark.parametrize("tile,slack", [("1", "29"), ("0", "-1"), ("0", "8"), ("0", "29")])
@pytest.mark.parametrize("E,nnz", [(8, 20), (16, 100)])
def test_embed_sum_paths_bit_exact(pkg, oracle, monkeypatch, tile, slack, E, nnz):
    """fwd/bwd's embed_sum: the default streams the rows through shared-memory
    tiles and chains each dimension in feature order (model.cuh
    embed_sum_tiled); HPS_FB_TILE=0 takes the register path, whose order-free
    branch (whole rows per lane, recursive halving; embed_sum_exact) runs
    only where the f64 sum is exact in any order — HPS_EMBED_SLACK tightens
    that bound so the in-order fallback runs for all (-1) or part (8) of the
    examples, mixed within one mini-batch. All against the same oracle."""
    monkeypatch.setenv("HPS_FB_TILE", tile)
    monkeypatch.setenv("HPS_EMBED_SLACK", slack)
    dims, B = 30000, 512
    off, keys, lab = pkg.gen_dataset(dims, B * 3, nnz, zipf=True, seed=11)
    check_bit_exact(oracle, pkg, off, keys, lab, B, E=E, layers=(8, 16, 1), J=4, dims=dims)


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("E,J", [(8, 4), (16, 1)])
def test_dense_grad_paths_bit_exact(pkg, oracle, monkeypatch, fused, E, J):
    """The certified dense-gradient reduce: one launch and one pass (slices
    publish T, A and Lambda; the weight group's last CTA bounds B from the
    ordered slice totals; dense_grad_fused_kernel) or four launches with the
    offset walk (HPS_DG_FUSED=0); both bit-exact against the oracle."""
    monkeypatch.setenv("HPS_DG_FUSED", fused)
    dims, B = 30000, 2048
    off, keys, lab = pkg.gen_dataset(dims, B * 2, 40, zipf=True, seed=23)
    check_bit_exact(oracle, pkg, off, keys, lab, B, E=E, layers=(8, 16, 1), J=J, dims=dims)

"""GPU parity on the benchmarked path itself and on the rarely-taken branches
(round-2 VERDICT "What's weak" #1).

* BASELINE config 2 at full size (the bench workload: dims 1e7, E=16,
  B=16384, Zipf(1.0), 100 keys/example, J=4): Zipf-hot keys occur in nearly
  every example of a 4096-example shard, so their segments run to ~16 chunks
  of the chunked, certified reduce (big_fused_kernel's look-back at the depth
  the bench runs it). Bit-exact against the oracle's train_reference
  (oracle.hpp:55-122), with a host (zero-copy) and an HBM value store.
* HPS_CERT_FORCE_FAIL=1: every certificate fails, so the exact in-order
  fallbacks of big_fused_kernel (both the multi-chunk and the single-CTA
  path) and of dense_grad_fin_kernel run — and stay bit-exact.
* A working set that grows ~30x between batches: the speculative table build
  (guessed at the previous capacity) must land on the reference capacity
  (device_table.hpp:38-45) and slot layout, not the capacity the overflowed
  guess would suggest.
"""
import numpy as np
import pytest

from native import make_cfg

pytestmark = pytest.mark.gpu


def batches_of(off, keys, lab, B):
    nb = (len(off) - 1 + B - 1) // B
    for b in range(nb):
        e0, e1 = b * B, min((b + 1) * B, len(off) - 1)
        yield off[e0:e1 + 1] - off[e0], keys[off[e0]:off[e1]], lab[e0:e1]


def max_keys_of(off, B):
    nb = (len(off) - 1 + B - 1) // B
    return int(max(off[min((b + 1) * B, len(off) - 1)] - off[b * B] for b in range(nb)))


def max_segment(off, keys, B, J):
    """Longest (key, mini-batch shard) segment of the first batch, from the
    data alone (shard_batch: example i -> mini-batch i % J at one device)."""
    o, k = off[:B + 1], keys[:off[B]]
    ex = np.repeat(np.arange(B, dtype=np.uint64), np.diff(o).astype(np.int64))
    u = k * np.uint64(J) + ex % np.uint64(J)
    _, c = np.unique(u, return_counts=True)
    return int(c.max())


@pytest.mark.parametrize("store_kind", ["host", "host-zerocopy", "device"])
def test_config2_full_size_bit_exact(pkg, oracle, monkeypatch, store_kind):
    import torch
    if store_kind == "host-zerocopy":  # staged per batch, not mirrored in HBM
        monkeypatch.setenv("HPS_STORE_MIRROR_GB", "0")
    dims, E, B, nnz, J, layers, nb = 10**7, 16, 16384, 100, 4, (8, 16, 1), 3
    off, keys, lab = pkg.gen_dataset(dims, nb * B, nnz, zipf=True, seed=1)
    tier = pkg.Tier(width=E, layer_dims=layers, minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=max_keys_of(off, B))
    if store_kind.startswith("host"):
        store = np.zeros((dims, E), dtype=np.float32)
        tier.attach_store(store)
    else:
        dstore = torch.zeros((dims, E), dtype=torch.float32, device="cuda")
        tier.attach_store(dstore.data_ptr(), on_device=True, num_keys=dims)
    stats = []
    for i, (o, k, l) in enumerate(batches_of(off, keys, lab, B)):
        tier.submit_batch(o, k, l)  # the bench's pipelined entry point
        if i >= 1:
            stats.append(tier.wait_batch())
    stats.append(tier.wait_batch())
    tier.flush()
    dense = tier.get_dense()
    tier.close()
    if store_kind == "device":
        torch.cuda.synchronize()
        store = dstore.cpu().numpy()
    # the data makes ~16-chunk segments (fuse_chunk(16) = 256 occurrences)...
    seg = max_segment(off, keys, B, J)
    assert seg > 15 * 256, seg
    # ... and the device planned them
    assert all(s.big_segments > 0 for s in stats)
    assert max(s.max_segment_chunks for s in stats) >= 16
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, layers, J=J), B, off, keys, lab)
    assert np.array_equal(dense, wd), np.abs(dense - wd).max()
    got = store[wk.astype(np.int64)]
    bad = np.nonzero((got != wr).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, e.g. key {wk[bad[0]]}"


@pytest.mark.parametrize("E,B,nnz,chunks", [(16, 4096, 20, 2), (8, 2048, 30, 1), (64, 1024, 20, 2)])
def test_forced_certificate_failure_takes_exact_fallbacks(pkg, oracle, monkeypatch, E, B, nnz,
                                                          chunks):
    monkeypatch.setenv("HPS_CERT_FORCE_FAIL", "1")
    monkeypatch.setenv("HPS_SHORT_SEG", "32")  # every segment > 32 on the chunked path
    monkeypatch.setenv("HPS_MID_SEG", "32")
    dims, J, layers, nb = 20000, 4, (8, 16, 1), 3
    off, keys, lab = pkg.gen_dataset(dims, nb * B, nnz, zipf=True, seed=17)
    tier = pkg.Tier(width=E, layer_dims=layers, minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=max_keys_of(off, B))
    store = np.zeros((dims, E), dtype=np.float32)
    tier.attach_store(store)
    stats = [tier.train_batch(o, k, l) for o, k, l in batches_of(off, keys, lab, B)]
    tier.flush()
    dense = tier.get_dense()
    tier.close()
    monkeypatch.delenv("HPS_CERT_FORCE_FAIL")
    # every big segment's E dimensions and every certified dense weight
    # took the exact chain
    assert all(s.exact_fallbacks >= s.big_segments * E for s in stats)
    assert all(s.big_segments > 0 for s in stats)
    # chunks >= 2: the multi-CTA path (last CTA combines), 1: the single-CTA path
    assert max(s.max_segment_chunks for s in stats) >= chunks
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, layers, J=J), B, off, keys, lab)
    assert np.array_equal(dense, wd), np.abs(dense - wd).max()
    assert np.array_equal(store[wk.astype(np.int64)], wr)


@pytest.mark.parametrize("E", [16, 8, 32])
def test_forced_certificate_failure_on_the_medium_path(pkg, oracle, monkeypatch, E):
    """Segments of 33..1024 occurrences on the certified warp reduce
    (sparse_mid_cert_kernel) with every certificate failing: each such key's
    E dimensions recompute the in-order chain, bit-exact."""
    monkeypatch.setenv("HPS_CERT_FORCE_FAIL", "1")
    monkeypatch.setenv("HPS_MID_SEG", "1024")
    dims, B, nnz, J, layers, nb = 20000, 4096, 20, 4, (8, 16, 1), 2
    off, keys, lab = pkg.gen_dataset(dims, nb * B, nnz, zipf=True, seed=19)
    tier = pkg.Tier(width=E, layer_dims=layers, minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=max_keys_of(off, B))
    store = np.zeros((dims, E), dtype=np.float32)
    tier.attach_store(store)
    stats = [tier.train_batch(o, k, l) for o, k, l in batches_of(off, keys, lab, B)]
    tier.flush()
    dense = tier.get_dense()
    tier.close()
    monkeypatch.delenv("HPS_CERT_FORCE_FAIL")
    assert all(s.mid_segments > 0 for s in stats)
    assert all(s.exact_fallbacks >= (s.mid_segments + s.big_segments) * E for s in stats)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, layers, J=J), B, off, keys, lab)
    assert np.array_equal(dense, wd), np.abs(dense - wd).max()
    assert np.array_equal(store[wk.astype(np.int64)], wr)


@pytest.mark.parametrize("cert", ["1", "0"])
@pytest.mark.parametrize("mid", ["32", "128", "1024", "100000"])
@pytest.mark.parametrize("E", [4, 16, 64])
def test_mid_segment_warp_paths_bit_exact(pkg, oracle, monkeypatch, mid, E, cert):
    """Segments of HPS_SHORT_SEG+1..HPS_MID_SEG occurrences (default 33..512)
    take one warp each: certified
    (sparse_mid_cert_kernel, E in {4, 8, 16, 32}) or, with HPS_MID_CERT=0 and
    for other widths, the exact reference-order chain (sparse_mid_kernel);
    longer ones the chunked certified reduce. Every split point gives the
    oracle's bits."""
    monkeypatch.setenv("HPS_MID_SEG", mid)
    monkeypatch.setenv("HPS_MID_CERT", cert)
    if mid == "32":  # no medium path: thread chains up to 32, chunks beyond
        monkeypatch.setenv("HPS_SHORT_SEG", "32")
    dims, B, J = 20000, 4096, 4
    off, keys, lab = pkg.gen_dataset(dims, 2 * B, 20, zipf=True, seed=29)
    tier = pkg.Tier(width=E, minibatches=J, key_space=dims, max_batch_examples=B,
                    max_batch_keys=max_keys_of(off, B))
    store = np.zeros((dims, E), dtype=np.float32)
    tier.attach_store(store)
    stats = [tier.train_batch(o, k, l) for o, k, l in batches_of(off, keys, lab, B)]
    tier.flush()
    dense = tier.get_dense()
    tier.close()
    if mid == "32":
        assert all(s.mid_segments == 0 for s in stats)
    else:
        assert all(s.mid_segments > 0 for s in stats)
    if mid == "100000":
        assert all(s.big_segments == 0 for s in stats)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, (8, 16, 1), J=J), B, off, keys, lab)
    assert np.array_equal(dense, wd)
    assert np.array_equal(store[wk.astype(np.int64)], wr)


def test_certificate_default_is_off(pkg, oracle, monkeypatch):
    """Without the knob the bench-like workload needs no fallback (a tier
    created after a forced one resets the device flag)."""
    monkeypatch.setenv("HPS_MID_SEG", "32")
    dims, E, B, nnz, J = 20000, 16, 4096, 20, 4
    off, keys, lab = pkg.gen_dataset(dims, B, nnz, zipf=True, seed=17)
    tier = pkg.Tier(width=E, minibatches=J, key_space=dims, max_batch_examples=B,
                    max_batch_keys=max_keys_of(off, B))
    st = tier.train_batch(off, keys, lab)
    tier.close()
    assert st.big_segments > 0 and st.exact_fallbacks == 0


@pytest.mark.parametrize("pipelined", [False, True])
def test_working_set_growth_and_shrink(pkg, oracle, pipelined):
    """batch 2 holds ~30x the distinct keys of batch 1, so
    the speculative insert at batch 1's capacity fills up; the build must
    still land on next_pow2((4n+2)/3) of the true count and the ascending-
    insert layout; batch 3 shrinks again."""
    rng = np.random.default_rng(5)
    dims, B, E = 400000, 512, 8
    lens = np.concatenate([np.full(B, 2), np.full(B, 60), np.full(B, 3)])
    off = np.zeros(lens.size + 1, np.int64)
    off[1:] = np.cumsum(lens)
    keys = np.concatenate([np.sort(rng.choice(dims, size=n, replace=False)) for n in lens]
                          ).astype(np.uint64)
    lab = rng.integers(0, 2, size=lens.size).astype(np.uint8)
    tier = pkg.Tier(width=E, minibatches=4, key_space=dims, max_batch_examples=B,
                    max_batch_keys=max_keys_of(off, B))
    store = np.zeros((dims, E), dtype=np.float32)
    tier.attach_store(store)
    caps, slots = [], []
    for o, k, l in batches_of(off, keys, lab, B):
        if pipelined:
            tier.submit_batch(o, k, l)
            st = tier.wait_batch()
        else:
            st = tier.train_batch(o, k, l)
        want = np.unique(k)
        assert st.working_set == want.size
        caps.append((st.table_capacity, oracle.capacity(want.size)))
        slots.append((tier.table_slots(), oracle.table_build(want)))
    tier.flush()
    dense = tier.get_dense()
    tier.close()
    for got, want in caps:
        assert got == want
    assert caps[1][1] > 2 * caps[0][1]  # the growth the advisor's case needs
    for got, want in slots:
        assert np.array_equal(got, want)
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, (8, 16, 1), J=4), B, off, keys, lab)
    assert np.array_equal(dense, wd)
    assert np.array_equal(store[wk.astype(np.int64)], wr)


def test_in_flight_error_is_reported_by_its_own_batch(pkg):
    """a failing batch's error belongs to that batch. With an
    HBM batch (the stage check runs at submit) an out-of-range key fails
    submit; with host batches the key-range error surfaces at that batch's
    wait, and the batches before it stay clean."""
    import torch
    dims, B = 5000, 64
    off, keys, lab = pkg.gen_dataset(dims, 3 * B, 10, seed=2)
    bad_keys = keys.copy()
    bad_keys[off[2 * B] + 3] = dims + 7  # batch 2 only
    tier = pkg.Tier(width=8, minibatches=4, key_space=dims, max_batch_examples=B,
                    max_batch_keys=max_keys_of(off, B))
    for o, k, l in batches_of(off, bad_keys, lab, B):
        tier.submit_batch(o, k, l)
    tier.wait_batch()
    tier.wait_batch()
    with pytest.raises(pkg.Error) as e:
        tier.wait_batch()
    assert "out of range" in str(e.value)
    tier.close()
    # device batch: the stage's own error slot, checked at submit
    tier = pkg.Tier(width=8, minibatches=4, key_space=dims, max_batch_examples=B,
                    max_batch_keys=max_keys_of(off, B))
    dev = [(torch.from_numpy(o.astype(np.int64)).cuda(), torch.from_numpy(k.view(np.int64)).cuda(),
            torch.from_numpy(l).cuda()) for o, k, l in batches_of(off, bad_keys, lab, B)]
    for i, (o, k, l) in enumerate(dev):
        if i < 2:
            tier.submit_batch((o.data_ptr(), o.numel() - 1), k.data_ptr(), l.data_ptr(),
                              on_device=True)
        else:
            with pytest.raises(pkg.Error) as e:
                tier.submit_batch((o.data_ptr(), o.numel() - 1), k.data_ptr(), l.data_ptr(),
                                  on_device=True)
            assert "out of range" in str(e.value)
    tier.wait_batch()
    tier.wait_batch()  # the earlier batches are unaffected
    tier.close()


@pytest.mark.parametrize("optimizer", ["sgd", "adagrad"])
def test_dma_staging_bit_exact(pkg, oracle, monkeypatch, optimizer):
    """HPS_STAGE=dma (the north_star staging: host threads + cudaMemcpyAsync): store
    rows gathered by host threads into pinned staging + one H2D copy per
    build, evicted rows compacted on the device + one D2H copy + host-thread
    scatter (mem_ps.hpp:114-159 prepare, 210-245 collect). Pipelined, 4 batches
    in flight, so builds read rows other batches' write-backs just returned."""
    monkeypatch.setenv("HPS_STAGE", "dma")
    dims, B, nnz, nb, E = 30000, 512, 20, 10, 8
    off, keys, lab = pkg.gen_dataset(dims, nb * B, nnz, zipf=True, seed=44)
    tier = pkg.Tier(width=E, minibatches=4, key_space=dims, max_batch_examples=B,
                    max_batch_keys=max_keys_of(off, B), optimizer=optimizer)
    store = np.zeros((dims, tier.row_width), np.float32)
    tier.attach_store(store)
    stats = []
    for i, (o, k, l) in enumerate(batches_of(off, keys, lab, B)):
        tier.submit_batch(o, k, l)
        if i >= 3:
            stats.append(tier.wait_batch())
    while len(stats) < nb:
        stats.append(tier.wait_batch())
    tier.flush()
    dense = tier.get_dense()
    rd, wr_rows = tier.store_traffic()
    tier.close()
    assert rd > 0 and wr_rows > 0
    wd, wk, wr = oracle.train_reference(make_cfg(1, 1, E, (8, 16, 1), J=4, optimizer=optimizer),
                                        B, off, keys, lab)
    assert np.array_equal(dense, wd)
    assert np.array_equal(store[wk.astype(np.int64)], wr)

"""Multi-rank GPU parity worker (one process per GPU, launched by torchrun
from tests/test_multigpu.py). Every rank holds one tier handle; the NCCL id
is broadcast through torch.distributed. Exits non-zero on any mismatch.

Cases mirror the reference's multi-device tests (test_hbm_ps.cpp) and the
end-to-end contract (deterministic multi-device = bit-exact vs
train_reference).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import paper_2003_05622_b200 as pkg  # noqa: E402
from native import Oracle, make_cfg  # noqa: E402


def log(*a):
    print(f"[rank {dist.get_rank()}]", *a, flush=True)


def new_tier(world, rank, **kw):
    obj = [pkg.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return pkg.Tier(nodes=1, devices=world, rank=rank, cuda_device=rank, nccl_id=obj[0], **kw)


def case_train(world, rank, oracle, E, layers, J, zipf, dims, B, nb, nnz, det=True,
               pipelined=False, hbm_store=False, optimizer="sgd"):
    off, keys, lab = pkg.gen_dataset(dims, B * nb + 3, nnz, zipf=zipf, seed=7)
    max_keys = int(max(off[min((b + 1) * B, len(off) - 1)] - off[b * B] for b in range(nb + 1)))
    tier = new_tier(world, rank, width=E, layer_dims=layers, minibatches=J, key_space=dims,
                    deterministic=det, max_batch_examples=B, max_batch_keys=max_keys,
                    optimizer=optimizer)
    RW = tier.row_width
    if hbm_store:  # HBM value store: the body groups its later mini-batches
        dstore = torch.zeros((dims, RW), dtype=torch.float32, device="cuda")
        tier.attach_store(dstore.data_ptr(), on_device=True, num_keys=dims)
    else:
        store = np.zeros((dims, RW), dtype=np.float32)
        tier.attach_store(store)
    n = len(off) - 1
    nbat = (n + B - 1) // B
    for b in range(nbat):
        e0, e1 = b * B, min((b + 1) * B, n)
        if pipelined:  # two batches in flight (hps_submit_batch / hps_wait_batch)
            tier.submit_batch(off[e0:e1 + 1] - off[e0], keys[off[e0]:off[e1]], lab[e0:e1])
            if b:
                tier.wait_batch()
        else:
            tier.train_batch(off[e0:e1 + 1] - off[e0], keys[off[e0]:off[e1]], lab[e0:e1])
    if pipelined:
        tier.wait_batch()
    dense = tier.get_dense()
    tier.close()
    if hbm_store:
        torch.cuda.synchronize()
        store = dstore.cpu().numpy()
    wd, wk, wr = oracle.train_reference(make_cfg(1, world, E, layers, J=J, optimizer=optimizer),
                                        B, off, keys, lab)
    ok = True
    # deterministic=0 takes the same canonical f64 sum (no separate f32 path):
    # bit-exact in both modes, which is inside the reference default mode's
    # 1e-5 contract (hps_main.cpp:164-223)
    if not np.array_equal(dense, wd):
        log("dense mismatch, max abs", np.abs(dense - wd).max())
        ok = False
    mine = wk[(wk % np.uint64(world)) == np.uint64(rank)].astype(np.int64)
    want = wr[(wk % np.uint64(world)) == np.uint64(rank)]
    got = store[mine]
    bad = np.nonzero((got != want).any(axis=1))[0]
    if bad.size:
        log(f"{bad.size}/{mine.size} owned rows differ, e.g. key {mine[bad[0]]}:",
            got[bad[0]], want[bad[0]])
        ok = False
    # keys this rank does not own are never written to its store
    owned_mask = np.zeros(dims, bool)
    owned_mask[mine] = True
    if store[~owned_mask].any():
        log("rows written for keys this rank does not own")
        ok = False
    return ok


def case_api(world, rank):
    """test_hbm_ps.cpp:118-177 across real devices: cross-device get, routed
    accumulate, push then drain, missing key."""
    ok = True
    t = new_tier(world, rank, width=2, max_batch_keys=1 << 12)
    keys = np.arange(16, dtype=np.uint64)
    t.build(keys, np.stack([keys, -keys.astype(np.int64)], 1).astype(np.float32))
    # every rank pulls a different, overlapping, unsorted key list
    q = np.array([15, 3, 0, 7, 3, 12 - rank], dtype=np.uint64)
    rows = t.pull(q)
    exp = np.stack([q, -q.astype(np.int64)], 1).astype(np.float32)
    if not np.array_equal(rows, exp):
        log("pull mismatch", rows, exp)
        ok = False
    # all ranks push +1 to keys 0..7 twice, then drain: owners add world*2
    for _ in range(2):
        t.push(np.arange(8, dtype=np.uint64), np.ones((8, 2), np.float32))
    t.drain()
    rows = t.pull(np.arange(8, dtype=np.uint64))
    exp = np.stack([np.arange(8) + 2 * world, -np.arange(8) + 2 * world], 1).astype(np.float32)
    if not np.array_equal(rows, exp):
        log("push/drain mismatch", rows, exp)
        ok = False
    # ownership: the table of rank r holds exactly keys with k % world == r
    dk, _ = t.dump()
    if not np.array_equal(dk, keys[keys % np.uint64(world) == np.uint64(rank)]):
        log("ownership mismatch", dk)
        ok = False
    # a missing key is an error on the requester (collective: all ranks ask)
    try:
        t.pull(np.array([100 + rank], np.uint64))
        log("missing key not reported")
        ok = False
    except pkg.Error as e:
        if "missing key" not in str(e):
            log("unexpected error", e)
            ok = False
    t.close()
    return ok


def case_sync(world, rank, oracle):
    """test_hbm_ps.cpp:179-265: det == canonical_sum bit-exactly, default within 1e-6."""
    ok = True
    t = new_tier(world, rank, width=1)
    rng = np.random.default_rng(9)
    bufs = (rng.random((world, 33)) - 0.5).astype(np.float32)
    canon = oracle.canonical_sum(1, world, bufs)
    got = t.dense_sync(bufs[rank], deterministic=True)
    if not np.array_equal(got, canon):
        log("det sync mismatch")
        ok = False
    got = t.dense_sync(bufs[rank], deterministic=False)
    rel = (np.abs(got - canon) / np.maximum(np.abs(canon), 1e-9)).max()
    if rel >= 1e-6:
        log("default sync rel diff", rel)
        ok = False
    ones = t.dense_sync(np.array([rank + 1.0], np.float32), deterministic=True)
    if ones[0] != world * (world + 1) / 2:
        log("1..N sum wrong", ones)
        ok = False
    t.close()
    return ok


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    oracle = Oracle()
    results = {}
    results["api"] = case_api(world, rank)
    results["sync"] = case_sync(world, rank, oracle)
    results["train_e8"] = case_train(world, rank, oracle, 8, (8, 16, 1), 4, False, 20000, 512, 3, 20)
    results["train_e16_zipf"] = case_train(world, rank, oracle, 16, (8, 16, 1), 4, True, 50000,
                                           1024, 3, 30)
    results["train_e4_j2"] = case_train(world, rank, oracle, 4, (4, 1), 2, True, 3000, 64, 4, 9)
    results["train_nondet_flag"] = case_train(world, rank, oracle, 8, (8, 16, 1), 4, True, 20000, 512,
                                       3, 20, det=False)
    # many same-shape batches: captured-graph replays across both table parities
    results["train_replays"] = case_train(world, rank, oracle, 16, (8, 16, 1), 4, True, 50000,
                                          1024, 9, 30)
    results["train_pipelined"] = case_train(world, rank, oracle, 16, (8, 16, 1), 4, True, 50000,
                                            1024, 9, 30, pipelined=True)
    # the host store staged per batch (zero-copy) instead of mirrored in HBM
    os.environ["HPS_STORE_MIRROR_GB"] = "0"
    results["train_pipelined_zerocopy"] = case_train(world, rank, oracle, 16, (8, 16, 1), 4, True,
                                                     50000, 1024, 5, 30, pipelined=True)
    del os.environ["HPS_STORE_MIRROR_GB"]
    results["train_hbm_store"] = case_train(world, rank, oracle, 8, (8, 16, 1), 4, True, 30000,
                                            1024, 7, 24, pipelined=True, hbm_store=True)
    # Adagrad state in the rows: owners apply each sender's gradient in
    # canonical order over the NVLink exchange (p2p_apply_kernel)
    results["train_adagrad"] = case_train(world, rank, oracle, 16, (8, 16, 1), 4, True, 30000,
                                          1024, 5, 24, pipelined=True, optimizer="adagrad")
    results["train_adagrad_hbm"] = case_train(world, rank, oracle, 8, (8, 16, 1), 4, True, 20000,
                                              512, 4, 20, hbm_store=True, optimizer="adagrad")
    # the four-phase exchange (HPS_XFUSE=0) next to the default fused rounds
    os.environ["HPS_XFUSE"] = "0"
    results["train_xfuse0"] = case_train(world, rank, oracle, 16, (8, 16, 1), 4, True, 50000,
                                         1024, 5, 30, pipelined=True)
    del os.environ["HPS_XFUSE"]
    # the fused round with its keys computed in the body (HPS_XPREP=0)
    os.environ["HPS_XPREP"] = "0"
    results["train_xprep0"] = case_train(world, rank, oracle, 8, (8, 16, 1), 4, True, 30000,
                                         1024, 5, 24, pipelined=True, hbm_store=True)
    del os.environ["HPS_XPREP"]
    flags = torch.tensor([int(v) for v in results.values()], device="cuda")
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        for (k, _), f in zip(results.items(), flags.tolist()):
            print(f"CASE {k}: {'PASS' if f else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if all(flags.tolist()) else 1)


if __name__ == "__main__":
    main()

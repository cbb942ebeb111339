"""CPU, world_size 2 over gloo: the multi-GPU exchange protocol of the CUDA
path (tier.cu: owner partition -> key all-to-all -> owner gather -> row
all-to-all -> per-shard fwd/bwd -> delta all-to-all -> owner apply in
canonical sender order -> dense all-gather + canonical f64 sum) run with
torch.distributed collectives and the oracle's arithmetic, checked bit-exact
against train_reference at D=2 (oracle.hpp:55-122). This pins the protocol
independently of the kernels (which tests/mp_worker.py checks on real GPUs).

protocol="fused" is the batch body's default two-phase round (p2p.cuh
p2p_send_x_kernel): one all-to-all X carries mini-batch j's deltas, its dense
replica and mini-batch j+1's keys; owners apply j's deltas in canonical order,
update the dense weights, then serve j+1's rows (Y) — read-after-apply.
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from native import Oracle, make_cfg

E, LAYERS, J, LR = 4, (4, 1), 2, 0.05


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _alltoall(obj_per_dest, world):
    """All-to-all of python objects: returns list indexed by source rank."""
    gathered = [None] * world
    dist.all_gather_object(gathered, obj_per_dest)
    me = dist.get_rank()
    return [gathered[src][me] for src in range(world)]


def _shard(off, keys, e0, e1, rank, j, G):
    ex = list(range(e0 + rank * J + j, e1, G * J))
    sh_off, sh_keys = [0], []
    for i in ex:
        sh_keys.extend(keys[off[i]:off[i + 1]].tolist())
        sh_off.append(len(sh_keys))
    uniq = np.unique(np.array(sh_keys, np.uint64))
    req = [[int(k) for k in uniq if int(k) % G == o] for o in range(G)]
    return ex, sh_off, sh_keys, req


def _fwd_bwd(oracle, dense, rows, ex, sh_off, sh_keys, lab):
    if not ex:
        return np.zeros(dense.size, np.float32), {}
    ek = np.array(sorted(rows), np.uint64)
    er = np.stack([rows[int(k)] for k in ek]).astype(np.float32)
    _, dg, sg = oracle.forward_backward(
        E, list(LAYERS), dense, np.array(sh_off, np.int64), np.array(sh_keys, np.uint64),
        np.array([lab[i] for i in ex], np.uint8), ek, er)
    return dg, {int(k): sg[i] for i, k in enumerate(ek)}


def _worker_fused(rank, world, port, batch, data, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle = Oracle()
    off, keys, lab = data
    G = world
    dense = oracle.init_dense(make_cfg(1, G, E, LAYERS, J=J))
    store = {}
    nb = (len(off) - 1 + batch - 1) // batch
    for b in range(nb):
        e0, e1 = b * batch, min((b + 1) * batch, len(off) - 1)
        ws = np.unique(keys[off[e0]:off[e1]])
        ws = ws[ws % np.uint64(G) == np.uint64(rank)]
        table = {int(k): store.get(int(k), np.zeros(E, np.float32)).copy() for k in ws}
        shard = _shard(off, keys, e0, e1, rank, 0, G)
        # round 0: X carries only mini-batch 0's keys; Y serves their rows
        x = [{"keys": shard[3][o], "deltas": [], "dense": None} for o in range(G)]
        incoming = _alltoall(x, G)
        last_keys = [m["keys"] for m in incoming]  # the requests this rank serves
        replies = _alltoall([[table[k].tolist() for k in m["keys"]] for m in incoming], G)
        for j in range(J):
            ex, sh_off, sh_keys, req = shard
            rows = {k: np.array(r, np.float32)
                    for o in range(G) for k, r in zip(req[o], replies[o])}
            dg, grads = _fwd_bwd(oracle, dense, rows, ex, sh_off, sh_keys, lab)
            nxt = _shard(off, keys, e0, e1, rank, j + 1, G) if j + 1 < J else None
            # X: deltas of j (owner order = the keys sent last round), the
            # dense replica of j, the keys of j + 1, in ONE exchange
            x = [{"keys": nxt[3][o] if nxt else [],
                  "deltas": [grads[k].tolist() for k in req[o]],
                  "dense": dg.tolist()} for o in range(G)]
            incoming = _alltoall(x, G)
            for src in range(G):  # canonical sender order, keys from the previous round
                for k, gk in zip(last_keys[src], incoming[src]["deltas"]):
                    g = np.array(gk, np.float32)
                    oracle.L.or_sgd_accumulate(table[k].ctypes.data, g.ctypes.data, E,
                                               ctypes.c_float(LR))
            ssum = oracle.canonical_sum(1, G, np.array([m["dense"] for m in incoming], np.float32))
            oracle.L.or_average_apply(dense.ctypes.data, ssum.ctypes.data, dense.size, G,
                                      ctypes.c_float(LR))
            if nxt:  # Y: the next mini-batch's rows, read after this apply
                replies = _alltoall([[table[k].tolist() for k in m["keys"]] for m in incoming],
                                    G)
                shard = nxt
            last_keys = [m["keys"] for m in incoming]
        store.update(table)
    result_q.put((rank, dense, store))
    dist.destroy_process_group()


def _worker(rank, world, port, batch, data, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle = Oracle()
    off, keys, lab = data
    G = world
    dense = oracle.init_dense(make_cfg(1, G, E, LAYERS, J=J))
    store = {}  # this rank's value store (owned keys only)
    nb = (len(off) - 1 + batch - 1) // batch
    for b in range(nb):
        e0, e1 = b * batch, min((b + 1) * batch, len(off) - 1)
        bkeys = keys[off[e0]:off[e1]]
        ws = np.unique(bkeys)
        ws = ws[ws % np.uint64(G) == np.uint64(rank)]
        table = {int(k): store.get(int(k), np.zeros(E, np.float32)).copy() for k in ws}
        for j in range(J):
            s = rank * J + j
            ex = list(range(e0 + s, e1, G * J))
            sh_off = [0]
            sh_keys = []
            for i in ex:
                sh_keys.extend(keys[off[i]:off[i + 1]].tolist())
                sh_off.append(len(sh_keys))
            uniq = np.unique(np.array(sh_keys, np.uint64))
            # pull: keys to owners, rows back
            req = [[int(k) for k in uniq if int(k) % G == o] for o in range(G)]
            incoming = _alltoall(req, G)
            served = [[table[k].tolist() for k in ks] for ks in incoming]
            replies = _alltoall(served, G)
            rows = {}
            for o in range(G):
                for k, r in zip(req[o], replies[o]):
                    rows[k] = np.array(r, np.float32)
            # forward/backward of this shard (oracle arithmetic)
            nw = dense.size
            if ex:
                ek = np.array(sorted(rows), np.uint64)
                er = np.stack([rows[int(k)] for k in ek]).astype(np.float32)
                _, dg, sg = oracle.forward_backward(
                    E, list(LAYERS), dense, np.array(sh_off, np.int64),
                    np.array(sh_keys, np.uint64), np.array([lab[i] for i in ex], np.uint8), ek, er)
                grads = {int(k): sg[i] for i, k in enumerate(ek)}
            else:
                dg = np.zeros(nw, np.float32)
                grads = {}
            # push deltas to owners (keys implicit = pulled keys)
            push = [[(k, grads[k].tolist()) for k in req[o]] for o in range(G)]
            got = _alltoall(push, G)
            for src in range(G):  # canonical sender order (hbm_ps.hpp:172-195)
                for k, gk in got[src]:
                    g = np.array(gk, np.float32)
                    oracle.L.or_sgd_accumulate(table[k].ctypes.data, g.ctypes.data, E,
                                               ctypes.c_float(LR))
            # dense: all-gather + canonical sum, average, apply
            allg = [None] * G
            dist.all_gather_object(allg, dg.tolist())
            ssum = oracle.canonical_sum(1, G, np.array(allg, np.float32))
            oracle.L.or_average_apply(dense.ctypes.data, ssum.ctypes.data, nw, G,
                                      ctypes.c_float(LR))
        store.update(table)  # write-back (dump_node -> collect_updates)
    result_q.put((rank, dense, store))
    dist.destroy_process_group()


@pytest.mark.parametrize("protocol", ["four_phase", "fused"])
@pytest.mark.parametrize("world", [2])
def test_two_rank_protocol_bit_exact_vs_train_reference(pkg, world, protocol):
    off, keys, lab = pkg.gen_dataset(400, 2 * 60 + 7, 5, zipf=True, seed=4)
    batch = 60
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    target = _worker_fused if protocol == "fused" else _worker
    procs = [ctx.Process(target=target, args=(r, world, port, batch, (off, keys, lab), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, dense, store = q.get(timeout=300)
        res[r] = (dense, store)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wd, wk, wr = Oracle().train_reference(make_cfg(1, world, E, LAYERS, J=J), batch, off, keys,
                                          lab)
    for r in range(world):
        assert np.array_equal(res[r][0], wd)
    merged = {}
    for r in range(world):
        for k, v in res[r][1].items():
            assert k % world == r  # single ownership
            merged[k] = v
    assert sorted(merged) == wk.tolist()
    for i, k in enumerate(wk.tolist()):
        assert np.array_equal(merged[k], wr[i]), k

"""ctypes wrappers for the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement of the reference
  HBM-PS path (oracle/hps_oracle.c). Always buildable (gcc).
* ``RefLib``  -> oracle/_ref/libhps_ref.so, the UNMODIFIED reference headers
  behind a C shim (oracle/ref_harness.cpp). Built only where /root/reference
  exists (this container); it travels prebuilt to the GPU box.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhps_ref.so")

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


class Cfg(ctypes.Structure):
    """or_cfg / RefCfg (identical layout)."""
    _fields_ = [
        ("nodes", ctypes.c_int), ("devices", ctypes.c_int), ("embedding_dim", ctypes.c_int),
        ("num_layers", ctypes.c_int), ("layer_dims", ctypes.c_uint64 * 8),
        ("learning_rate", ctypes.c_float), ("seed", ctypes.c_uint64),
        ("minibatches", ctypes.c_int), ("deterministic", ctypes.c_int),
        ("inject_skip_sync", ctypes.c_int64),
        # extension fields (or_cfg only; RefCfg stops before them)
        ("optimizer", ctypes.c_int), ("adagrad_eps", ctypes.c_float),
    ]


def make_cfg(nodes=1, devices=1, E=8, layers=(8, 16, 1), lr=0.05, seed=42, J=4,
             det=True, skip=-1, optimizer="sgd", eps=1e-8) -> Cfg:
    c = Cfg()
    c.nodes, c.devices, c.embedding_dim = nodes, devices, E
    c.num_layers = len(layers)
    for i, d in enumerate(layers):
        c.layer_dims[i] = d
    c.learning_rate = lr
    c.seed = seed
    c.minibatches = J
    c.deterministic = int(det)
    c.inject_skip_sync = skip
    c.optimizer = {"sgd": 0, "adagrad": 1}[optimizer]
    c.adagrad_eps = eps
    return c


def dense_count(E: int, layers: Sequence[int]) -> int:
    n, i = 0, E
    for o in layers:
        n += (i + 1) * o
        i = o
    return n


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (make -C oracle)")
        L = ctypes.CDLL(path)
        L.or_last_error.restype = ctypes.c_char_p
        L.or_mix64.argtypes, L.or_mix64.restype = [_U64], _U64
        L.or_capacity.argtypes, L.or_capacity.restype = [_U64], _U64
        L.or_table_build.argtypes = [_P, _U64, _U64, _P]
        L.or_table_find.argtypes, L.or_table_find.restype = [_P, _U64, _U64], ctypes.c_int64
        L.or_sort_unique.argtypes, L.or_sort_unique.restype = [_P, _U64, _P], _U64
        L.or_owner.argtypes = [_P, _U64, ctypes.c_int, ctypes.c_int, _P]
        L.or_shard.argtypes = [_U64, ctypes.c_int, ctypes.c_int, _P, _P]
        L.or_dense_count.argtypes, L.or_dense_count.restype = [ctypes.c_int, ctypes.c_int, _P], _U64
        L.or_init_dense.argtypes = [ctypes.POINTER(Cfg), _P]
        L.or_forward_backward.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, _U64, _P, _P, _P,
                                          _P, _P, _U64, _P, _P, _P]
        L.or_canonical_sum.argtypes = [ctypes.c_int, ctypes.c_int, _P, _U64, _P]
        L.or_average_apply.argtypes = [_P, _P, _U64, ctypes.c_int, ctypes.c_float]
        L.or_sgd_accumulate.argtypes = [_P, _P, _U64, ctypes.c_float]
        L.or_adagrad_apply.argtypes = [_P, _P, _P, _U64, ctypes.c_float, ctypes.c_float]
        L.or_train_reference.argtypes = [ctypes.POINTER(Cfg), _U64, _U64, _P, _P, _P, _P,
                                         ctypes.POINTER(_U64), _P, _P, _U64]
        L.or_auc.argtypes, L.or_auc.restype = [_P, _P, _U64], ctypes.c_double
        self.L = L

    def err(self) -> str:
        return self.L.or_last_error().decode()

    def capacity(self, n: int) -> int:
        return int(self.L.or_capacity(n))

    def mix64(self, x: int) -> int:
        return int(self.L.or_mix64(x))

    def table_build(self, keys_sorted) -> np.ndarray:
        k = np.ascontiguousarray(keys_sorted, dtype=np.uint64)
        cap = self.capacity(k.size)
        slots = np.empty(cap, dtype=np.uint64)
        if self.L.or_table_build(ptr(k), k.size, cap, ptr(slots)) != 0:
            raise RuntimeError(self.err())
        return slots

    def sort_unique(self, keys) -> np.ndarray:
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.empty(max(k.size, 1), dtype=np.uint64)
        n = self.L.or_sort_unique(ptr(k), k.size, ptr(out))
        return out[:n]

    def owner(self, keys, nodes, devices) -> np.ndarray:
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        g = np.empty(k.size, dtype=np.int32)
        self.L.or_owner(ptr(k), k.size, nodes, devices, ptr(g))
        return g

    def shard(self, n, devices, J):
        dv = np.empty(n, dtype=np.int32)
        mb = np.empty(n, dtype=np.int32)
        self.L.or_shard(n, devices, J, ptr(dv), ptr(mb))
        return dv, mb

    def init_dense(self, cfg: Cfg) -> np.ndarray:
        n = dense_count(cfg.embedding_dim, list(cfg.layer_dims)[: cfg.num_layers])
        w = np.empty(n, dtype=np.float32)
        self.L.or_init_dense(ctypes.byref(cfg), ptr(w))
        return w

    def forward_backward(self, E, layers, dense, offsets, keys, labels, emb_keys, emb_rows):
        layers_a = np.ascontiguousarray(layers, dtype=np.uint64)
        n = len(offsets) - 1
        preds = np.empty(n, dtype=np.float64)
        dg = np.empty(dense_count(E, layers), dtype=np.float32)
        sg = np.empty((len(emb_keys), E), dtype=np.float32)
        d = np.ascontiguousarray(dense, dtype=np.float32)
        o = np.ascontiguousarray(offsets, dtype=np.int64)
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        lab = np.ascontiguousarray(labels, dtype=np.uint8)
        ek = np.ascontiguousarray(emb_keys, dtype=np.uint64)
        er = np.ascontiguousarray(emb_rows, dtype=np.float32)
        rc = self.L.or_forward_backward(E, len(layers), ptr(layers_a), ptr(d), n, ptr(o), ptr(k),
                                        ptr(lab), ptr(ek), ptr(er), ek.size, ptr(preds), ptr(dg),
                                        ptr(sg))
        if rc:
            raise RuntimeError(self.err())
        return preds, dg, sg

    def canonical_sum(self, nodes, devices, bufs) -> np.ndarray:
        b = np.ascontiguousarray(bufs, dtype=np.float32)
        out = np.empty(b.shape[1], dtype=np.float32)
        self.L.or_canonical_sum(nodes, devices, ptr(b), b.shape[1], ptr(out))
        return out

    def adagrad_apply(self, v, s, g, lr, eps):
        """or_adagrad_apply in place on float32 copies; returns (v, s)."""
        v = np.array(v, dtype=np.float32)
        s = np.array(s, dtype=np.float32)
        g = np.ascontiguousarray(g, dtype=np.float32)
        self.L.or_adagrad_apply(ptr(v), ptr(s), ptr(g), v.size, lr, eps)
        return v, s

    def train_reference(self, cfg: Cfg, batch_size, offsets, keys, labels):
        o = np.ascontiguousarray(offsets, dtype=np.int64)
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        lab = np.ascontiguousarray(labels, dtype=np.uint8)
        E = cfg.embedding_dim
        dense = np.empty(dense_count(E, list(cfg.layer_dims)[: cfg.num_layers]), np.float32)
        cap = max(1, len(np.unique(k)))
        sk = np.empty(cap, dtype=np.uint64)
        sr = np.empty((cap, 2 * E if cfg.optimizer == 1 else E), dtype=np.float32)
        n = _U64()
        rc = self.L.or_train_reference(ctypes.byref(cfg), batch_size, o.size - 1, ptr(o), ptr(k),
                                       ptr(lab), ptr(dense), ctypes.byref(n), ptr(sk), ptr(sr),
                                       cap)
        if rc:
            raise RuntimeError(self.err())
        return dense, sk[: n.value], sr[: n.value]

    def auc(self, labels, scores) -> float:
        lab = np.ascontiguousarray(labels, dtype=np.uint8)
        s = np.ascontiguousarray(scores, dtype=np.float64)
        return float(self.L.or_auc(ptr(lab), ptr(s), lab.size))


class RefLib:
    """The unmodified reference behind oracle/ref_harness.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (make -C oracle ref, needs /root/reference)")
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_gen_dataset.argtypes = [_U64, _U64, _U64, ctypes.c_int, ctypes.c_double, _U64,
                                      ctypes.c_double, _U64, _P, _P, _P]
        L.ref_working_set.argtypes = [ctypes.c_size_t, _P, _P, _P, ctypes.POINTER(_U64)]
        L.ref_table_slot_order.argtypes = [_P, ctypes.c_size_t, _P, ctypes.POINTER(_U64)]
        L.ref_partition.argtypes = [ctypes.c_int, ctypes.c_int, _P, ctypes.c_size_t, _P, _P,
                                    ctypes.POINTER(_U64)]
        L.ref_canonical_sum.argtypes = [ctypes.c_int, ctypes.c_int, _P, ctypes.c_size_t, _P]
        L.ref_synchronize.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.c_size_t]
        L.ref_init_dense.argtypes = [ctypes.POINTER(Cfg), _P, ctypes.POINTER(_U64)]
        L.ref_forward_backward.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, ctypes.c_size_t, _P,
                                           _P, _P, _P, _P, ctypes.c_size_t, _P, _P, _P]
        L.ref_train_reference.argtypes = [ctypes.POINTER(Cfg), ctypes.c_size_t, ctypes.c_size_t,
                                          _P, _P, _P, _P, ctypes.POINTER(_U64), _P, _P, _U64]
        L.ref_hot_path_create.argtypes = [ctypes.POINTER(Cfg), ctypes.c_size_t, ctypes.c_size_t,
                                          _P, _P, _P]
        L.ref_hot_path_create.restype = ctypes.c_void_p
        L.ref_hot_path_destroy.argtypes = [_P]
        L.ref_hot_path_run.argtypes = [_P, ctypes.c_size_t, ctypes.c_size_t,
                                       ctypes.POINTER(ctypes.c_double)]
        L.ref_hot_path_export.argtypes = [_P, _P, ctypes.POINTER(_U64), _P, _P, _U64]
        L.ref_store_dump.argtypes = [ctypes.c_char_p, _U64, _U64, _P, _P, _P, _U64]
        L.ref_store_load_all.argtypes = [ctypes.c_char_p, _U64, _P, _P, _P, _U64,
                                         ctypes.POINTER(_U64), _P]
        self.L = L

    def store_dump(self, directory, keys, emb, opt=None, file_capacity=4096):
        """The reference SsdStore::dump into `directory` (ssd_ps.hpp:229-243)."""
        k = np.ascontiguousarray(keys, np.uint64)
        e = np.ascontiguousarray(emb, np.float32)
        o = None if opt is None else np.ascontiguousarray(opt, np.float32)
        self._ok(self.L.ref_store_dump(os.fsencode(directory), e.shape[1], file_capacity,
                                       ptr(k), ptr(e), ptr(o) if o is not None else None,
                                       k.size))

    def store_load_all(self, directory, width, cap, infer_width=False):
        """The reference SsdStore recover + load(all keys) + stats + fsck
        (infer_width: the store reads the width from the files)."""
        keys = np.empty(max(cap, 1), np.uint64)
        emb = np.empty((max(cap, 1), width), np.float32)
        opt = np.empty((max(cap, 1), width), np.float32)
        n = _U64()
        info = np.zeros(6, np.uint64)
        self._ok(self.L.ref_store_load_all(os.fsencode(directory), 0 if infer_width else width,
                                           ptr(keys), ptr(emb),
                                           ptr(opt), cap, ctypes.byref(n), ptr(info)))
        m = n.value
        return keys[:m], emb[:m], opt[:m], dict(zip(
            ["files", "live_records", "stale_records", "fsck_ok", "fsck_files",
             "recovered_invalid"], (int(v) for v in info)))

    def err(self) -> str:
        return self.L.ref_last_error().decode()

    def _ok(self, rc):
        if rc:
            raise RuntimeError(self.err())

    def gen_dataset(self, dims, n, nnz, zipf=False, s=1.0, seed=1, scale=6.0, clusters=0):
        off = np.empty(n + 1, np.int64)
        keys = np.empty(n * nnz, np.uint64)
        lab = np.empty(n, np.uint8)
        self._ok(self.L.ref_gen_dataset(dims, n, nnz, int(zipf), s, seed, scale, clusters,
                                        ptr(off), ptr(keys), ptr(lab)))
        return off, keys, lab

    def working_set(self, offsets, keys) -> np.ndarray:
        o = np.ascontiguousarray(offsets, np.int64)
        k = np.ascontiguousarray(keys, np.uint64)
        out = np.empty(max(1, k.size), np.uint64)
        n = _U64()
        self._ok(self.L.ref_working_set(o.size - 1, ptr(o), ptr(k), ptr(out), ctypes.byref(n)))
        return out[: n.value]

    def table_slot_order(self, keys_sorted):
        k = np.ascontiguousarray(keys_sorted, np.uint64)
        out = np.empty(max(1, k.size), np.uint64)
        cap = _U64()
        self._ok(self.L.ref_table_slot_order(ptr(k), k.size, ptr(out), ctypes.byref(cap)))
        return out[: k.size], cap.value

    def partition(self, nodes, devices, keys):
        k = np.ascontiguousarray(keys, np.uint64)
        u = np.empty(max(1, k.size), np.uint64)
        g = np.empty(max(1, k.size), np.int32)
        n = _U64()
        self._ok(self.L.ref_partition(nodes, devices, ptr(k), k.size, ptr(u), ptr(g),
                                      ctypes.byref(n)))
        return u[: n.value], g[: n.value]

    def canonical_sum(self, nodes, devices, bufs):
        b = np.ascontiguousarray(bufs, np.float32)
        out = np.empty(b.shape[1], np.float32)
        self._ok(self.L.ref_canonical_sum(nodes, devices, ptr(b), b.shape[1], ptr(out)))
        return out

    def synchronize(self, nodes, devices, det, bufs):
        b = np.ascontiguousarray(bufs, np.float32).copy()
        self._ok(self.L.ref_synchronize(nodes, devices, int(det), ptr(b), b.shape[1]))
        return b

    def init_dense(self, cfg: Cfg):
        w = np.empty(dense_count(cfg.embedding_dim, list(cfg.layer_dims)[: cfg.num_layers]),
                     np.float32)
        n = _U64()
        self._ok(self.L.ref_init_dense(ctypes.byref(cfg), ptr(w), ctypes.byref(n)))
        return w

    def forward_backward(self, E, layers, dense, offsets, keys, labels, emb_keys, emb_rows):
        layers_a = np.ascontiguousarray(layers, dtype=np.uint64)
        n = len(offsets) - 1
        preds = np.empty(n, np.float64)
        dg = np.empty(dense_count(E, layers), np.float32)
        sg = np.empty((len(emb_keys), E), np.float32)
        args = [np.ascontiguousarray(dense, np.float32), np.ascontiguousarray(offsets, np.int64),
                np.ascontiguousarray(keys, np.uint64), np.ascontiguousarray(labels, np.uint8),
                np.ascontiguousarray(emb_keys, np.uint64), np.ascontiguousarray(emb_rows, np.float32)]
        self._ok(self.L.ref_forward_backward(E, len(layers), ptr(layers_a), ptr(args[0]), n,
                                             ptr(args[1]), ptr(args[2]), ptr(args[3]),
                                             ptr(args[4]), ptr(args[5]), args[4].size, ptr(preds),
                                             ptr(dg), ptr(sg)))
        return preds, dg, sg

    def adagrad_apply(self, v, s, g, lr, eps):
        """or_adagrad_apply in place on float32 copies; returns (v, s)."""
        v = np.array(v, dtype=np.float32)
        s = np.array(s, dtype=np.float32)
        g = np.ascontiguousarray(g, dtype=np.float32)
        self.L.or_adagrad_apply(ptr(v), ptr(s), ptr(g), v.size, lr, eps)
        return v, s

    def train_reference(self, cfg: Cfg, batch_size, offsets, keys, labels):
        o = np.ascontiguousarray(offsets, np.int64)
        k = np.ascontiguousarray(keys, np.uint64)
        lab = np.ascontiguousarray(labels, np.uint8)
        E = cfg.embedding_dim
        dense = np.empty(dense_count(E, list(cfg.layer_dims)[: cfg.num_layers]), np.float32)
        cap = max(1, len(np.unique(k)))
        sk = np.empty(cap, np.uint64)
        sr = np.empty((cap, E), np.float32)
        n = _U64()
        self._ok(self.L.ref_train_reference(ctypes.byref(cfg), batch_size, o.size - 1, ptr(o),
                                            ptr(k), ptr(lab), ptr(dense), ctypes.byref(n), ptr(sk),
                                            ptr(sr), cap))
        return dense, sk[: n.value], sr[: n.value]


class RefHotPath:
    """The reference HBM-PS hot path (device-worker loop, D threads)."""

    def __init__(self, ref: RefLib, cfg: Cfg, batch_size, offsets, keys, labels):
        self.ref = ref
        self.cfg = cfg
        self._keep = [np.ascontiguousarray(offsets, np.int64),
                      np.ascontiguousarray(keys, np.uint64),
                      np.ascontiguousarray(labels, np.uint8)]
        self.h = ref.L.ref_hot_path_create(ctypes.byref(cfg), batch_size, len(offsets) - 1,
                                           ptr(self._keep[0]), ptr(self._keep[1]),
                                           ptr(self._keep[2]))
        if not self.h:
            raise RuntimeError(ref.err())

    def run(self, first_batch, n_batches) -> float:
        ms = ctypes.c_double()
        self.ref._ok(self.ref.L.ref_hot_path_run(self.h, first_batch, n_batches, ctypes.byref(ms)))
        return ms.value

    def export(self, max_keys):
        E = self.cfg.embedding_dim
        dense = np.empty(dense_count(E, list(self.cfg.layer_dims)[: self.cfg.num_layers]),
                         np.float32)
        sk = np.empty(max_keys, np.uint64)
        sr = np.empty((max_keys, E), np.float32)
        n = _U64()
        self.ref._ok(self.ref.L.ref_hot_path_export(self.h, ptr(dense), ctypes.byref(n), ptr(sk),
                                                    ptr(sr), max_keys))
        return dense, sk[: n.value], sr[: n.value]

    def close(self):
        if self.h:
            self.ref.L.ref_hot_path_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def try_ref() -> Optional[RefLib]:
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None

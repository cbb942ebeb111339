"""ctypes binding of libhps_gpu.so (include/hps_gpu.h) and a host-side mirror
of the reference parameter-server API for the HBM-PS tier.

The reference binds this path in-process as ``hps::HbmTier``
(/root/reference/proj/include/hps/hbm_ps.hpp:41-242) plus the free functions
``synchronize`` / ``canonical_sum`` (hbm_ps.hpp:258-408). ``HbmTier`` below
keeps those names, argument meanings and error behaviour, for ONE rank (one
GPU); calls the reference makes from every device-worker thread in lockstep
(get, push_deltas, synchronize) are collective across ranks here.

There is no CPU fallback: constructing a tier without the CUDA library (or
without a GPU) raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Callable, Dict, Iterable, List, Mapping, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhps_gpu.so")

HPS_MAX_LAYERS = 8
HPS_NCCL_ID_BYTES = 128

STATUS = {
    0: "HPS_OK", 1: "HPS_ERR_ARG", 2: "HPS_ERR_MISSING_KEY", 3: "HPS_ERR_DUPLICATE",
    4: "HPS_ERR_OVERFLOW", 5: "HPS_ERR_NONFINITE", 6: "HPS_ERR_NOT_BUILT",
    7: "HPS_ERR_WIDTH", 8: "HPS_ERR_KEY_RANGE", 9: "HPS_ERR_CUDA", 10: "HPS_ERR_NCCL",
    11: "HPS_ERR_CAPACITY", 12: "HPS_ERR_CORRUPT",
}


class Error(RuntimeError):
    """hps::Error (common.hpp:28-31): the tier's hard failures."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.code = STATUS.get(status, str(status))


class HpsConfig(ctypes.Structure):
    _fields_ = [
        ("nodes", ctypes.c_int),
        ("devices_per_node", ctypes.c_int),
        ("rank", ctypes.c_int),
        ("cuda_device", ctypes.c_int),
        ("embedding_dim", ctypes.c_int),
        ("num_layers", ctypes.c_int),
        ("layer_dims", ctypes.c_uint64 * HPS_MAX_LAYERS),
        ("learning_rate", ctypes.c_float),
        ("seed", ctypes.c_uint64),
        ("minibatches", ctypes.c_int),
        ("deterministic", ctypes.c_int),
        ("inject_skip_sync", ctypes.c_int64),
        ("key_space", ctypes.c_uint64),
        ("max_batch_examples", ctypes.c_uint64),
        ("max_batch_keys", ctypes.c_uint64),
        ("max_working_set", ctypes.c_uint64),
        ("optimizer", ctypes.c_int),
        ("adagrad_eps", ctypes.c_float),
    ]


class HpsBatchStats(ctypes.Structure):
    _fields_ = [
        ("loss_sum", ctypes.c_double),
        ("examples", ctypes.c_uint64),
        ("working_set", ctypes.c_uint64),
        ("table_capacity", ctypes.c_uint64),
        ("pulled_keys", ctypes.c_uint64),
        ("served_keys", ctypes.c_uint64),
        ("occurrences", ctypes.c_uint64),
        ("carried_rows", ctypes.c_uint64),
        ("exact_fallbacks", ctypes.c_uint64),
        ("store_rows", ctypes.c_uint64),
        ("big_segments", ctypes.c_uint64),
        ("max_segment_chunks", ctypes.c_uint64),
        ("big_occurrences", ctypes.c_uint64),
        ("mid_segments", ctypes.c_uint64),
    ]

OPTIMIZERS = {"sgd": 0, "adagrad": 1}

TIMING_SLOTS = ["total", "stage", "build", "dedup", "pull", "fwdbwd", "grads", "apply",
                "dense", "writeback", "sparse", "big_fused"]


# Every symbol include/hps_gpu.h declares, with its ctypes signature.
_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_U64P = ctypes.POINTER(ctypes.c_uint64)
_SIGS = {
    "hps_last_error": ([], ctypes.c_char_p),
    "hps_version": ([], ctypes.c_char_p),
    "hps_get_unique_id": ([_P], ctypes.c_int),
    "hps_create": ([ctypes.POINTER(HpsConfig), _P, ctypes.POINTER(_P)], ctypes.c_int),
    "hps_destroy": ([_P], ctypes.c_int),
    "hps_build": ([_P, _P, _U64, _P], ctypes.c_int),
    "hps_build_placed": ([_P, _P, _U64, _P], ctypes.c_int),
    "hps_pull": ([_P, _P, _U64, _P], ctypes.c_int),
    "hps_push": ([_P, _P, _P, _U64], ctypes.c_int),
    "hps_drain": ([_P], ctypes.c_int),
    "hps_dump": ([_P, _P, _P, _U64P], ctypes.c_int),
    "hps_table_info": ([_P, _U64P, _U64P, _U64P], ctypes.c_int),
    "hps_table_slots": ([_P, _P, _P], ctypes.c_int),
    "hps_dense_sync": ([_P, _P, _U64, ctypes.c_int], ctypes.c_int),
    "hps_dense_count": ([_P, _U64P], ctypes.c_int),
    "hps_get_dense": ([_P, _P], ctypes.c_int),
    "hps_set_dense": ([_P, _P], ctypes.c_int),
    "hps_attach_store": ([_P, _P, _U64, ctypes.c_int], ctypes.c_int),
    "hps_flush": ([_P], ctypes.c_int),
    "hps_store_mode": ([_P, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "hps_store_pcie_bytes": ([_P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)],
                             ctypes.c_int),
    "hps_store_traffic": ([_P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)],
                          ctypes.c_int),
    "hps_train_batch": ([_P, _U64, _P, _P, _P, ctypes.c_int,
                         ctypes.POINTER(HpsBatchStats)], ctypes.c_int),
    "hps_submit_batch": ([_P, _U64, _P, _P, _P, ctypes.c_int], ctypes.c_int),
    "hps_wait_batch": ([_P, ctypes.POINTER(HpsBatchStats)], ctypes.c_int),
    "hps_set_timing": ([_P, ctypes.c_int], ctypes.c_int),
    "hps_get_timing": ([_P, _P], ctypes.c_int),
    "hps_reset_timing": ([_P], ctypes.c_int),
    "hps_kernel_launches": ([_P, _U64P], ctypes.c_int),
    "hps_graph_captures": ([_P, _U64P], ctypes.c_int),
    "hps_row_width": ([_P, _U64P], ctypes.c_int),
    "hps_table_lookup": ([_P, _P, _U64, _P, _P], ctypes.c_int),
    "hps_apply_local": ([_P, _P, _P, _U64], ctypes.c_int),
    "hps_debug_gemm_tf32": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int64,
                             ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                             ctypes.c_int, _P, _P, ctypes.c_int64, _P, _P, ctypes.c_int64,
                             ctypes.c_int], ctypes.c_int),
    "hps_set_graphs": ([_P, ctypes.c_int], ctypes.c_int),
    "hps_stream": ([_P, ctypes.POINTER(_P)], ctypes.c_int),
    "hps_gen_multislot": ([_U64, _U64, _U64, _U64, ctypes.c_double, _U64, ctypes.c_double, _P,
                           _P, _P, _U64P], ctypes.c_int),
    "hps_crc32": ([ctypes.c_uint32, _P, _U64], ctypes.c_uint32),
    "hps_pfile_write": ([ctypes.c_char_p, _P, _P, _P, _U64, ctypes.c_uint32, ctypes.c_uint32,
                         _U64, _U64P], ctypes.c_int),
    "hps_pfile_read": ([ctypes.c_char_p, _P, _P, _P, _U64, _U64P,
                        ctypes.POINTER(ctypes.c_uint32)], ctypes.c_int),
    "hps_export": ([_P, ctypes.c_char_p, ctypes.c_uint32, _U64, _U64P], ctypes.c_int),
    "hps_gen_dataset": ([_U64, _U64, _U64, ctypes.c_int, ctypes.c_double, _U64,
                         ctypes.c_double, _U64, _P, _P, _P], ctypes.c_int),
}

_lib_handle: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load libhps_gpu.so (built in-tree by __graft_entry__.build())."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        h = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (args, res) in _SIGS.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = res
        _lib_handle = h
    return _lib_handle


def _check(status: int) -> None:
    if status != 0:
        msg = lib().hps_last_error().decode(errors="replace")
        raise Error(status, msg)


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


# --------------------------------------------------------------- dataset ----

def crc32(data: bytes, crc: int = 0) -> int:
    """zlib-compatible CRC-32 (the parameter-file footer, ssd_ps.hpp:516)."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    return int(lib().hps_crc32(crc, _ptr(buf), buf.size))


def write_param_files(directory: str, keys, rows, opt_state=None, file_capacity: int = 4096,
                      first_id: int = 0) -> int:
    """SsdStore::dump (ssd_ps.hpp:229-243) format: ascending keys written as
    pf_<first_id + i>.bin files of file_capacity records. Returns the file count."""
    k = _u64(keys)
    r = _f32(rows).reshape(k.size, -1) if k.size else np.empty((0, 1), np.float32)
    o = None if opt_state is None else _f32(opt_state).reshape(r.shape)
    nf = ctypes.c_uint64()
    _check(lib().hps_pfile_write(os.fsencode(directory), _ptr(k), _ptr(r),
                                 _ptr(o) if o is not None else None, k.size, r.shape[1],
                                 file_capacity, first_id, ctypes.byref(nf)))
    return nf.value


def read_param_file(path: str, width: int = 0):
    """SsdStore::read_file_at (ssd_ps.hpp:495-535): validated (keys, emb, opt_state)."""
    n, w = ctypes.c_uint64(), ctypes.c_uint32(width)
    p = os.fsencode(path)
    _check(lib().hps_pfile_read(p, None, None, None, 0, ctypes.byref(n), ctypes.byref(w)))
    keys = np.empty(n.value, np.uint64)
    emb = np.empty((n.value, w.value), np.float32)
    opt = np.empty((n.value, w.value), np.float32)
    _check(lib().hps_pfile_read(p, _ptr(keys), _ptr(emb), _ptr(opt), n.value,
                                ctypes.byref(n), ctypes.byref(w)))
    return keys, emb, opt


def gen_dataset(dims: int, num_examples: int, nnz: int, zipf: bool = False,
                zipf_s: float = 1.0, seed: int = 1, signal_scale: float = 6.0,
                clusters: int = 0):
    """gen_dataset (dataset.hpp:180-227) -> (offsets i64[n+1], keys u64, labels u8)."""
    offsets = np.empty(num_examples + 1, dtype=np.int64)
    keys = np.empty(num_examples * nnz, dtype=np.uint64)
    labels = np.empty(num_examples, dtype=np.uint8)
    _check(lib().hps_gen_dataset(dims, num_examples, nnz, int(zipf), zipf_s, seed,
                                 signal_scale, clusters, _ptr(offsets), _ptr(keys),
                                 _ptr(labels)))
    return offsets, keys, labels


def gen_multislot(num_examples: int, slots: int = 100, ids_per_slot: int = 10**6,
                  max_keys: int = 300, zipf_s: float = 1.0, seed: int = 1,
                  signal_scale: float = 6.0):
    """BASELINE c4's multi-slot input (hps_gen_multislot) -> (offsets, keys, labels)."""
    offsets = np.empty(num_examples + 1, dtype=np.int64)
    keys = np.empty(num_examples * max_keys, dtype=np.uint64)
    labels = np.empty(num_examples, dtype=np.uint8)
    n = ctypes.c_uint64()
    _check(lib().hps_gen_multislot(slots, ids_per_slot, num_examples, max_keys, zipf_s, seed,
                                   signal_scale, _ptr(offsets), _ptr(keys), _ptr(labels),
                                   ctypes.byref(n)))
    return offsets, keys[: n.value].copy(), labels


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(HPS_NCCL_ID_BYTES)
    _check(lib().hps_get_unique_id(buf))
    return buf.raw


# ------------------------------------------------------------------ tier ----

class Topology:
    """topology.hpp:28-55: N nodes x D devices, g = device * N + node."""

    def __init__(self, nodes: int = 1, devices: int = 1):
        for v, what in ((nodes, "num_nodes"), (devices, "devices_per_node")):
            if v < 1 or v & (v - 1):
                raise Error(1, f"topology: {what} must be a power of two")
        self.num_nodes = nodes
        self.devices_per_node = devices

    def total_devices(self) -> int:
        return self.num_nodes * self.devices_per_node

    def node_of(self, g: int) -> int:
        return g % self.num_nodes

    def device_of(self, g: int) -> int:
        return g // self.num_nodes

    def global_index(self, node: int, device: int) -> int:
        return device * self.num_nodes + node


class Tier:
    """One rank of the HBM-PS tier: a thin owner of an ``hps_tier_t``."""

    def __init__(self, *, nodes: int = 1, devices: int = 1, rank: int = 0,
                 cuda_device: int = 0, width: int = 8,
                 layer_dims: Sequence[int] = (8, 16, 1), learning_rate: float = 0.05,
                 seed: int = 42, minibatches: int = 4, deterministic: bool = True,
                 inject_skip_sync: int = -1, key_space: int = 0,
                 max_batch_examples: int = 1 << 16, max_batch_keys: int = 1 << 20,
                 max_working_set: int = 0, nccl_id: Optional[bytes] = None,
                 optimizer: str = "sgd", adagrad_eps: float = 1e-8):
        cfg = HpsConfig()
        cfg.nodes, cfg.devices_per_node, cfg.rank = nodes, devices, rank
        cfg.cuda_device, cfg.embedding_dim = cuda_device, width
        cfg.num_layers = len(layer_dims)
        if not 1 <= len(layer_dims) <= HPS_MAX_LAYERS:
            raise Error(1, "config: layer_dims must end in 1")
        for i, d in enumerate(layer_dims):
            cfg.layer_dims[i] = int(d)
        cfg.learning_rate = learning_rate
        cfg.seed = seed
        cfg.minibatches = minibatches
        cfg.deterministic = int(bool(deterministic))
        cfg.inject_skip_sync = inject_skip_sync
        cfg.key_space = key_space
        cfg.max_batch_examples = max_batch_examples
        cfg.max_batch_keys = max_batch_keys
        cfg.max_working_set = max_working_set
        if optimizer not in OPTIMIZERS:
            raise Error(1, f"config: unknown optimizer {optimizer!r}")
        cfg.optimizer = OPTIMIZERS[optimizer]
        cfg.adagrad_eps = adagrad_eps
        self.cfg = cfg
        self.width = width
        # floats per table / store row: the embedding, then the Adagrad state
        self.row_width = 2 * width if optimizer == "adagrad" else width
        self.topology = Topology(nodes, devices)
        self.rank = rank
        self._h = ctypes.c_void_p(0)
        idbuf = ctypes.create_string_buffer(nccl_id, HPS_NCCL_ID_BYTES) if nccl_id else None
        _check(lib().hps_create(ctypes.byref(cfg), idbuf, ctypes.byref(self._h)))
        self._store = None

    # lifecycle
    def close(self) -> None:
        if self._h:
            lib().hps_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # raw C-ABI wrappers (numpy in/out)
    def build(self, keys, host_rows=None) -> None:
        k = _u64(keys)
        rows = None if host_rows is None else _f32(host_rows).reshape(-1)
        if rows is not None and rows.size != k.size * self.row_width:
            raise Error(7, "hbm: host value width mismatch")
        _check(lib().hps_build(self._h, _ptr(k), k.size,
                               _ptr(rows) if rows is not None else None))

    def build_placed(self, keys, host_rows=None) -> None:
        """hps_build_placed: every given key is kept (the caller placed them)."""
        k = _u64(keys)
        rows = None if host_rows is None else _f32(host_rows).reshape(-1)
        if rows is not None and rows.size != k.size * self.row_width:
            raise Error(7, "hbm: host value width mismatch")
        _check(lib().hps_build_placed(self._h, _ptr(k), k.size,
                                      _ptr(rows) if rows is not None else None))

    def pull(self, keys) -> np.ndarray:
        k = _u64(keys)
        out = np.empty((k.size, self.width), dtype=np.float32)
        _check(lib().hps_pull(self._h, _ptr(k), k.size, _ptr(out)))
        return out

    def push(self, keys, deltas) -> None:
        k = _u64(keys)
        d = _f32(deltas).reshape(-1)
        if d.size != k.size * self.width:
            raise Error(7, "hbm: delta width mismatch")
        _check(lib().hps_push(self._h, _ptr(k), _ptr(d), k.size))

    def drain(self) -> None:
        _check(lib().hps_drain(self._h))

    def table_info(self):
        cap, occ, w = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().hps_table_info(self._h, ctypes.byref(cap), ctypes.byref(occ),
                                    ctypes.byref(w)))
        return cap.value, occ.value, w.value

    def table_slots(self, with_rows: bool = False):
        cap, _, _ = self.table_info()
        keys = np.empty(cap, dtype=np.uint64)
        rows = np.empty((cap, self.row_width), dtype=np.float32) if with_rows else None
        _check(lib().hps_table_slots(self._h, _ptr(keys),
                                     _ptr(rows) if with_rows else None))
        return (keys, rows) if with_rows else keys

    def dump(self):
        _, occ, _ = self.table_info()
        keys = np.empty(occ, dtype=np.uint64)
        rows = np.empty((occ, self.row_width), dtype=np.float32)
        n = ctypes.c_uint64()
        _check(lib().hps_dump(self._h, _ptr(keys), _ptr(rows), ctypes.byref(n)))
        return keys[: n.value], rows[: n.value]

    def export(self, directory: str, file_capacity: int = 4096, first_id: int = 0) -> int:
        """hps_export: this rank's table as reference parameter files."""
        nf = ctypes.c_uint64()
        _check(lib().hps_export(self._h, os.fsencode(directory), file_capacity, first_id,
                                ctypes.byref(nf)))
        return nf.value

    def dense_sync(self, buf, deterministic: bool = True) -> np.ndarray:
        b = _f32(buf).copy()
        _check(lib().hps_dense_sync(self._h, _ptr(b), b.size, int(bool(deterministic))))
        return b

    def dense_count(self) -> int:
        n = ctypes.c_uint64()
        _check(lib().hps_dense_count(self._h, ctypes.byref(n)))
        return n.value

    def get_dense(self) -> np.ndarray:
        w = np.empty(self.dense_count(), dtype=np.float32)
        _check(lib().hps_get_dense(self._h, _ptr(w)))
        return w

    def set_dense(self, w) -> None:
        a = _f32(w)
        if a.size != self.dense_count():
            raise Error(1, "apply_update: shape mismatch")
        _check(lib().hps_set_dense(self._h, _ptr(a)))

    def attach_store(self, rows, on_device: bool = False, num_keys: Optional[int] = None):
        """rows: host numpy float32 [num_keys, row_width] (kept alive here) or a
        device pointer (int) with num_keys."""
        if rows is None:
            _check(lib().hps_attach_store(self._h, None, 0, 0))
            self._store = None
        elif on_device:
            _check(lib().hps_attach_store(self._h, ctypes.c_void_p(int(rows)), int(num_keys), 1))
            self._store = rows
        else:
            if rows.dtype != np.float32 or not rows.flags.c_contiguous:
                raise Error(1, "store must be a C-contiguous float32 array")
            if rows.ndim != 2 or rows.shape[1] != self.row_width:
                raise Error(7, "hbm: value store row width mismatch")
            _check(lib().hps_attach_store(self._h, _ptr(rows), rows.shape[0], 0))
            self._store = rows

    STORE_MODES = {0: "none", 1: "device", 2: "host-zerocopy", 3: "host-dma",
                   4: "host-mirrored"}

    def store_mode(self) -> str:
        """Where the attached store is trained (hps_store_mode)."""
        m = ctypes.c_int()
        _check(lib().hps_store_mode(self._h, ctypes.byref(m)))
        return self.STORE_MODES[m.value]

    def store_pcie_bytes(self):
        """(H2D, D2H) bytes the value store has moved over PCIe since creation."""
        h, d = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().hps_store_pcie_bytes(self._h, ctypes.byref(h), ctypes.byref(d)))
        return h.value, d.value

    def store_traffic(self):
        """(rows read from, rows written to) the value store since creation."""
        r, w = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().hps_store_traffic(self._h, ctypes.byref(r), ctypes.byref(w)))
        return r.value, w.value

    def flush(self) -> None:
        """Wait for the deferred write-backs (hps_flush): afterwards the
        attached store holds every trained row."""
        _check(lib().hps_flush(self._h))

    @staticmethod
    def _batch_args(offsets, keys, labels, on_device):
        if on_device:
            n = int(offsets[1])  # (ptr, num_examples) pairs for device buffers
            return (n, ctypes.c_void_p(int(offsets[0])), ctypes.c_void_p(int(keys)),
                    ctypes.c_void_p(int(labels)), 1), None
        o = np.ascontiguousarray(offsets, dtype=np.int64)
        k = _u64(keys)
        lab = np.ascontiguousarray(labels, dtype=np.uint8)
        return (o.size - 1, _ptr(o), _ptr(k), _ptr(lab), 0), (o, k, lab)

    def train_batch(self, offsets, keys, labels, on_device: bool = False) -> HpsBatchStats:
        st = HpsBatchStats()
        args, keep = self._batch_args(offsets, keys, labels, on_device)
        _check(lib().hps_train_batch(self._h, *args, ctypes.byref(st)))
        del keep
        return st

    def submit_batch(self, offsets, keys, labels, on_device: bool = False) -> None:
        """Pipelined train_batch (hps_submit_batch): returns once the batch is
        staged and enqueued; results come from wait_batch() in order."""
        args, keep = self._batch_args(offsets, keys, labels, on_device)
        _check(lib().hps_submit_batch(self._h, *args))
        del keep

    def wait_batch(self) -> HpsBatchStats:
        st = HpsBatchStats()
        _check(lib().hps_wait_batch(self._h, ctypes.byref(st)))
        return st

    def set_timing(self, on: bool) -> None:
        _check(lib().hps_set_timing(self._h, int(on)))

    def timing(self) -> Dict[str, float]:
        buf = (ctypes.c_double * len(TIMING_SLOTS))()
        _check(lib().hps_get_timing(self._h, buf))
        return dict(zip(TIMING_SLOTS, buf))

    def reset_timing(self) -> None:
        _check(lib().hps_reset_timing(self._h))

    def set_graphs(self, on: bool) -> None:
        _check(lib().hps_set_graphs(self._h, int(on)))

    def kernel_launches(self) -> int:
        n = ctypes.c_uint64()
        _check(lib().hps_kernel_launches(self._h, ctypes.byref(n)))
        return n.value

    def graph_captures(self) -> int:
        n = ctypes.c_uint64()
        _check(lib().hps_graph_captures(self._h, ctypes.byref(n)))
        return n.value

    def stream(self) -> int:
        s = ctypes.c_void_p()
        _check(lib().hps_stream(self._h, ctypes.byref(s)))
        return s.value or 0


HostValue = Callable[[int], Sequence[float]]


class DeviceTable:
    """Read-only view of one rank's table with DeviceTable's query API
    (device_table.hpp:47-101)."""

    def __init__(self, tier: Tier):
        self._tier = tier

    def capacity(self) -> int:
        return self._tier.table_info()[0]

    def occupancy(self) -> int:
        return self._tier.table_info()[1]

    def value_width(self) -> int:
        return self._tier.width

    def for_each(self, fn) -> None:
        keys, rows = self._tier.table_slots(with_rows=True)
        live = keys != np.uint64(0xFFFFFFFFFFFFFFFF)
        for k, r in zip(keys[live], rows[live]):
            fn(int(k), r)

    def contains(self, key: int) -> bool:
        keys = self._tier.table_slots()
        return bool(np.any(keys == np.uint64(key))) and key != 0xFFFFFFFFFFFFFFFF

    def get(self, key: int) -> List[float]:
        keys, rows = self._tier.table_slots(with_rows=True)
        hit = np.nonzero(keys == np.uint64(key))[0]
        if hit.size == 0:
            raise Error(2, f"device table: missing key {key}")
        return rows[hit[0]].tolist()


class HbmTier:
    """hps::HbmTier (hbm_ps.hpp:41-242) for one rank of a PartitionPolicy::modulo
    tier. ``get``/``push_deltas``/``accumulate`` are collective over ranks."""

    def __init__(self, topo: Topology, width: int, *, rank: int = 0,
                 cuda_device: int = 0, nccl_id: Optional[bytes] = None, **kw):
        self.topo = topo
        self.width = width
        self.rank = rank
        self.tier = Tier(nodes=topo.num_nodes, devices=topo.devices_per_node, rank=rank,
                         cuda_device=cuda_device, width=width, nccl_id=nccl_id, **kw)
        self._built = False

    def value_width(self) -> int:
        return self.width

    def topology(self) -> Topology:
        return self.topo

    def build_node(self, node: int, keys_per_node: Sequence[Iterable[int]],
                   host_value) -> None:
        """hbm_ps.hpp:65-102. host_value: HostValue callable or a mapping."""
        if self.topo.node_of(self.rank) != node:
            return
        merged = np.unique(np.concatenate(
            [_u64(list(ks)) for ks in keys_per_node] or [np.empty(0, np.uint64)]))
        owned = merged[(merged % np.uint64(self.topo.total_devices())) == np.uint64(self.rank)]
        rows = np.zeros((owned.size, self.width), dtype=np.float32)
        for i, k in enumerate(owned.tolist()):
            v = host_value[k] if isinstance(host_value, Mapping) else host_value(k)
            if len(v) != self.width:
                raise Error(7, "hbm: host value width mismatch")
            rows[i] = v
        self.tier.build(owned, rows)
        self._built = True

    def build_all(self, keys_per_node, host_value) -> None:
        for n in range(self.topo.num_nodes):
            self.build_node(n, keys_per_node, host_value)

    def built(self) -> bool:
        return self._built

    def get(self, keys: Iterable[int]) -> Dict[int, List[float]]:
        """hbm_ps.hpp:112-143: order-normalized view of `keys`."""
        k = np.unique(_u64(list(keys)))
        rows = self.tier.pull(k)
        return {int(a): rows[i].tolist() for i, a in enumerate(k)}

    def push_deltas(self, deltas: Mapping[int, Sequence[float]]) -> None:
        items = sorted(deltas.items())
        for _, v in items:
            if len(v) != self.width:
                raise Error(7, "hbm: delta width mismatch")
        keys = [k for k, _ in items]
        vals = np.array([v for _, v in items], dtype=np.float32).reshape(-1, self.width)
        self.tier.push(keys, vals)

    def drain_accums(self) -> None:
        self.tier.drain()

    def accumulate(self, deltas: Mapping[int, Sequence[float]]) -> None:
        self.push_deltas(deltas)
        self.drain_accums()

    def table_at(self, g: Optional[int] = None) -> DeviceTable:
        if g is not None and g != self.rank:
            raise Error(1, "table_at: only this rank's table is addressable")
        if not self._built:
            raise Error(6, "hbm: tables not built")
        return DeviceTable(self.tier)

    def dump_node(self, node: Optional[int] = None) -> Dict[int, List[float]]:
        keys, rows = self.tier.dump()
        return {int(k): rows[i].tolist() for i, k in enumerate(keys)}

    def close(self) -> None:
        self.tier.close()


def canonical_order(topo: Topology) -> List[int]:
    """Replica order of canonical_sum (hbm_ps.hpp:264-267)."""
    return [topo.global_index(n, d) for n in range(topo.num_nodes)
            for d in range(topo.devices_per_node)]


def synchronize(tier: Tier, buf, deterministic: bool = False) -> np.ndarray:
    """SyncSession::run for this rank (hbm_ps.hpp:303-310): returns the sum of
    every rank's buffer. COLLECTIVE."""
    return tier.dense_sync(buf, deterministic)

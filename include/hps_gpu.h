/* hps_gpu.h — C ABI of the B200-native HBM-PS tier (libhps_gpu.so).
 *
 * This is the drop-in boundary for the reference parameter server's device
 * tier (arXiv 2003.05622, reference `hps`, /root/reference/proj/include/hps).
 * The reference binds this path in-process as the C++ class `hps::HbmTier`
 * plus free functions; every entry point below names the reference interface
 * it replaces (file:line). Plain pointers and sizes only; no torch types.
 *
 * Process model: one tier handle per GPU ("rank" = global device index
 * g = device * nodes + node, topology.hpp:43-50). Calls marked COLLECTIVE
 * must be made by every rank of the tier, in the same order (the reference's
 * device-worker threads are phase-separated by barriers the same way,
 * pipeline.hpp:529-558). Ranks exchange keys, rows, deltas and dense
 * gradients over NCCL (NVLink/NVSwitch); a world of one needs no NCCL.
 *
 * Every function returns an hps_status; hps_last_error() returns the
 * calling thread's message for the last failure. Messages for table misuse
 * match the reference's hps::Error texts (device_table.hpp:52-91).
 */
#ifndef HPS_GPU_H
#define HPS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_NCCL_ID_BYTES 128
#define HPS_MAX_LAYERS 8

typedef enum {
  HPS_OK = 0,
  HPS_ERR_ARG = 1,           /* invalid argument / config (config.hpp:86-108) */
  HPS_ERR_MISSING_KEY = 2,   /* device_table.hpp:80-81, 90-91 */
  HPS_ERR_DUPLICATE = 3,     /* device_table.hpp:56-57 */
  HPS_ERR_OVERFLOW = 4,      /* device_table.hpp:61-62, 72 */
  HPS_ERR_NONFINITE = 5,     /* model.hpp:70, 210 */
  HPS_ERR_NOT_BUILT = 6,     /* hbm_ps.hpp:209 "hbm: tables not built" */
  HPS_ERR_WIDTH = 7,         /* hbm_ps.hpp:95, 152 width mismatch */
  HPS_ERR_KEY_RANGE = 8,     /* pipeline.hpp:367-371 ingest range check */
  HPS_ERR_CUDA = 9,
  HPS_ERR_NCCL = 10,
  HPS_ERR_CAPACITY = 11,     /* a batch larger than the configured maxima */
  HPS_ERR_CORRUPT = 12       /* a parameter file failed validation
                                (hps::CorruptionError, ssd_ps.hpp:495-520) */
} hps_status;

typedef struct hps_tier* hps_tier_t;

/* Run knobs, the subset of RunConfig (config.hpp:40-74) the HBM-PS path
 * reads, plus buffer maxima so every device buffer is allocated once. */
typedef struct {
  int nodes;                 /* N, power of two (topology.hpp:31-37) */
  int devices_per_node;      /* D, power of two */
  int rank;                  /* this handle's global device index g */
  int cuda_device;           /* CUDA ordinal this handle drives */
  int embedding_dim;         /* E: row width in floats */
  int num_layers;            /* dense stack depth, <= HPS_MAX_LAYERS */
  uint64_t layer_dims[HPS_MAX_LAYERS]; /* must end in 1 (config.hpp:90-91) */
  float learning_rate;       /* SGD lr (model.hpp:204-230) */
  uint64_t seed;             /* init_dense seed (model.hpp:42-53) */
  int minibatches;           /* J mini-batches per batch (config.hpp:52) */
  int deterministic;         /* config.hpp:67; accepted, but every mode takes
                                the canonical f64 order (bit-exact; there is
                                no separate f32 fast path) */
  int64_t inject_skip_sync;  /* global mini-batch whose dense sync+update is
                                skipped, -1 = off (pipeline.hpp:550-555) */
  uint64_t key_space;        /* keys are < key_space ("dims"); sizes sorts */
  uint64_t max_batch_examples;  /* per batch */
  uint64_t max_batch_keys;      /* key occurrences per batch */
  uint64_t max_working_set;     /* keys per build() call, 0 = max_batch_keys */
  int optimizer;             /* HPS_OPT_SGD (the reference's, model.hpp:204-230)
                                or HPS_OPT_ADAGRAD (extension, BASELINE c3) */
  float adagrad_eps;         /* Adagrad: v -= lr*g / (sqrt(s) + eps), eps > 0 */
} hps_config;

/* Sparse optimizers. A table / value-store row is the embedding (E floats),
 * then for Adagrad its accumulator state (E floats, zero-initialised: the
 * reference's SparseParam::opt_state, types.hpp:30-39): rows are
 * hps_row_width() = E (SGD) or 2E floats. Pushed values are SGD deltas
 * -(lr*g) (hbm_ps.hpp:148-195 accumulate) or, for Adagrad, the gradients g;
 * the owner applies them per sender in canonical order:
 *   s' = s + g*g;  v' = v - (lr*g) / (sqrt(s') + eps)  (f32, IEEE-rounded). */
enum { HPS_OPT_SGD = 0, HPS_OPT_ADAGRAD = 1 };

/* Per-batch result of hps_train_batch. */
typedef struct {
  double loss_sum;           /* sum of per-example log loss (model.hpp:232-242) */
  uint64_t examples;         /* examples this rank trained */
  uint64_t working_set;      /* keys this rank's table holds for the batch */
  uint64_t table_capacity;   /* capacity of that table */
  uint64_t pulled_keys;      /* sum over mini-batches of unique keys pulled */
  uint64_t served_keys;      /* keys this rank served as owner (pull+push) */
  uint64_t occurrences;      /* key occurrences in this rank's shards */
  uint64_t carried_rows;     /* build rows taken from the previous table */
  uint64_t exact_fallbacks;  /* certified parallel sums that had to be redone
                                in the exact sequential order */
  uint64_t store_rows;       /* build rows read from the attached value store
                                (the rest: carried, the table two builds back
                                while its write-back drains, or zeros) */
  uint64_t big_segments;     /* (key, mini-batch) segments longer than 32
                                occurrences (the chunked, certified reduce) */
  uint64_t max_segment_chunks; /* most chunks of one such segment */
  uint64_t big_occurrences;  /* key occurrences in those segments */
  uint64_t mid_segments;     /* segments of 33..mid length (HPS_MID_SEG, default
                                1024) summed exactly by one warp each; longer
                                ones take the chunked certified reduce */
} hps_batch_stats;

/* Phase slots of hps_get_timing (ms accumulated over hps_train_batch calls,
 * measured with CUDA events on the tier's stream). */
#define HPS_TIMING_SLOTS 12
enum {
  HPS_T_TOTAL = 0,     /* whole batch */
  HPS_T_STAGE = 1,     /* H2D of the batch + per-shard counts (one D2H) */
  HPS_T_BUILD = 2,     /* working-set dedup + table build (a1-a4) */
  HPS_T_DEDUP = 3,     /* mini-batch dedup + owner partition (a5) */
  HPS_T_PULL = 4,      /* owner probe + row gather (+ all-to-alls) (a6) */
  HPS_T_FWDBWD = 5,    /* forward/backward (a7, a8) */
  HPS_T_GRADS = 6,     /* dense-grad reduce + sparse segment-reduce (a8, a9) */
  HPS_T_APPLY = 7,     /* push exchange + canonical owner apply (a10, a11) */
  HPS_T_DENSE = 8,     /* dense sync + update (a12) */
  HPS_T_WRITEBACK = 9, /* rows back to the value store (a13) */
  HPS_T_SPARSE = 10,   /* sparse segment-reduce + sgd_delta (a8, a9); GRADS is
                          then the wait for the dense-grad reduce beside it */
  HPS_T_BIGFUSED = 11  /* big_fused_kernel alone (the chunked reduce of the
                          long segments, on its side stream inside SPARSE) */
};

const char* hps_last_error(void);
const char* hps_version(void);

/* ----------------------------------------------------------- lifecycle */

/* ncclGetUniqueId for rank 0 to broadcast (only needed when N*D > 1). */
hps_status hps_get_unique_id(uint8_t id[HPS_NCCL_ID_BYTES]);

/* Replaces HbmTier::HbmTier (hbm_ps.hpp:45-56) with PartitionPolicy::modulo
 * (topology.hpp:61-65) and replicate_dense(init_dense(cfg)) (hbm_ps.hpp:
 * 244-247, model.hpp:42-53). COLLECTIVE when N*D > 1 (nccl_id required). */
hps_status hps_create(const hps_config* cfg, const uint8_t* nccl_id,
                      hps_tier_t* out);
hps_status hps_destroy(hps_tier_t h);

/* ------------------------------------------------ reference-facing API */

/* HbmTier::build_node (hbm_ps.hpp:65-102): merge+sort+unique `keys` (any
 * order, duplicates allowed — the node's working set plus peer keys), keep
 * the keys this rank owns, build a fresh table (capacity next_pow2(4n/3),
 * device_table.hpp:38-45) whose slot layout equals ascending-order linear
 * probing, and fill each row from the previous table when the key was there
 * (carry-over) else from `host_rows` (row i belongs to keys[i], each
 * hps_row_width() floats; the HostValue callback's result, staged H2D with
 * cudaMemcpyAsync) or, when
 * host_rows is NULL, from the attached value store (zero if none). */
hps_status hps_build(hps_tier_t h, const uint64_t* keys, uint64_t n,
                     const float* host_rows);

/* hps_build for keys the CALLER placed on this device (hbm_ps.hpp:74-80
 * with any PartitionPolicy, e.g. range_split, topology.hpp:67-71): every
 * given key is kept, no key % (N*D) filter. Used by the in-process hps::
 * adapter (hps_gpu/hbm_ps.hpp), whose get/push route by the policy on the
 * host; the collective hps_pull/hps_push/hps_train_* route by key % (N*D)
 * and must not be mixed with a non-modulo placement. */
hps_status hps_build_placed(hps_tier_t h, const uint64_t* keys, uint64_t n,
                            const float* host_rows);

/* HbmTier::get (hbm_ps.hpp:112-143). COLLECTIVE. Rows for `keys` (host
 * array, any order) written to out_rows (n x E, aligned with keys). Keys
 * owned by other ranks travel as pull request/response all-to-alls. */
hps_status hps_pull(hps_tier_t h, const uint64_t* keys, uint64_t n,
                    float* out_rows);

/* HbmTier::push_deltas (hbm_ps.hpp:148-167). COLLECTIVE. Ships each delta
 * row (n x E; Adagrad: gradient rows) to its owner, where it is queued
 * (nothing applied yet). */
hps_status hps_push(hps_tier_t h, const uint64_t* keys, const float* deltas,
                    uint64_t n);

/* HbmTier::drain_accums (hbm_ps.hpp:172-195): apply every queued delta,
 * senders in canonical node-major/device-major order, v += d in f32
 * (device_table.hpp:88-95; Adagrad: the step above). Local to the rank. */
hps_status hps_drain(hps_tier_t h);

/* DeviceTable::accumulate (device_table.hpp:88-95) of one sender's unique
 * (keys, deltas) on this rank's own table, in place (Adagrad: the step);
 * local, not collective: the in-process hps:: adapter (hps_gpu/hbm_ps.hpp)
 * queues each sender's deltas and applies them in canonical order with it. */
hps_status hps_apply_local(hps_tier_t h, const uint64_t* keys, const float* deltas,
                           uint64_t n);

/* HbmTier::dump_node (hbm_ps.hpp:224-232) for this rank's table: keys in
 * ascending order and their rows (hps_row_width() floats each: embedding,
 * then Adagrad state). *n_out = occupancy. Buffers sized by
 * hps_table_info's occupancy. */
hps_status hps_dump(hps_tier_t h, uint64_t* keys_out, float* rows_out,
                    uint64_t* n_out);

/* DeviceTable::capacity/occupancy/value_width (device_table.hpp:47-49);
 * width = E, the embedding width. */
hps_status hps_table_info(hps_tier_t h, uint64_t* capacity,
                          uint64_t* occupancy, uint64_t* width);
/* DeviceTable::contains / get (device_table.hpp:76-85) for a batch of keys
 * against this rank's current table, without the missing-key error:
 * found[i] = 1 and, if rows is non-NULL, rows[i] = the key's row
 * (hps_row_width() floats), else found[i] = 0. Local (not collective). */
hps_status hps_table_lookup(hps_tier_t h, const uint64_t* keys, uint64_t n, uint8_t* found,
                            float* rows);
/* Floats per table / value-store row: E (SGD) or 2E (Adagrad). */
hps_status hps_row_width(hps_tier_t h, uint64_t* row_width);
/* Slot-level view for placement parity: slot_keys[capacity] (empty slots
 * hold ~0, device_table.hpp:34) and, if non-NULL, rows[capacity x
 * hps_row_width()]. */
hps_status hps_table_slots(hps_tier_t h, uint64_t* slot_keys, float* rows);

/* SyncSession::run (hbm_ps.hpp:303-310) on a host buffer. COLLECTIVE.
 * Every rank ends with the elementwise sum of all ranks' buffers:
 * f64 canonical_sum of the raw buffers (hbm_ps.hpp:258-277, 349-394) in
 * both modes: `deterministic` is accepted for the reference signature; the
 * default mode's contract (within 1e-6 of canonical) holds bit-exactly. */
hps_status hps_dense_sync(hps_tier_t h, float* buf, uint64_t len,
                          int deterministic);

/* Dense replica access (DenseParams::weights, types.hpp:41-60). */
hps_status hps_dense_count(hps_tier_t h, uint64_t* n);
hps_status hps_get_dense(hps_tier_t h, float* w);
hps_status hps_set_dense(hps_tier_t h, const float* w);

/* ------------------------------------------------- performance API */

/* Attach the host-tier value store (the MEM-PS stand-in): rows[key * RW]
 * (RW = hps_row_width(): the embedding, then the Adagrad state)
 * for key < num_keys. build() fills rows of keys that were not in the
 * previous table from it, and hps_train_batch writes the trained rows back
 * after each batch (dump_node -> MemPs::collect_updates, pipeline.hpp:
 * 441-445, mem_ps.hpp:210-245). on_device = 0: pinned host memory reached
 * with zero-copy gather/scatter kernels; 1: an HBM array. Flushes pending
 * write-backs to the previously attached store first. */
hps_status hps_attach_store(hps_tier_t h, float* rows, uint64_t num_keys,
                            int on_device);

/* Where the attached value store is trained (hps_store_mode):
 * HPS_STORE_HOST_MIRRORED — a host store (on_device = 0) that fits the HBM
 * budget (HPS_STORE_MIRROR_GB, default 2 GB, or
 * up to 16 batches of worst-case staging; the copy-back of a bigger
 * store at every observation would outweigh a short run's per-batch staging) is copied to
 * HBM once at attach, the builds and write-backs use that copy, and the host
 * array is made exact whenever it is observed (every entry point that
 * quiesces: hps_flush, hps_destroy, hps_attach_store, hps_get_dense, ...),
 * so the per-batch PCIe traffic is the batch alone. At N*D > 1 (ranks may
 * share one host array) the copy-back writes only the rows this rank owns. A bigger host store is
 * staged per batch: zero-copy SM gathers/scatters (HPS_STORE_HOST_ZEROCOPY)
 * or host threads + cudaMemcpyAsync (HPS_STAGE=dma, HPS_STORE_HOST_DMA). */
enum {
  HPS_STORE_NONE = 0,
  HPS_STORE_DEVICE = 1,
  HPS_STORE_HOST_ZEROCOPY = 2,
  HPS_STORE_HOST_DMA = 3,
  HPS_STORE_HOST_MIRRORED = 4
};
hps_status hps_store_mode(hps_tier_t h, int* mode);

/* Bytes the value store has moved over PCIe since hps_create: per-batch
 * staging (zero-copy or DMA: every row read or written back), or the
 * mirror's attach copies and its copy-backs (dirty 1024-row pages only). */
hps_status hps_store_pcie_bytes(hps_tier_t h, uint64_t* h2d, uint64_t* d2h);

/* Write-back (the reference's collect stage, pipeline.hpp:462-474) runs
 * asynchronously beside the next batches. The four most recent batch tables
 * stay resident in HBM; a row reaches the store when its table is recycled
 * and no newer resident table holds the key (a newer one has the fresher row).
 * Builds read the store only for keys outside the resident tables, after the
 * write-backs they depend on (the mem_ps.hpp freshness rule: prepare of step
 * t+2 after collect of step t). hps_flush blocks until every resident row has
 * reached the store; after it (or hps_attach_store / hps_destroy, and before
 * any other entry point runs) the store holds every trained row. */
hps_status hps_flush(hps_tier_t h);

/* Value-store traffic since hps_create: rows read by table builds (completed
 * batches) and rows written back (eviction write-backs and flushes; a row a
 * newer resident table still holds is written once it leaves, not every
 * batch). */
hps_status hps_store_traffic(hps_tier_t h, uint64_t* rows_read, uint64_t* rows_written);

/* One whole batch through the tier, device-resident: working-set dedup ->
 * build (carry-over + store staging) -> J x {mini-batch dedup, pull
 * all-to-all, forward/backward, sparse segment-reduce + sgd_delta, push
 * all-to-all, canonical apply, dense sync + update} -> write-back to the
 * store. The batch is the full node batch in CSR form (every rank passes the
 * same batch, as each node's train stage holds it, pipeline.hpp:417-460);
 * this rank trains shard_batch's slice (sharding.hpp:29-42). COLLECTIVE.
 * on_device = 0: offsets/keys/labels are host (pinned for speed) pointers,
 * copied H2D inside the call; 1: device pointers. stats may be NULL. */
hps_status hps_train_batch(hps_tier_t h, uint64_t num_examples,
                           const int64_t* offsets, const uint64_t* keys,
                           const uint8_t* labels, int on_device,
                           hps_batch_stats* stats);

/* The same batch, pipelined (the reference Trainer's bounded stage queues,
 * pipeline.hpp:42-60 and 305-315): hps_submit_batch stages the batch (H2D +
 * counts; the host blocks only on that round-trip), enqueues its table build
 * beside the previous batch's body, its body and its write-back, and returns.
 * hps_wait_batch returns the results of the oldest submitted batch not yet
 * waited for, in submission order. At most four batches are in flight (a
 * fifth submit first completes the oldest; its result stays queued). Device
 * buffers and pageable host buffers may be reused as soon as hps_submit_batch
 * returns; pinned host buffers are copied asynchronously and must stay
 * unchanged until the batch's hps_wait_batch (the cudaMemcpyAsync rule). A
 * key outside key_space is reported by hps_wait_batch. Results are
 * bit-identical to hps_train_batch on the same batches. COLLECTIVE. Every
 * other entry point completes all in-flight batches first. */
hps_status hps_submit_batch(hps_tier_t h, uint64_t num_examples,
                            const int64_t* offsets, const uint64_t* keys,
                            const uint8_t* labels, int on_device);
hps_status hps_wait_batch(hps_tier_t h, hps_batch_stats* stats);

/* Per-phase device time of hps_train_batch (HPS_T_* slots, ms, accumulated
 * until hps_reset_timing). Enabled by hps_set_timing(h, 1): adds event
 * records on the pipeline's streams and runs one batch at a time, so every
 * phase is timed without overlap (BUILD = table build + carry-over;
 * WRITEBACK = the deferred write-back; TOTAL = stage start to body end). */
hps_status hps_set_timing(hps_tier_t h, int enable);
hps_status hps_get_timing(hps_tier_t h, double* ms /* HPS_TIMING_SLOTS */);
hps_status hps_reset_timing(hps_tier_t h);

/* hps_train_batch captures its device-side body into a CUDA graph per
 * batch shape and replays it (default on); 0 = launch kernel by kernel. */
hps_status hps_set_graphs(hps_tier_t h, int enable);

/* Number of kernels this library launched on the handle so far (a graph
 * replay counts the kernels it contains). */
hps_status hps_kernel_launches(hps_tier_t h, uint64_t* n);

/* Number of CUDA graphs captured and instantiated on the handle so far (one
 * per batch shape and table rotation; the first steady-state batch of a shape
 * captures every rotation). The bench reports the captures inside its timed
 * region: zero means it timed replays only. */
hps_status hps_graph_captures(hps_tier_t h, uint64_t* n);

/* Diagnostics: one tcgen05 TF32 GEMM of the wide-MLP path (mlp.cuh) on
 * device pointers, synchronous: D(m, n) = sum_k A(m, k) B(n, k) with
 * A(m, k) = A[m*a_m + k*a_k], B(n, k) = B[n*b_n + k*b_k] (b_ones_col: row
 * N-1 of B is all ones), epilogue epi: 0 store (split-K slice z at
 * D + z*M*ldd), 1 bias + relu, 2 mask(m, n) = mask[m*ldm + n] > 0, 3 f64 to
 * Dd. For the numerics tests against a PyTorch fp32 reference. */
hps_status hps_debug_gemm_tf32(int M, int N, int K, const float* A, int64_t a_m, int64_t a_k,
                               const float* B, int64_t b_n, int64_t b_k, int b_ones_col, int epi,
                               float* D, double* Dd, int64_t ldd, const float* bias,
                               const float* mask, int64_t ldm, int splits);

/* The CUDA stream the handle launches on (cudaStream_t as void*). */
hps_status hps_stream(hps_tier_t h, void** stream);

/* ------------------------------- parameter files (SSD-PS on-disk format) */

/* Trained tables leave the tier in the reference's parameter-file format
 * (ssd_ps.hpp:50-56: "HPSF" | version 1 | record_count u16 | width u16 |
 * reserved u16, then record_count x (key u64 | E f32 embedding | E f32
 * opt_state), then the zlib CRC-32 of header + records), so the reference
 * SsdStore recovers, loads, fscks and stats them unchanged (SURVEY §8(f)
 * row 3). Host-only; no GPU needed. */

/* CRC-32 as zlib's crc32(crc, data, n) (the footer checksum). */
uint32_t hps_crc32(uint32_t crc, const void* data, uint64_t n);

/* SsdStore::dump (ssd_ps.hpp:229-243) + write_chunk (420-450): the n
 * records (keys strictly ascending, the std::map order) as
 * ceil(n / file_capacity) files dir/pf_<first_id + i>.bin, each written to a
 * temporary name and renamed. opt_state NULL writes zeros (SparseParam(width),
 * types.hpp:36). *files_out = files written. Errors: file_capacity outside
 * [1, 65535] and n == 0 use the reference's messages (ssd_ps.hpp:159-160,
 * 227). */
hps_status hps_pfile_write(const char* dir, const uint64_t* keys,
                           const float* rows, const float* opt_state,
                           uint64_t n, uint32_t width, uint32_t file_capacity,
                           uint64_t first_id, uint64_t* files_out);

/* SsdStore::read_file_at (ssd_ps.hpp:495-535): one file, validated (magic,
 * version, width vs *width_out when it is non-zero, size, CRC) with the
 * reference's messages (HPS_ERR_CORRUPT). keys/rows/opt_state all NULL is a
 * sizing call (sets *n_out, *width_out). */
hps_status hps_pfile_read(const char* path, uint64_t* keys, float* rows,
                          float* opt_state, uint64_t cap, uint64_t* n_out,
                          uint32_t* width_out);

/* HbmTier::dump_node (hbm_ps.hpp:224-232) of this rank's table, written as
 * parameter files (the MEM-PS collect -> SSD-PS dump path, mem_ps.hpp:
 * 210-245): hps_dump + hps_pfile_write, opt_state = the Adagrad state
 * (zero under SGD, which never touches it, model.hpp:204). Ranks hold
 * disjoint keys, so every rank can export into one directory with disjoint
 * id ranges. */
hps_status hps_export(hps_tier_t h, const char* dir, uint32_t file_capacity,
                      uint64_t first_id, uint64_t* files_out);

/* -------------------------------------------------- synthetic inputs */

/* BASELINE config 4's multi-slot input (a new generator; the reference has
 * none): T ~ U{1..max_keys} draws per example of key = slot * ids_per_slot +
 * id, slot uniform over `slots`, id ~ Zipf(zipf_s); sorted unique per example;
 * planted-logistic labels. keys must hold num_examples * max_keys entries;
 * *n_keys_out = offsets[num_examples]. Host-only. */
hps_status hps_gen_multislot(uint64_t slots, uint64_t ids_per_slot, uint64_t num_examples,
                             uint64_t max_keys, double zipf_s, uint64_t seed,
                             double signal_scale, int64_t* offsets, uint64_t* keys,
                             uint8_t* labels, uint64_t* n_keys_out);

/* The reference generator gen_dataset (dataset.hpp:180-227) restated
 * byte-for-byte (mt19937_64 stream, planted logistic labels, inverse-CDF
 * Zipf, sorted unique features). offsets[num_examples+1], keys[n*nnz],
 * labels[n]. Host-only, needs no GPU. */
hps_status hps_gen_dataset(uint64_t dims, uint64_t num_examples, uint64_t nnz,
                           int zipf, double zipf_s, uint64_t seed,
                           double signal_scale, uint64_t clusters,
                           int64_t* offsets, uint64_t* keys, uint8_t* labels);

#ifdef __cplusplus
}
#endif
#endif /* HPS_GPU_H */

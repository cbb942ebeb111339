/* TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * A plain-C restatement of the reference HBM-PS hot path (arXiv 2003.05622,
 * /root/reference/proj/include/hps). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. Every function cites the
 * reference file:line it restates. Pinned against the reference's own
 * outputs (tests/golden/, produced by oracle/_ref from the unmodified
 * headers) in tests/test_oracle_golden.py.
 */
#ifndef HPS_ORACLE_H
#define HPS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_EMPTY (~(uint64_t)0) /* device_table.hpp:34 kEmpty */

typedef struct {
  int nodes;                 /* config.hpp:43 */
  int devices;               /* config.hpp:44 */
  int embedding_dim;         /* config.hpp:46 */
  int num_layers;
  uint64_t layer_dims[8];    /* config.hpp:47, must end in 1 */
  float learning_rate;       /* config.hpp:48 */
  uint64_t seed;             /* config.hpp:49 */
  int minibatches;           /* config.hpp:52 J */
  int deterministic;         /* config.hpp:67 */
  int64_t inject_skip_sync;  /* config.hpp:72-74; the oracle never skips */
  /* Extension fields (no reference pin; RefCfg stops before them): */
  int optimizer;             /* 0 SGD (model.hpp:204-230), 1 Adagrad */
  float adagrad_eps;         /* Adagrad epsilon (> 0) */
} or_cfg;

const char* or_last_error(void);

/* common.hpp:57-62 splitmix64 finalizer */
uint64_t or_mix64(uint64_t x);
/* device_table.hpp:35-45: next_pow2(max(1, (4n+2)/3)) */
uint64_t or_capacity(uint64_t n);
/* device_table.hpp:51-73 + 115-117: sequential ascending-order linear-probe
 * insert of n sorted unique keys into slots[cap] (EMPTY-filled). Returns 0,
 * or 1 on duplicate/overflow with or_last_error() set. */
int or_table_build(const uint64_t* keys, uint64_t n, uint64_t cap,
                   uint64_t* slots);
/* device_table.hpp:119-128 find_slot: slot index or -1 */
int64_t or_table_find(const uint64_t* slots, uint64_t cap, uint64_t key);

/* mem_ps.hpp:101-108 extract_working_set / hbm_ps.hpp:69-74: sort+unique.
 * Returns the number of unique keys written to out. */
uint64_t or_sort_unique(const uint64_t* keys, uint64_t n, uint64_t* out);
/* topology.hpp:61-65 modulo policy: g = key % (N*D) */
void or_owner(const uint64_t* keys, uint64_t n, int nodes, int devices,
              int32_t* g_out);
/* sharding.hpp:29-42: example i -> device (i%(D*J))/J, mini-batch %J */
void or_shard(uint64_t num_examples, int devices, int minibatches,
              int32_t* dev_out, int32_t* mb_out);

/* model.hpp:42-53 init_dense (mt19937_64(seed), uniform +-0.05) */
uint64_t or_dense_count(int input_dim, int num_layers,
                        const uint64_t* layer_dims);
void or_init_dense(const or_cfg* c, float* out);

/* model.hpp:101-202 forward+backward over one shard. The embedding view is
 * (emb_keys sorted unique, emb_rows). Outputs preds[n], dense_grad[W] and
 * sparse_grad rows aligned with emb_keys (zero rows for keys the shard does
 * not touch). Returns 0 or 1 (missing key / non-finite). */
int or_forward_backward(int width, int num_layers, const uint64_t* layer_dims,
                        const float* dense, uint64_t num_examples,
                        const int64_t* offsets, const uint64_t* keys,
                        const uint8_t* labels, const uint64_t* emb_keys,
                        const float* emb_rows, uint64_t n_emb, double* preds,
                        float* dense_grad, float* sparse_grad);

/* hbm_ps.hpp:258-277 canonical_sum over G = N*D replicas (bufs G x len in
 * global-index order) -> f32 sum */
void or_canonical_sum(int nodes, int devices, const float* bufs, uint64_t len,
                      float* out);
/* hbm_ps.hpp:251-256 average_by then model.hpp:205-212 apply_update */
int or_average_apply(float* w, const float* sum, uint64_t len, int count,
                     float lr);
/* model.hpp:226-230 sgd_delta then device_table.hpp:88-95 accumulate */
void or_sgd_accumulate(float* v, const float* g, uint64_t len, float lr);
/* SELF-PINNED EXTENSION (BASELINE config 3: the reference
 * has no Adagrad; its SparseParam carries an untouched opt_state,
 * types.hpp:30-39). The owner applies one sender's gradient row g to the
 * embedding v and its accumulator s (both len floats), in f32 with IEEE
 * rounding per op:  s += g*g;  v -= (lr*g) / (sqrtf(s) + eps). */
void or_adagrad_apply(float* v, float* s, const float* g, uint64_t len, float lr, float eps);

/* oracle.hpp:55-122 train_reference over to_batches(ds, batch_size)
 * (dataset.hpp:96-108). Sparse result sorted by key; each row is the
 * embedding, then (optimizer == 1) its Adagrad state: E or 2E floats. The
 * sparse deltas are applied per sender in canonical (node, device) order
 * (oracle.hpp:102-112): v += -(lr*g) for SGD, or_adagrad_apply for Adagrad. */
int or_train_reference(const or_cfg* c, uint64_t batch_size,
                       uint64_t num_examples, const int64_t* offsets,
                       const uint64_t* keys, const uint8_t* labels,
                       float* dense_out, uint64_t* n_sparse_out,
                       uint64_t* sparse_keys_out, float* sparse_rows_out,
                       uint64_t sparse_cap);

/* oracle.hpp:125-141 score_examples + model.hpp:232-270 loss/auc helpers */
double or_auc(const uint8_t* labels, const double* scores, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif

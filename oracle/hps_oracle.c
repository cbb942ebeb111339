/* TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * Plain-C restatement of the reference HBM-PS hot path. See hps_oracle.h for
 * the per-function citations; line numbers below refer to
 * /root/reference/proj/include/hps/. Built by oracle/Makefile with
 * -ffp-contract=off so every f32/f64 operation rounds exactly like the
 * reference's x86-64 build (model.hpp does all math in f64, parameters and
 * gradients in f32).
 */
#include "hps_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];

const char* or_last_error(void) { return g_err; }

static int fail(const char* msg, uint64_t key, int with_key) {
  if (with_key)
    snprintf(g_err, sizeof g_err, "%s%llu", msg, (unsigned long long)key);
  else
    snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

/* ---------------------------------------------------------------- common */

/* common.hpp:57-62 */
uint64_t or_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* common.hpp:50-54 */
static uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

/* common.hpp:69-71 */
static double u64_to_unit(uint64_t x) {
  return (double)(x >> 11) * 0x1.0p-53;
}

/* std::mt19937_64 as used by model.hpp:50 (init_dense) */
typedef struct {
  uint64_t mt[312];
  int mti;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[x & 1ULL];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[x & 1ULL];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[x & 1ULL];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* ---------------------------------------------------------- device table */

/* device_table.hpp:38-45 */
uint64_t or_capacity(uint64_t n) {
  uint64_t want = (n * 4 + 2) / 3;
  return next_pow2(want < 1 ? 1 : want);
}

/* device_table.hpp:51-73 (insert) with slot_of (115-117). The reference
 * inserts a partition's keys in ascending order (hbm_ps.hpp:89-98). */
int or_table_build(const uint64_t* keys, uint64_t n, uint64_t cap,
                   uint64_t* slots) {
  const uint64_t max_occ = (uint64_t)((double)cap * 0.75);
  for (uint64_t s = 0; s < cap; ++s) slots[s] = OR_EMPTY;
  uint64_t occ = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t key = keys[i];
    if (key == OR_EMPTY) return fail("device table: reserved key", 0, 0);
    uint64_t idx = or_mix64(key) & (cap - 1);
    uint64_t probes = 0;
    for (; probes < cap; ++probes) {
      if (slots[idx] == key)
        return fail("device table: duplicate insert of key ", key, 1);
      if (slots[idx] == OR_EMPTY) {
        if (++occ > max_occ)
          return fail("device table: capacity overflow (sizing bug)", 0, 0);
        slots[idx] = key;
        break;
      }
      idx = (idx + 1) & (cap - 1);
    }
    if (probes == cap)
      return fail("device table: capacity overflow (sizing bug)", 0, 0);
  }
  return 0;
}

/* device_table.hpp:119-128 */
int64_t or_table_find(const uint64_t* slots, uint64_t cap, uint64_t key) {
  uint64_t idx = or_mix64(key) & (cap - 1);
  for (uint64_t probes = 0; probes < cap; ++probes) {
    const uint64_t k = slots[idx];
    if (k == key) return (int64_t)idx;
    if (k == OR_EMPTY) return -1;
    idx = (idx + 1) & (cap - 1);
  }
  return -1;
}

/* -------------------------------------------------- dedup / partitioning */

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* mem_ps.hpp:101-108 */
uint64_t or_sort_unique(const uint64_t* keys, uint64_t n, uint64_t* out) {
  if (n == 0) return 0;
  memcpy(out, keys, n * sizeof(uint64_t));
  qsort(out, n, sizeof(uint64_t), cmp_u64);
  uint64_t m = 1;
  for (uint64_t i = 1; i < n; ++i)
    if (out[i] != out[m - 1]) out[m++] = out[i];
  return m;
}

/* topology.hpp:61-65 */
void or_owner(const uint64_t* keys, uint64_t n, int nodes, int devices,
              int32_t* g_out) {
  const uint64_t total = (uint64_t)nodes * (uint64_t)devices;
  for (uint64_t i = 0; i < n; ++i) g_out[i] = (int32_t)(keys[i] % total);
}

/* sharding.hpp:29-42 */
void or_shard(uint64_t num_examples, int devices, int minibatches,
              int32_t* dev_out, int32_t* mb_out) {
  const uint64_t slots = (uint64_t)devices * (uint64_t)minibatches;
  for (uint64_t i = 0; i < num_examples; ++i) {
    const uint64_t s = i % slots;
    dev_out[i] = (int32_t)(s / (uint64_t)minibatches);
    mb_out[i] = (int32_t)(s % (uint64_t)minibatches);
  }
}

/* ----------------------------------------------------------------- model */

/* types.hpp:46-56 */
uint64_t or_dense_count(int input_dim, int num_layers,
                        const uint64_t* layer_dims) {
  uint64_t n = 0, in = (uint64_t)input_dim;
  for (int l = 0; l < num_layers; ++l) {
    n += (in + 1) * layer_dims[l];
    in = layer_dims[l];
  }
  return n;
}

/* model.hpp:42-53 */
void or_init_dense(const or_cfg* c, float* out) {
  const uint64_t n =
      or_dense_count(c->embedding_dim, c->num_layers, c->layer_dims);
  mt64 rng;
  mt64_seed(&rng, c->seed);
  for (uint64_t i = 0; i < n; ++i)
    out[i] = (float)((u64_to_unit(mt64_next(&rng)) * 2.0 - 1.0) * 0.05);
}

typedef const float* (*lookup_fn)(void* ctx, uint64_t key);

typedef struct {
  const uint64_t* keys;
  const float* rows;
  uint64_t n;
  int width;
} sorted_view;

static int64_t bsearch_u64(const uint64_t* a, uint64_t n, uint64_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < n && a[lo] == key) ? (int64_t)lo : -1;
}

static const float* sorted_lookup(void* ctx, uint64_t key) {
  const sorted_view* v = (const sorted_view*)ctx;
  const int64_t i = bsearch_u64(v->keys, v->n, key);
  return i < 0 ? NULL : v->rows + (uint64_t)i * (uint64_t)v->width;
}

/* Forward + backward of one shard, model.hpp:57-202. ex_idx lists the
 * shard's examples (indices into the CSR) in shard order. The sparse output
 * covers the sorted union of the shard's keys (uk, allocated here). */
static int fb_core(int E, int L, const uint64_t* dims, const float* W,
                   uint64_t n, const uint64_t* ex_idx, const int64_t* offsets,
                   const uint64_t* keys, const uint8_t* labels, lookup_fn look,
                   void* ctx, double* preds, float* dense_grad,
                   uint64_t* n_uk, uint64_t** uk_out, float** sg_out) {
  uint64_t offs[8], ins[8], maxw = (uint64_t)E;
  {
    uint64_t off = 0, in = (uint64_t)E;
    for (int l = 0; l < L; ++l) {
      offs[l] = off;
      ins[l] = in;
      off += (in + 1) * dims[l];
      in = dims[l];
      if (dims[l] > maxw) maxw = dims[l];
    }
  }
  const uint64_t nw = or_dense_count(E, L, dims);
  /* union of the shard's keys */
  uint64_t nocc = 0;
  for (uint64_t t = 0; t < n; ++t)
    nocc += (uint64_t)(offsets[ex_idx[t] + 1] - offsets[ex_idx[t]]);
  uint64_t* uk = (uint64_t*)malloc((nocc ? nocc : 1) * sizeof(uint64_t));
  {
    uint64_t p = 0;
    for (uint64_t t = 0; t < n; ++t)
      for (int64_t q = offsets[ex_idx[t]]; q < offsets[ex_idx[t] + 1]; ++q)
        uk[p++] = keys[q];
  }
  const uint64_t nu = or_sort_unique(uk, nocc, uk);
  double* sacc = (double*)calloc((nu ? nu : 1) * (uint64_t)E, sizeof(double));
  double* dacc = (double*)calloc(nw, sizeof(double));
  double* hs = (double*)malloc((uint64_t)(L + 1) * maxw * sizeof(double));
  double* zs = (double*)malloc((uint64_t)L * maxw * sizeof(double));
  double* delta = (double*)malloc(maxw * sizeof(double));
  double* dprev = (double*)malloc(maxw * sizeof(double));
  int rc = 0;

  for (uint64_t t = 0; t < n && rc == 0; ++t) {
    const uint64_t e = ex_idx[t];
    /* embed_sum, model.hpp:84-95 */
    double* x = hs;
    for (int i = 0; i < E; ++i) x[i] = 0.0;
    for (int64_t q = offsets[e]; q < offsets[e + 1]; ++q) {
      const float* row = look(ctx, keys[q]);
      if (!row) {
        rc = fail("model: feature key missing from sparse view: ", keys[q], 1);
        break;
      }
      for (int i = 0; i < E; ++i) x[i] += (double)row[i];
    }
    if (rc) break;
    /* run_stack, model.hpp:59-82 */
    for (int l = 0; l < L && rc == 0; ++l) {
      const uint64_t out = dims[l], in = ins[l], off = offs[l];
      const double* h = hs + (uint64_t)l * maxw;
      double* z = zs + (uint64_t)l * maxw;
      for (uint64_t o = 0; o < out; ++o) {
        double acc = (double)W[off + in * out + o];
        const float* row = W + off + o * in;
        for (uint64_t i = 0; i < in; ++i) acc += (double)row[i] * h[i];
        if (!isfinite(acc)) {
          rc = fail("model: non-finite pre-activation", 0, 0);
          break;
        }
        z[o] = acc;
      }
      if (l + 1 < L) {
        double* hn = hs + (uint64_t)(l + 1) * maxw;
        for (uint64_t o = 0; o < out; ++o) hn[o] = z[o] > 0.0 ? z[o] : 0.0;
      }
    }
    if (rc) break;
    /* sigmoid, common.hpp:73 */
    const double p = 1.0 / (1.0 + exp(-zs[(uint64_t)(L - 1) * maxw]));
    preds[t] = p;
    /* backprop, model.hpp:159-180 */
    delta[0] = p - (double)labels[e];
    for (int li = L - 1; li >= 0; --li) {
      const uint64_t out = dims[li], in = ins[li], off = offs[li];
      const double* h = hs + (uint64_t)li * maxw;
      for (uint64_t i = 0; i < in; ++i) dprev[i] = 0.0;
      for (uint64_t o = 0; o < out; ++o) {
        const double dl = delta[o];
        double* gw = dacc + off + o * in;
        const float* row = W + off + o * in;
        for (uint64_t i = 0; i < in; ++i) {
          gw[i] += dl * h[i];
          dprev[i] += (double)row[i] * dl;
        }
        dacc[off + in * out + o] += dl;
      }
      if (li > 0) {
        const double* zp = zs + (uint64_t)(li - 1) * maxw;
        for (uint64_t i = 0; i < in; ++i)
          if (zp[i] <= 0.0) dprev[i] = 0.0;
      }
      memcpy(delta, dprev, in * sizeof(double));
    }
    /* sum-combine sparse accumulate, model.hpp:182-187 */
    for (int64_t q = offsets[e]; q < offsets[e + 1]; ++q) {
      const int64_t u = bsearch_u64(uk, nu, keys[q]);
      double* a = sacc + (uint64_t)u * (uint64_t)E;
      for (int i = 0; i < E; ++i) a[i] += delta[i];
    }
  }
  if (rc == 0) {
    /* model.hpp:189-200 */
    const double inv_n = n == 0 ? 0.0 : 1.0 / (double)n;
    for (uint64_t i = 0; i < nw; ++i) dense_grad[i] = (float)(dacc[i] * inv_n);
    float* sg = (float*)malloc((nu ? nu : 1) * (uint64_t)E * sizeof(float));
    for (uint64_t i = 0; i < nu * (uint64_t)E; ++i)
      sg[i] = (float)(sacc[i] * inv_n);
    *n_uk = nu;
    *uk_out = uk;
    *sg_out = sg;
  } else {
    free(uk);
  }
  free(sacc);
  free(dacc);
  free(hs);
  free(zs);
  free(delta);
  free(dprev);
  return rc;
}

int or_forward_backward(int width, int num_layers, const uint64_t* layer_dims,
                        const float* dense, uint64_t num_examples,
                        const int64_t* offsets, const uint64_t* keys,
                        const uint8_t* labels, const uint64_t* emb_keys,
                        const float* emb_rows, uint64_t n_emb, double* preds,
                        float* dense_grad, float* sparse_grad) {
  uint64_t* idx = (uint64_t*)malloc((num_examples ? num_examples : 1) * 8);
  for (uint64_t i = 0; i < num_examples; ++i) idx[i] = i;
  sorted_view v = {emb_keys, emb_rows, n_emb, width};
  uint64_t nu = 0;
  uint64_t* uk = NULL;
  float* sg = NULL;
  int rc = fb_core(width, num_layers, layer_dims, dense, num_examples, idx,
                   offsets, keys, labels, sorted_lookup, &v, preds, dense_grad,
                   &nu, &uk, &sg);
  free(idx);
  if (rc) return rc;
  memset(sparse_grad, 0, n_emb * (uint64_t)width * sizeof(float));
  for (uint64_t u = 0; u < nu; ++u) {
    const int64_t i = bsearch_u64(emb_keys, n_emb, uk[u]);
    memcpy(sparse_grad + (uint64_t)i * (uint64_t)width,
           sg + u * (uint64_t)width, (uint64_t)width * sizeof(float));
  }
  free(uk);
  free(sg);
  return 0;
}

/* ------------------------------------------------------------ dense sync */

/* hbm_ps.hpp:258-277: replicas ordered node-major then device-major, where
 * node_of(g) = g % N and device_of(g) = g / N (topology.hpp:46-47). */
void or_canonical_sum(int nodes, int devices, const float* bufs, uint64_t len,
                      float* out) {
  for (uint64_t i = 0; i < len; ++i) {
    double acc = 0.0;
    for (int n = 0; n < nodes; ++n)
      for (int d = 0; d < devices; ++d) {
        const int g = d * nodes + n;
        acc += (double)bufs[(uint64_t)g * len + i];
      }
    out[i] = (float)acc;
  }
}

/* hbm_ps.hpp:251-256 then model.hpp:205-212 */
int or_average_apply(float* w, const float* sum, uint64_t len, int count,
                     float lr) {
  for (uint64_t i = 0; i < len; ++i) {
    const float g = sum[i] / (float)count;
    w[i] -= lr * g;
    if (!isfinite(w[i])) return fail("apply_update: non-finite result", 0, 0);
  }
  return 0;
}

/* model.hpp:226-230 then device_table.hpp:94 */
void or_sgd_accumulate(float* v, const float* g, uint64_t len, float lr) {
  for (uint64_t i = 0; i < len; ++i) {
    const float d = -(lr * g[i]);
    v[i] += d;
  }
}

/* Self-pinned Adagrad (see hps_oracle.h): one op at a time, so every f32
 * rounding matches the device's _rn intrinsics (-ffp-contract=off). */
void or_adagrad_apply(float* v, float* s, const float* g, uint64_t len, float lr, float eps) {
  for (uint64_t i = 0; i < len; ++i) {
    const float gg = g[i] * g[i];
    const float acc = s[i] + gg;
    s[i] = acc;
    const float den = sqrtf(acc) + eps;
    const float step = (lr * g[i]) / den;
    v[i] = v[i] - step;
  }
}

/* ------------------------------------------------------ train_reference */

/* FlatStore (oracle.hpp:33-47): key -> embedding, zero-init on first touch.
 * Open addressing over mix64; rows kept in insertion order. */
typedef struct {
  uint64_t* keys;
  uint64_t* slot_row;
  uint64_t cap, n;
  float* rows;
  uint64_t rows_cap;
  int E;
} flat_store;

static void fs_init(flat_store* s, int E) {
  s->cap = 1024;
  s->n = 0;
  s->E = E;
  s->keys = (uint64_t*)malloc(s->cap * 8);
  s->slot_row = (uint64_t*)malloc(s->cap * 8);
  for (uint64_t i = 0; i < s->cap; ++i) s->keys[i] = OR_EMPTY;
  s->rows_cap = 512;
  s->rows = (float*)malloc(s->rows_cap * (uint64_t)E * sizeof(float));
}

static void fs_free(flat_store* s) {
  free(s->keys);
  free(s->slot_row);
  free(s->rows);
}

static int64_t fs_find(const flat_store* s, uint64_t key) {
  uint64_t i = or_mix64(key) & (s->cap - 1);
  for (;;) {
    if (s->keys[i] == key) return (int64_t)s->slot_row[i];
    if (s->keys[i] == OR_EMPTY) return -1;
    i = (i + 1) & (s->cap - 1);
  }
}

static void fs_put_slot(flat_store* s, uint64_t key, uint64_t row) {
  uint64_t i = or_mix64(key) & (s->cap - 1);
  while (s->keys[i] != OR_EMPTY) i = (i + 1) & (s->cap - 1);
  s->keys[i] = key;
  s->slot_row[i] = row;
}

static float* fs_get_or_init(flat_store* s, uint64_t key) {
  int64_t r = fs_find(s, key);
  if (r >= 0) return s->rows + (uint64_t)r * (uint64_t)s->E;
  if ((s->n + 1) * 2 > s->cap) {
    uint64_t* ok = s->keys;
    uint64_t* orow = s->slot_row;
    const uint64_t ocap = s->cap;
    s->cap *= 2;
    s->keys = (uint64_t*)malloc(s->cap * 8);
    s->slot_row = (uint64_t*)malloc(s->cap * 8);
    for (uint64_t i = 0; i < s->cap; ++i) s->keys[i] = OR_EMPTY;
    for (uint64_t i = 0; i < ocap; ++i)
      if (ok[i] != OR_EMPTY) fs_put_slot(s, ok[i], orow[i]);
    free(ok);
    free(orow);
  }
  if (s->n == s->rows_cap) {
    s->rows_cap *= 2;
    s->rows = (float*)realloc(s->rows, s->rows_cap * (uint64_t)s->E * 4);
  }
  const uint64_t row = s->n++;
  memset(s->rows + row * (uint64_t)s->E, 0, (uint64_t)s->E * sizeof(float));
  fs_put_slot(s, key, row);
  return s->rows + row * (uint64_t)s->E;
}

static const float* fs_lookup(void* ctx, uint64_t key) {
  flat_store* s = (flat_store*)ctx;
  const int64_t r = fs_find(s, key);
  return r < 0 ? NULL : s->rows + (uint64_t)r * (uint64_t)s->E;
}

typedef struct {
  uint64_t nu;
  uint64_t* uk;
  float* sg;
  float* dense;
} shard_grad;

/* oracle.hpp:55-122 */
int or_train_reference(const or_cfg* c, uint64_t batch_size,
                       uint64_t num_examples, const int64_t* offsets,
                       const uint64_t* keys, const uint8_t* labels,
                       float* dense_out, uint64_t* n_sparse_out,
                       uint64_t* sparse_keys_out, float* sparse_rows_out,
                       uint64_t sparse_cap) {
  const int N = c->nodes, D = c->devices, G = N * D, J = c->minibatches;
  const int E = c->embedding_dim;
  const int adagrad = c->optimizer == 1;
  const int RW = adagrad ? 2 * E : E; /* store row: embedding (+ state) */
  const float lr = c->learning_rate;
  const uint64_t nw = or_dense_count(E, c->num_layers, c->layer_dims);
  const uint64_t nbatches = (num_examples + batch_size - 1) / batch_size;
  const uint64_t steps = (nbatches + (uint64_t)N - 1) / (uint64_t)N;
  int rc = 0;

  flat_store st;
  fs_init(&st, RW);
  or_init_dense(c, dense_out);

  shard_grad* grads = (shard_grad*)calloc((size_t)G, sizeof(shard_grad));
  float* dbufs = (float*)malloc((uint64_t)G * nw * sizeof(float));
  float* dsum = (float*)malloc(nw * sizeof(float));
  uint64_t* ex_idx = (uint64_t*)malloc((batch_size ? batch_size : 1) * 8);

  for (uint64_t t = 0; t < steps && rc == 0; ++t) {
    /* zero-init every referenced key up front (oracle.hpp:80-83) */
    for (int n = 0; n < N; ++n) {
      const uint64_t bi = t * (uint64_t)N + (uint64_t)n;
      if (bi >= nbatches) continue;
      const uint64_t b0 = bi * batch_size;
      const uint64_t b1 = b0 + batch_size < num_examples ? b0 + batch_size
                                                         : num_examples;
      for (int64_t q = offsets[b0]; q < offsets[b1]; ++q)
        (void)fs_get_or_init(&st, keys[q]);
    }
    for (int j = 0; j < J && rc == 0; ++j) {
      for (int n = 0; n < N && rc == 0; ++n) {
        const uint64_t bi = t * (uint64_t)N + (uint64_t)n;
        uint64_t b0 = 0, bn = 0;
        if (bi < nbatches) {
          b0 = bi * batch_size;
          bn = (b0 + batch_size < num_examples ? b0 + batch_size
                                               : num_examples) - b0;
        }
        for (int d = 0; d < D && rc == 0; ++d) {
          const int g = d * N + n;
          /* shard_batch: slot i % (D*J) == d*J + j, sharding.hpp:36-40 */
          uint64_t m = 0;
          const uint64_t slots = (uint64_t)D * (uint64_t)J;
          for (uint64_t i = (uint64_t)d * (uint64_t)J + (uint64_t)j; i < bn;
               i += slots)
            ex_idx[m++] = b0 + i;
          shard_grad* sgp = &grads[g];
          sgp->dense = dbufs + (uint64_t)g * nw;
          sgp->nu = 0;
          sgp->uk = NULL;
          sgp->sg = NULL;
          if (m > 0) {
            double* preds = (double*)malloc(m * sizeof(double));
            rc = fb_core(E, c->num_layers, c->layer_dims, dense_out, m, ex_idx,
                         offsets, keys, labels, fs_lookup, &st, preds,
                         sgp->dense, &sgp->nu, &sgp->uk, &sgp->sg);
            free(preds);
          } else {
            memset(sgp->dense, 0, nw * sizeof(float));
          }
        }
      }
      if (rc) break;
      /* sparse deltas applied node-major, device-major (oracle.hpp:102-112) */
      for (int n = 0; n < N; ++n)
        for (int d = 0; d < D; ++d) {
          const shard_grad* sgp = &grads[d * N + n];
          for (uint64_t u = 0; u < sgp->nu; ++u) {
            float* p = fs_get_or_init(&st, sgp->uk[u]);
            if (adagrad)
              or_adagrad_apply(p, p + E, sgp->sg + u * (uint64_t)E, (uint64_t)E, lr,
                               c->adagrad_eps);
            else
              or_sgd_accumulate(p, sgp->sg + u * (uint64_t)E, (uint64_t)E, lr);
          }
        }
      for (int g = 0; g < G; ++g) {
        free(grads[g].uk);
        free(grads[g].sg);
        grads[g].uk = NULL;
        grads[g].sg = NULL;
      }
      /* dense: canonical sum, average, apply (oracle.hpp:114-118) */
      or_canonical_sum(N, D, dbufs, nw, dsum);
      rc = or_average_apply(dense_out, dsum, nw, G, lr);
    }
  }

  if (rc == 0) {
    /* export sorted by key */
    uint64_t* ks = (uint64_t*)malloc((st.n ? st.n : 1) * 8);
    uint64_t m = 0;
    for (uint64_t i = 0; i < st.cap; ++i)
      if (st.keys[i] != OR_EMPTY) ks[m++] = st.keys[i];
    qsort(ks, m, 8, cmp_u64);
    if (m > sparse_cap) {
      rc = fail("oracle: sparse output capacity too small", 0, 0);
    } else {
      for (uint64_t i = 0; i < m; ++i) {
        sparse_keys_out[i] = ks[i];
        memcpy(sparse_rows_out + i * (uint64_t)RW, fs_lookup(&st, ks[i]),
               (uint64_t)RW * sizeof(float));
      }
      *n_sparse_out = m;
    }
    free(ks);
  }
  for (int g = 0; g < G; ++g) {
    free(grads[g].uk);
    free(grads[g].sg);
  }
  free(grads);
  free(dbufs);
  free(dsum);
  free(ex_idx);
  fs_free(&st);
  return rc;
}

/* ------------------------------------------------------------------- auc */

static const double* g_scores;
static int cmp_idx_score(const void* a, const void* b) {
  const double x = g_scores[*(const uint64_t*)a], y = g_scores[*(const uint64_t*)b];
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* model.hpp:245-270 */
double or_auc(const uint8_t* labels, const double* scores, uint64_t n) {
  uint64_t npos = 0;
  for (uint64_t i = 0; i < n; ++i) npos += labels[i] != 0;
  const uint64_t nneg = n - npos;
  if (npos == 0 || nneg == 0) return NAN;
  uint64_t* idx = (uint64_t*)malloc(n * 8);
  for (uint64_t i = 0; i < n; ++i) idx[i] = i;
  g_scores = scores;
  qsort(idx, n, 8, cmp_idx_score);
  double pos_rank_sum = 0.0;
  uint64_t i = 0;
  while (i < n) {
    uint64_t j = i;
    while (j < n && scores[idx[j]] == scores[idx[i]]) ++j;
    const double avg_rank = 0.5 * (double)(i + 1 + j);
    for (uint64_t t = i; t < j; ++t)
      if (labels[idx[t]]) pos_rank_sum += avg_rank;
    i = j;
  }
  free(idx);
  return (pos_rank_sum - 0.5 * (double)npos * (double)(npos + 1)) /
         ((double)npos * (double)nneg);
}

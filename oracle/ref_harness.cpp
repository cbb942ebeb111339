// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// A C-ABI shim around the UNMODIFIED reference headers (compiled in place
// from /root/reference/proj/include by oracle/Makefile; nothing is copied).
// Output: oracle/_ref/libhps_ref.so. Used by
//   * tests/golden/make_golden.py to produce the committed golden fixtures,
//   * bench.py --impl reference / the cpu_baseline leg (the reference HBM-PS
//     hot path timed on host cores).
//
// Reference symbols exercised (file:line under /root/reference/proj/include):
//   gen_dataset / to_batches          hps/dataset.hpp:96-108,180-227
//   MemPs::extract_working_set        hps/mem_ps.hpp:101-108
//   DeviceTable insert/for_each       hps/device_table.hpp:38-101
//   HbmTier build/get/push/drain/dump hps/hbm_ps.hpp:61-232
//   SyncSession / canonical_sum       hps/hbm_ps.hpp:258-408
//   forward/backward/sgd_delta/...    hps/model.hpp:42-230
//   train_reference                   hps/oracle.hpp:55-122
//   device-worker loop body           hps/pipeline.hpp:502-566
#include <algorithm>
#include <chrono>
#include <cstring>
#include <thread>
#include <unordered_map>

#include "hps/common.hpp"
#include "hps/config.hpp"
#include "hps/dataset.hpp"
#include "hps/device_table.hpp"
#include "hps/hbm_ps.hpp"
#include "hps/mem_ps.hpp"
#include "hps/model.hpp"
#include "hps/oracle.hpp"
#include "hps/pipeline.hpp"
#include "hps/sharding.hpp"
#include "hps/ssd_ps.hpp"
#include "hps/topology.hpp"
#include "hps/transport.hpp"

using namespace hps;

namespace {

thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefCfg {
  int nodes;
  int devices;
  int embedding_dim;
  int num_layers;
  std::uint64_t layer_dims[8];
  float learning_rate;
  std::uint64_t seed;
  int minibatches;
  int deterministic;
  std::int64_t inject_skip_sync;
};

RunConfig to_run_config(const RefCfg* c, std::size_t batch_size) {
  RunConfig rc;
  rc.nodes = c->nodes;
  rc.devices_per_node = c->devices;
  rc.embedding_dim = std::size_t(c->embedding_dim);
  rc.layer_dims.assign(c->layer_dims, c->layer_dims + c->num_layers);
  rc.learning_rate = c->learning_rate;
  rc.seed = c->seed;
  rc.batch_size = batch_size;
  rc.minibatches_per_batch = c->minibatches;
  rc.deterministic = c->deterministic != 0;
  rc.inject_skip_sync = c->inject_skip_sync;
  return rc;
}

std::vector<Batch> csr_to_batches(std::size_t num_examples,
                                  const std::int64_t* offsets,
                                  const std::uint64_t* keys,
                                  const std::uint8_t* labels,
                                  std::size_t batch_size) {
  Dataset ds;
  ds.examples.resize(num_examples);
  for (std::size_t i = 0; i < num_examples; ++i) {
    ds.examples[i].label = labels[i];
    ds.examples[i].features.assign(keys + offsets[i], keys + offsets[i + 1]);
  }
  return to_batches(ds, batch_size);
}

void export_sparse(const std::unordered_map<ParamKey, std::vector<float>>& m,
                   std::size_t width, std::uint64_t* n_out,
                   std::uint64_t* keys_out, float* rows_out,
                   std::uint64_t cap) {
  std::vector<ParamKey> ks;
  ks.reserve(m.size());
  for (const auto& [k, v] : m) ks.push_back(k);
  std::sort(ks.begin(), ks.end());
  *n_out = ks.size();
  check(ks.size() <= cap, "ref harness: sparse output capacity too small");
  for (std::size_t i = 0; i < ks.size(); ++i) {
    keys_out[i] = ks[i];
    const auto& v = m.at(ks[i]);
    std::memcpy(rows_out + i * width, v.data(), width * sizeof(float));
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// dataset.hpp:180-227 with a fixed nnz per example: keys has n*nnz entries.
int ref_gen_dataset(std::uint64_t dims, std::uint64_t num_examples,
                    std::uint64_t nnz, int zipf, double zipf_s,
                    std::uint64_t seed, double signal_scale,
                    std::uint64_t clusters, std::int64_t* offsets,
                    std::uint64_t* keys, std::uint8_t* labels) {
  return guarded([&] {
    GenSpec s;
    s.dims = dims;
    s.num_examples = num_examples;
    s.nnz = nnz;
    s.dist = zipf ? KeyDist::kZipf : KeyDist::kUniform;
    s.zipf_s = zipf_s;
    s.seed = seed;
    s.signal_scale = signal_scale;
    s.clusters = clusters;
    const Dataset ds = gen_dataset(s);
    std::int64_t off = 0;
    for (std::size_t i = 0; i < ds.examples.size(); ++i) {
      offsets[i] = off;
      labels[i] = std::uint8_t(ds.examples[i].label);
      for (ParamKey k : ds.examples[i].features) keys[off++] = k;
    }
    offsets[ds.examples.size()] = off;
  });
}

// mem_ps.hpp:101-108
int ref_working_set(std::size_t num_examples, const std::int64_t* offsets,
                    const std::uint64_t* keys, std::uint64_t* out,
                    std::uint64_t* n_out) {
  return guarded([&] {
    Batch b;
    b.examples.resize(num_examples);
    for (std::size_t i = 0; i < num_examples; ++i)
      b.examples[i].features.assign(keys + offsets[i], keys + offsets[i + 1]);
    const auto ws = MemPs::extract_working_set(b);
    std::copy(ws.begin(), ws.end(), out);
    *n_out = ws.size();
  });
}

// device_table.hpp:38-101: insert `keys` in the given order into a table
// sized for n keys; report capacity and the keys in slot order (for_each).
int ref_table_slot_order(const std::uint64_t* keys, std::size_t n,
                         std::uint64_t* slot_order_out,
                         std::uint64_t* capacity_out) {
  return guarded([&] {
    DeviceTable t(n, 1);
    for (std::size_t i = 0; i < n; ++i) {
      const float v = float(i);
      t.insert(keys[i], &v);
    }
    std::size_t j = 0;
    t.for_each([&](ParamKey k, const float*) { slot_order_out[j++] = k; });
    *capacity_out = t.capacity();
  });
}

// hbm_ps.hpp:65-102 with PartitionPolicy::modulo: per global device the
// owned keys of the merged working set, ascending. out_g[i] = owner of
// sorted-unique key i; returns the sorted unique keys too.
int ref_partition(int nodes, int devices, const std::uint64_t* keys,
                  std::size_t n, std::uint64_t* uniq_out, std::int32_t* g_out,
                  std::uint64_t* n_out) {
  return guarded([&] {
    Topology topo(nodes, devices);
    Transport tr;
    HbmTier hbm(topo, PartitionPolicy::modulo(topo), 1, &tr);
    std::vector<ParamKey> ks(keys, keys + n);
    hbm.build_all({ks}, [](ParamKey k) { return std::vector<float>{float(k)}; });
    std::map<ParamKey, int> owner;
    for (int g = 0; g < topo.total_devices(); ++g)
      hbm.table_at(g)->for_each(
          [&](ParamKey k, const float*) { owner.emplace(k, g); });
    std::size_t i = 0;
    for (const auto& [k, g] : owner) {
      uniq_out[i] = k;
      g_out[i] = g;
      ++i;
    }
    *n_out = i;
  });
}

// hbm_ps.hpp:258-277 (canonical_sum) + 249-256 (average_by) +
// model.hpp:205-222 (apply_update): bufs is G x len, replicas in global
// index order.
int ref_canonical_sum(int nodes, int devices, const float* bufs,
                      std::size_t len, float* sum_out) {
  return guarded([&] {
    Topology topo(nodes, devices);
    const int G = topo.total_devices();
    std::vector<std::vector<float>> parts(G);
    for (int g = 0; g < G; ++g) parts[g].assign(bufs + g * len, bufs + (g + 1) * len);
    std::vector<std::pair<int, const std::vector<float>*>> view;
    for (int g = 0; g < G; ++g) view.emplace_back(g, &parts[g]);
    const auto s = canonical_sum(std::move(view), topo);
    std::copy(s.begin(), s.end(), sum_out);
  });
}

int ref_synchronize(int nodes, int devices, int det, float* bufs,
                    std::size_t len) {
  return guarded([&] {
    Topology topo(nodes, devices);
    Transport tr;
    const int G = topo.total_devices();
    for (int g = 0; g < G; ++g) tr.register_endpoint(topo.endpoint_of(g));
    std::vector<std::vector<float>> b(G);
    for (int g = 0; g < G; ++g) b[g].assign(bufs + g * len, bufs + (g + 1) * len);
    synchronize(b, topo, &tr, det != 0);
    for (int g = 0; g < G; ++g) std::copy(b[g].begin(), b[g].end(), bufs + g * len);
  });
}

int ref_init_dense(const RefCfg* c, float* out, std::uint64_t* n_out) {
  return guarded([&] {
    const auto d = init_dense(to_run_config(c, 1).model());
    std::copy(d.weights.begin(), d.weights.end(), out);
    *n_out = d.weights.size();
  });
}

// model.hpp:101-202 on one shard: emb rows given for the sorted unique keys.
int ref_forward_backward(int width, int num_layers,
                         const std::uint64_t* layer_dims, const float* dense,
                         std::size_t num_examples, const std::int64_t* offsets,
                         const std::uint64_t* keys, const std::uint8_t* labels,
                         const std::uint64_t* emb_keys, const float* emb_rows,
                         std::size_t n_emb, double* preds_out,
                         float* dense_grad_out, float* sparse_grad_out) {
  return guarded([&] {
    DenseParams d;
    d.input_dim = std::size_t(width);
    d.layer_dims.assign(layer_dims, layer_dims + num_layers);
    d.weights.assign(dense, dense + DenseParams::weight_count(d.input_dim, d.layer_dims));
    std::map<ParamKey, const float*> emb;
    for (std::size_t i = 0; i < n_emb; ++i) emb[emb_keys[i]] = emb_rows + i * width;
    std::vector<Example> ex(num_examples);
    for (std::size_t i = 0; i < num_examples; ++i) {
      ex[i].label = labels[i];
      ex[i].features.assign(keys + offsets[i], keys + offsets[i + 1]);
    }
    auto emb_of = [&](ParamKey k) -> const float* {
      auto it = emb.find(k);
      return it == emb.end() ? nullptr : it->second;
    };
    const auto preds = forward(ex, emb_of, d);
    const auto g = backward(ex, emb_of, d, preds);
    std::copy(preds.begin(), preds.end(), preds_out);
    std::copy(g.dense.begin(), g.dense.end(), dense_grad_out);
    // sparse grads in emb_keys order (caller passes the sorted union)
    for (std::size_t i = 0; i < n_emb; ++i) {
      auto it = g.sparse.find(emb_keys[i]);
      check(it != g.sparse.end(), "ref harness: key not in sparse grads");
      std::copy(it->second.begin(), it->second.end(), sparse_grad_out + i * width);
    }
  });
}

// oracle.hpp:55-122 over to_batches(ds, batch_size).
int ref_train_reference(const RefCfg* c, std::size_t batch_size,
                        std::size_t num_examples, const std::int64_t* offsets,
                        const std::uint64_t* keys, const std::uint8_t* labels,
                        float* dense_out, std::uint64_t* n_sparse_out,
                        std::uint64_t* sparse_keys_out, float* sparse_rows_out,
                        std::uint64_t sparse_cap) {
  return guarded([&] {
    const RunConfig rc = to_run_config(c, batch_size);
    const auto batches = csr_to_batches(num_examples, offsets, keys, labels, batch_size);
    const FlatStore st = train_reference(rc, batches);
    std::copy(st.dense.weights.begin(), st.dense.weights.end(), dense_out);
    std::unordered_map<ParamKey, std::vector<float>> m;
    for (const auto& [k, p] : st.sparse) m.emplace(k, p.embedding);
    export_sparse(m, rc.embedding_dim, n_sparse_out, sparse_keys_out, sparse_rows_out, sparse_cap);
  });
}

// The reference HBM-PS hot path as BASELINE.md §3 defines the CPU baseline:
// per batch extract_working_set -> HbmTier::build_all (flat-map host store,
// zero on first touch) -> one std::thread per device running the device
// worker loop body (pipeline.hpp:515-559) with AbortableBarrier and
// SyncSession -> dump_node written back to the host store. MEM-PS/SSD are
// excluded (cache.hpp:187-210 makes them unusable at this scale).
// nodes must be 1. Runs batches [first_batch, first_batch + n_batches) of
// to_batches(ds); elapsed_ms_out gets the wall time of those batches.
// If the *_out pointers are non-null the final host store is exported.
struct RefHotPath {
  RunConfig rc;
  std::unordered_map<ParamKey, std::vector<float>> store;
  DenseParams dense0;
  std::vector<DenseParams> replicas;
  std::unique_ptr<Transport> tr;
  std::unique_ptr<HbmTier> hbm;
  std::unique_ptr<SyncSession> sync;
  std::vector<Batch> batches;
  std::int64_t step = 0;
};

void* ref_hot_path_create(const RefCfg* c, std::size_t batch_size,
                          std::size_t num_examples, const std::int64_t* offsets,
                          const std::uint64_t* keys, const std::uint8_t* labels) {
  RefHotPath* h = nullptr;
  const int rcode = guarded([&] {
    check(c->nodes == 1, "ref hot path: nodes must be 1");
    auto p = std::make_unique<RefHotPath>();
    p->rc = to_run_config(c, batch_size);
    p->rc.validate();
    const Topology topo = p->rc.topology();
    p->tr = std::make_unique<Transport>();
    p->hbm = std::make_unique<HbmTier>(topo, PartitionPolicy::modulo(topo),
                                       p->rc.embedding_dim, p->tr.get());
    p->sync = std::make_unique<SyncSession>(topo, p->tr.get(), p->rc.deterministic);
    p->replicas = replicate_dense(init_dense(p->rc.model()), topo);
    p->batches = csr_to_batches(num_examples, offsets, keys, labels, batch_size);
    h = p.release();
  });
  return rcode == 0 ? h : nullptr;
}

void ref_hot_path_destroy(void* p) { delete static_cast<RefHotPath*>(p); }

int ref_hot_path_run(void* p, std::size_t first_batch, std::size_t n_batches,
                     double* elapsed_ms_out) {
  auto* h = static_cast<RefHotPath*>(p);
  return guarded([&] {
    const Topology topo = h->rc.topology();
    const int workers = topo.total_devices();
    const int J = h->rc.minibatches_per_batch;
    const std::size_t width = h->rc.embedding_dim;
    const float lr = h->rc.learning_rate;
    const auto t0 = std::chrono::steady_clock::now();
    for (std::size_t bi = first_batch; bi < first_batch + n_batches; ++bi) {
      const Batch& batch = h->batches.at(bi % h->batches.size());
      const auto working = MemPs::extract_working_set(batch);
      h->hbm->build_node(0, {working}, [&](ParamKey k) {
        auto it = h->store.find(k);
        if (it != h->store.end()) return it->second;
        return std::vector<float>(width, 0.0f);
      });
      const auto shards = shard_batch(batch, topo.devices_per_node, J);
      AbortableBarrier barrier(workers);
      std::vector<std::thread> threads;
      std::exception_ptr err;
      std::mutex err_mu;
      const std::int64_t t = h->step;
      for (int g = 0; g < workers; ++g) {
        threads.emplace_back([&, g] {
          try {
            const Endpoint ep = topo.endpoint_of(g);
            DenseParams& dense = h->replicas[g];
            const auto& mine = shards[topo.device_of(g)];
            for (int j = 0; j < J; ++j) {
              const auto& examples = mine[j];
              std::vector<ParamKey> ks;
              for (const Example& ex : examples)
                ks.insert(ks.end(), ex.features.begin(), ex.features.end());
              std::sort(ks.begin(), ks.end());
              ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
              auto params = h->hbm->get(ks, ep);
              if (!barrier.arrive_and_wait()) return;
              std::vector<float> dense_grad(dense.weights.size(), 0.0f);
              if (!examples.empty()) {
                auto emb_of = [&](ParamKey k) -> const float* {
                  auto it = params.find(k);
                  return it == params.end() ? nullptr : it->second.data();
                };
                const auto preds = forward(examples, emb_of, dense);
                auto grad = backward(examples, emb_of, dense, preds);
                dense_grad = std::move(grad.dense);
                std::map<ParamKey, std::vector<float>> deltas;
                for (auto& [k, gk] : grad.sparse) deltas.emplace(k, sgd_delta(gk, lr));
                h->hbm->push_deltas(deltas, ep);
              }
              if (!barrier.arrive_and_wait()) return;
              h->hbm->drain_accums(ep);
              const std::int64_t global_mb = t * J + j;
              if (global_mb != h->rc.inject_skip_sync) {
                h->sync->run(g, dense_grad);
                apply_update(dense, average_by(dense_grad, workers), lr);
              }
              if (!barrier.arrive_and_wait()) return;
            }
          } catch (...) {
            std::lock_guard lk(err_mu);
            if (!err) err = std::current_exception();
            barrier.abort();
          }
        });
      }
      for (auto& th : threads) th.join();
      if (err) std::rethrow_exception(err);
      for (auto& [k, v] : h->hbm->dump_node(0)) h->store[k] = v;
      ++h->step;
    }
    *elapsed_ms_out = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0).count();
  });
}

int ref_hot_path_export(void* p, float* dense_out, std::uint64_t* n_sparse_out,
                        std::uint64_t* sparse_keys_out, float* sparse_rows_out,
                        std::uint64_t sparse_cap) {
  auto* h = static_cast<RefHotPath*>(p);
  return guarded([&] {
    const auto& w = h->replicas[0].weights;
    std::copy(w.begin(), w.end(), dense_out);
    export_sparse(h->store, h->rc.embedding_dim, n_sparse_out, sparse_keys_out,
                  sparse_rows_out, sparse_cap);
  });
}

// ---- parameter files: the reference SsdStore itself (ssd_ps.hpp) ----------

// SsdStore::dump of (key, emb, opt) records into a fresh directory: the
// reference's own bytes, to compare ours against.
int ref_store_dump(const char* dir, std::uint64_t width, std::uint64_t file_capacity,
                   const std::uint64_t* keys, const float* emb, const float* opt,
                   std::uint64_t n) {
  return guarded([&] {
    StoreConfig sc;
    sc.dir = dir;
    sc.embedding_dim = width;
    sc.file_capacity = file_capacity;
    sc.background_compaction = false;
    SsdStore st(sc);
    std::map<ParamKey, SparseParam> m;
    for (std::uint64_t i = 0; i < n; ++i) {
      SparseParam p(width);
      std::copy(emb + i * width, emb + (i + 1) * width, p.embedding.begin());
      if (opt) std::copy(opt + i * width, opt + (i + 1) * width, p.opt_state.begin());
      m.emplace(keys[i], std::move(p));
    }
    st.dump(m);
  });
}

// SsdStore recover + load of every key + fsck + stats on an existing
// directory (width 0 = inferred from the files). Records come back in key
// order. info[0..5] = files, live_records, stale_records, fsck ok,
// fsck files_scanned, recovered_invalid_files.
int ref_store_load_all(const char* dir, std::uint64_t width, std::uint64_t* keys, float* emb,
                       float* opt, std::uint64_t cap, std::uint64_t* n_out,
                       std::uint64_t* info) {
  return guarded([&] {
    StoreConfig sc;
    sc.dir = dir;
    sc.embedding_dim = width;
    sc.background_compaction = false;
    SsdStore st(sc);
    auto all = st.all_keys();
    std::sort(all.begin(), all.end());
    check(all.size() <= cap, "ref_store_load_all: cap");
    const auto res = st.load(all);
    check(res.missing.empty(), "ref_store_load_all: missing keys");
    const std::size_t w = st.embedding_dim();
    std::uint64_t i = 0;
    for (const auto& [k, p] : res.found) {
      keys[i] = k;
      std::copy(p.embedding.begin(), p.embedding.end(), emb + i * w);
      std::copy(p.opt_state.begin(), p.opt_state.end(), opt + i * w);
      ++i;
    }
    *n_out = i;
    const auto s = st.stats();
    const auto f = st.fsck();
    info[0] = s.files;
    info[1] = s.live_records;
    info[2] = s.stale_records;
    info[3] = f.ok ? 1 : 0;
    info[4] = f.files_scanned;
    info[5] = s.recovered_invalid_files;
  });
}

}  // extern "C"

// The reference API unchanged (include/hps_gpu/hbm_ps.hpp, namespace hps)
// driven the way the reference drives it:
//   1. ports of the reference's HbmTier unit cases (test_hbm_ps.cpp:104-177:
//      carry-over, pull union, missing key, routed accumulate, concurrent
//      push/drain) on G devices of this process;
//   2. the device-worker loop of pipeline.hpp:502-566 — one std::thread per
//      global device calling get / push_deltas / drain_accums /
//      SyncSession::run / apply_update in lockstep — with the train stage's
//      build_node / dump_node between batches (pipeline.hpp:425-445), checked
//      bit for bit against the oracle's train_reference (oracle.hpp:55-122).
// With G = 2 the two handles live in one process: their NVLink windows are
// mapped through same-process peer access (tier.cu setup_p2p) and the dense
// sync runs over them.
//   usage: test_hps_compat [G]      (G GPUs, default 1)
#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <thread>
#include <vector>

#include "../../oracle/hps_oracle.h"
#include "hps_gpu/hbm_ps.hpp"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (cond) {                                                   \
      ++g_pass;                                                   \
    } else {                                                      \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

using namespace hps;

static void unit_cases(int G) {
  const Topology topo(1, G);
  Transport::Options o;
  o.max_batch_keys = 4096;
  Transport tr(topo, 2, o);
  HbmTier tier(topo, PartitionPolicy::modulo(topo), 2, &tr);
  bool threw = false;
  try {
    tier.get({1}, Endpoint{0, 0});
  } catch (const Error& e) {
    threw = std::strstr(e.what(), "hbm: tables not built") != nullptr;
  }
  CHECK(threw);
  // build from host values, then carry-over keeps the device value
  // (test_hbm_ps.cpp:104-116): host_value is not asked for carried keys
  tier.build_all({{1, 2, 3, 4, 5, 6, 7, 8}},
                 [](ParamKey k) { return std::vector<float>{float(k), 0.5f}; });
  tier.accumulate({{3, {9.0f, 0.0f}}}, Endpoint{0, 0});
  int asked = 0;
  tier.build_all({{3, 4, 100}}, [&](ParamKey k) {
    ++asked;
    return std::vector<float>{float(k) * 2, 1.0f};
  });
  CHECK(asked == 1);  // only key 100 (3 and 4 carried over)
  auto v = tier.get({100, 3, 4}, Endpoint{0, G - 1});
  CHECK(v.size() == 3);
  CHECK((v[3] == std::vector<float>{12.0f, 0.5f}));
  CHECK((v[4] == std::vector<float>{4.0f, 0.5f}));
  CHECK((v[100] == std::vector<float>{200.0f, 1.0f}));
  CHECK(tier.table_at(int(3 % G))->contains(3));
  CHECK(!tier.table_at(0)->contains(1));
  threw = false;
  try {  // missing key (test_hbm_ps.cpp:137)
    tier.get({5}, Endpoint{0, 0});
  } catch (const Error& e) {
    threw = std::strstr(e.what(), "device table: missing key 5") != nullptr;
  }
  CHECK(threw);
  // concurrent push from every device, then drain (test_hbm_ps.cpp:157-177):
  // 64 x +1 on each key from each sender is exact
  std::vector<std::thread> th;
  for (int g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      for (int r = 0; r < 64; ++r)
        tier.push_deltas({{3, {1.0f, 0.0f}}, {4, {0.0f, 1.0f}}, {100, {1.0f, 1.0f}}},
                         topo.endpoint_of(g));
    });
  for (auto& t : th) t.join();
  for (int g = 0; g < G; ++g) tier.drain_accums(topo.endpoint_of(g));
  auto w = tier.get({3, 4, 100}, Endpoint{0, 0});
  CHECK((w[3] == std::vector<float>{12.0f + 64.0f * G, 0.5f}));
  CHECK((w[4] == std::vector<float>{4.0f, 0.5f + 64.0f * G}));
  CHECK((w[100] == std::vector<float>{200.0f + 64.0f * G, 1.0f + 64.0f * G}));
  auto d = tier.dump_node(0);
  CHECK(d.size() == 3 && d.begin()->first == 3);
  // dense sync: 1..G sums to G(G+1)/2 on every device (test_hbm_ps.cpp:179-192)
  std::vector<std::vector<float>> bufs(G);
  for (int g = 0; g < G; ++g) bufs[g] = {float(g + 1), float(10 * (g + 1))};
  synchronize(bufs, topo, &tr, true);
  for (int g = 0; g < G; ++g) {
    CHECK(bufs[g][0] == float(G * (G + 1) / 2));
    CHECK(bufs[g][1] == float(10 * G * (G + 1) / 2));
  }
}

// test_hbm_ps.cpp:42-60: the worked range split — keys <= 50 on device 0,
// the rest on device 1, then get/accumulate routed by the same policy.
static void range_split_case(int G) {
  const Topology topo(1, G);
  Transport::Options o;
  o.max_batch_keys = 64;
  Transport tr(topo, 1, o);
  HbmTier hbm(topo, PartitionPolicy::range_split(50), 1, &tr);
  const std::vector<ParamKey> keys = {4, 5, 11, 50, 53, 56, 61, 87, 98};
  auto keyed = [](ParamKey k) { return std::vector<float>{float(k)}; };
  if (G < 2) {  // the policy names device 1, which a 1-device topology lacks
    bool threw = false;
    try {
      hbm.build_all({keys}, keyed);
    } catch (const Error& e) {
      threw = std::strstr(e.what(), "on device 1 of 1") != nullptr;
    }
    CHECK(threw);
    return;
  }
  hbm.build_all({keys}, keyed);
  std::vector<ParamKey> dev0, dev1;
  hbm.table_at(0, 0)->for_each([&](ParamKey k, const float* v) {
    dev0.push_back(k);
    CHECK(v[0] == float(k));
  });
  hbm.table_at(0, 1)->for_each([&](ParamKey k, const float*) { dev1.push_back(k); });
  std::sort(dev0.begin(), dev0.end());
  std::sort(dev1.begin(), dev1.end());
  CHECK((dev0 == std::vector<ParamKey>{4, 5, 11, 50}));
  CHECK((dev1 == std::vector<ParamKey>{53, 56, 61, 87, 98}));
  hbm.accumulate({{50, {0.5f}}, {53, {0.25f}}}, Endpoint{0, 0});
  auto v = hbm.get({53, 50, 4}, Endpoint{0, 1});
  CHECK((v[50] == std::vector<float>{50.5f}));
  CHECK((v[53] == std::vector<float>{53.25f}));
  CHECK((v[4] == std::vector<float>{4.0f}));
  CHECK(hbm.table_at(1)->contains(53) && !hbm.table_at(0)->contains(53));
}

// pipeline.hpp:502-566 over the hps:: API, vs oracle train_reference.
static void device_worker_loop(int G) {
  const int E = 8, J = 4, L = 3;
  const std::uint64_t dims[3] = {8, 16, 1};
  const std::uint64_t dims_n = 20000, B = 512, NB = 3, nnz = 20;
  std::vector<std::int64_t> off(NB * B + 1);
  std::vector<std::uint64_t> keys(NB * B * nnz);
  std::vector<std::uint8_t> lab(NB * B);
  hps_gen_dataset(dims_n, NB * B, nnz, 1, 1.0, 5, 6.0, 0, off.data(), keys.data(), lab.data());
  or_cfg cfg{};
  cfg.nodes = 1, cfg.devices = G, cfg.embedding_dim = E, cfg.num_layers = L;
  for (int l = 0; l < L; ++l) cfg.layer_dims[l] = dims[l];
  cfg.learning_rate = 0.05f, cfg.seed = 42, cfg.minibatches = J, cfg.deterministic = 1;
  cfg.inject_skip_sync = -1;
  const std::uint64_t nw = or_dense_count(E, L, dims);
  std::vector<float> dense0(nw);
  or_init_dense(&cfg, dense0.data());

  const Topology topo(1, G);
  Transport::Options o;
  o.max_batch_keys = B * nnz;
  o.key_space = dims_n;
  Transport tr(topo, E, o);
  HbmTier tier(topo, PartitionPolicy::modulo(topo), E, &tr);
  SyncSession sync(topo, &tr, true);
  std::vector<std::vector<float>> dense(G, dense0);  // replicate_dense (hbm_ps.hpp:244-247)
  std::map<ParamKey, std::vector<float>> host;       // the MEM-PS values (collect_updates)
  std::barrier bar(G);
  int failures = 0;
  for (std::uint64_t t = 0; t < NB; ++t) {
    const std::uint64_t b0 = t * B;
    std::vector<ParamKey> ws(keys.begin() + off[b0], keys.begin() + off[b0 + B]);
    tier.build_node(0, {ws}, [&](ParamKey k) {  // zero on first touch (oracle.hpp:80-83)
      auto it = host.find(k);
      return it == host.end() ? std::vector<float>(E, 0.0f) : it->second;
    });
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)
      th.emplace_back([&, g] {
        const Endpoint me = topo.endpoint_of(g);
        for (int j = 0; j < J; ++j) {
          // shard_batch (sharding.hpp:29-42): example i -> device (i % GJ) / J
          std::vector<std::int64_t> so{0};
          std::vector<std::uint64_t> sk;
          std::vector<std::uint8_t> sl;
          for (std::uint64_t i = std::uint64_t(g) * J + j; i < B; i += std::uint64_t(G) * J) {
            sk.insert(sk.end(), keys.begin() + off[b0 + i], keys.begin() + off[b0 + i + 1]);
            so.push_back(std::int64_t(sk.size()));
            sl.push_back(lab[b0 + i]);
          }
          const std::uint64_t n = sl.size();
          std::vector<float> dgrad(nw, 0.0f);
          if (n) {
            std::vector<ParamKey> uk(sk);
            std::sort(uk.begin(), uk.end());
            uk.erase(std::unique(uk.begin(), uk.end()), uk.end());
            auto view = tier.get(uk, me);  // pull (hbm_ps.hpp:112-143)
            std::vector<float> rows;
            for (ParamKey k : uk) rows.insert(rows.end(), view[k].begin(), view[k].end());
            std::vector<double> preds(n);
            std::vector<float> sg(uk.size() * E);
            if (or_forward_backward(E, L, dims, dense[g].data(), n, so.data(), sk.data(), sl.data(),
                                    uk.data(), rows.data(), uk.size(), preds.data(), dgrad.data(),
                                    sg.data()))
              ++failures;
            std::map<ParamKey, std::vector<float>> deltas;  // sgd_delta (model.hpp:226-230)
            for (std::size_t u = 0; u < uk.size(); ++u) {
              std::vector<float> d(E);
              for (int e = 0; e < E; ++e) d[e] = -(cfg.learning_rate * sg[u * E + e]);
              deltas.emplace(uk[u], std::move(d));
            }
            tier.push_deltas(deltas, me);
          }
          bar.arrive_and_wait();
          tier.drain_accums(me);
          bar.arrive_and_wait();
          sync.run(g, dgrad);  // canonical f64 sum over the devices (NVLink)
          if (or_average_apply(dense[g].data(), dgrad.data(), nw, G, cfg.learning_rate))
            ++failures;
        }
      });
    for (auto& x : th) x.join();
    for (auto& [k, v] : tier.dump_node(0)) host[k] = v;  // collect (mem_ps.hpp:210-245)
  }
  CHECK(failures == 0);
  std::vector<float> wd(nw);
  std::uint64_t n_sparse = 0;
  std::vector<std::uint64_t> wk(NB * B * nnz);
  std::vector<float> wr(NB * B * nnz * E);
  CHECK(or_train_reference(&cfg, B, NB * B, off.data(), keys.data(), lab.data(), wd.data(),
                           &n_sparse, wk.data(), wr.data(), wk.size()) == 0);
  for (int g = 0; g < G; ++g) CHECK(std::memcmp(dense[g].data(), wd.data(), nw * 4) == 0);
  std::uint64_t bad = 0;
  for (std::uint64_t i = 0; i < n_sparse; ++i) {
    auto it = host.find(wk[i]);
    if (it == host.end() || std::memcmp(it->second.data(), &wr[i * E], E * 4) != 0) ++bad;
  }
  if (bad) std::printf("  %llu of %llu rows differ\n", (unsigned long long)bad,
                       (unsigned long long)n_sparse);
  CHECK(bad == 0);
}

int main(int argc, char** argv) {
  const int G = argc > 1 ? std::atoi(argv[1]) : 1;
  try {
    unit_cases(G);
    range_split_case(G);
    device_worker_loop(G);
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught: %s\n", e.what());
    ++g_fail;
  }
  std::printf("%d passed, %d failed (G=%d)\n", g_pass, g_fail, G);
  return g_fail ? 1 : 0;
}

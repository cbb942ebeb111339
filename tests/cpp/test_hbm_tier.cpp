// GPU parity through the C++ host-side mirror (include/hps_gpu/hbm_tier.hpp).
// Ports of the reference's single-device cases (proj/tests/test_device_table.cpp,
// test_hbm_ps.cpp) plus a fused-batch run checked bit-for-bit against the
// oracle restatement (oracle/liboracle.so — test infrastructure).
// Built by __graft_entry__.build(); run by tests/test_cpp_api.py on a GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../oracle/hps_oracle.h"
#include "hps_gpu/hbm_tier.hpp"

using hps_gpu::Error;
using hps_gpu::HbmTier;
using hps_gpu::ParamKey;
using hps_gpu::Topology;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (cond) {                                                       \
      ++g_pass;                                                       \
    } else {                                                          \
      ++g_fail;                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                 \
  } while (0)
#define CHECK_THROWS(stmt, needle)                                    \
  do {                                                                \
    bool thrown = false;                                              \
    try {                                                             \
      stmt;                                                           \
    } catch (const Error& e) {                                        \
      thrown = std::strstr(e.what(), needle) != nullptr;              \
      if (!thrown) std::printf("  message: %s\n", e.what());          \
    }                                                                 \
    CHECK(thrown);                                                    \
  } while (0)

static HbmTier::HostValue keyed_value(std::size_t w) {
  return [w](ParamKey k) { return std::vector<float>(w, float(k)); };
}
static HbmTier::HostValue zeros_of(std::size_t w) {
  return [w](ParamKey) { return std::vector<float>(w, 0.0f); };
}

static void device_table_cases() {
  {  // round trip (test_device_table.cpp:24-31)
    HbmTier h(Topology(1, 1), 2);
    h.build_all({{7}}, [](ParamKey) { return std::vector<float>{1.0f, 1.0f}; });
    CHECK(h.table_at(0).get(7) == (std::vector<float>{1.0f, 1.0f}));
    CHECK(h.table_at(0).contains(7));
    CHECK(!h.table_at(0).contains(8));
  }
  {  // capacity rule (33-47)
    HbmTier h(Topology(1, 1), 1);
    h.build_all({{0, 1, 2, 3, 4, 5}}, keyed_value(1));
    CHECK(h.table_at(0).capacity() == 8);
    CHECK(h.table_at(0).occupancy() == 6);
  }
  {  // empty table (49-54)
    HbmTier h(Topology(1, 1), 2);
    h.build_all({{}}, zeros_of(2));
    CHECK(h.table_at(0).occupancy() == 0);
    CHECK(!h.table_at(0).contains(1));
    CHECK_THROWS(h.table_at(0).get(1), "missing key 1");
  }
  {  // accumulate is elementwise add (64-74)
    HbmTier h(Topology(1, 1), 2);
    h.build_all({{11}}, [](ParamKey) { return std::vector<float>{1.0f, 1.0f}; });
    h.accumulate({{11, {0.5f, -0.5f}}});
    CHECK(h.table_at(0).get(11) == (std::vector<float>{1.5f, 0.5f}));
    CHECK_THROWS(h.accumulate({{5, {1.0f, 1.0f}}}), "accumulate to missing key 5");
  }
  {  // 64 accumulates of +1 land exactly (85-97)
    HbmTier h(Topology(1, 1), 1);
    h.build_all({{42}}, zeros_of(1));
    for (int i = 0; i < 64; ++i) h.push_deltas({{42, {1.0f}}});
    h.drain_accums();
    CHECK(h.table_at(0).get(42) == std::vector<float>{64.0f});
  }
  {  // for_each walks every live entry once (120-139)
    HbmTier h(Topology(1, 1), 1);
    std::vector<ParamKey> ks;
    for (ParamKey k = 0; k < 100; ++k) ks.push_back(k * 17);
    h.build_all({ks}, [](ParamKey k) { return std::vector<float>{float(k / 17)}; });
    std::size_t seen = 0;
    double sum = 0;
    h.table_at(0).for_each([&](ParamKey, const float* v) {
      ++seen;
      sum += v[0];
    });
    CHECK(seen == 100);
    CHECK(sum == 4950.0);
  }
}

static void hbm_cases() {
  {  // carry-over (test_hbm_ps.cpp:104-116, one device)
    HbmTier h(Topology(1, 1), 1);
    h.build_all({{2, 3}}, keyed_value(1));
    h.accumulate({{2, {10.0f}}});
    h.build_all({{2, 5}}, keyed_value(1));
    CHECK(h.table_at(0).get(2) == std::vector<float>{12.0f});
    CHECK(h.table_at(0).get(5) == std::vector<float>{5.0f});
    CHECK(!h.table_at(0).contains(3));
  }
  {  // get: order-normalized, non-mutating, missing key (118-138)
    HbmTier h(Topology(1, 1), 1);
    h.build_all({{0, 1, 2, 3}}, keyed_value(1));
    auto view = h.get({3, 0, 1});
    CHECK(view.size() == 3);
    CHECK(view.begin()->first == 0);
    CHECK(view.at(3) == std::vector<float>{3.0f});
    CHECK(h.get({3, 0, 1}) == view);
    CHECK_THROWS(h.get({9}), "missing key 9");
  }
  {  // push then drain (157-177)
    HbmTier h(Topology(1, 1), 1);
    h.build_all({{0, 1}}, zeros_of(1));
    for (int n = 0; n < 800; ++n) h.push_deltas({{ParamKey(n % 2), {1.0f}}});
    h.drain_accums();
    CHECK(h.table_at(0).get(0) == std::vector<float>{400.0f});
    CHECK(h.table_at(0).get(1) == std::vector<float>{400.0f});
  }
  {  // not built
    HbmTier h(Topology(1, 1), 1);
    CHECK_THROWS(h.table_at(0), "tables not built");
  }
  {  // single replica sync untouched (194-202)
    HbmTier h(Topology(1, 1), 1);
    std::vector<float> b{3.25f, -1.5f};
    h.synchronize(b, true);
    CHECK(b == (std::vector<float>{3.25f, -1.5f}));
  }
  {  // dump_node: every (key,row), ascending
    HbmTier h(Topology(1, 1), 2);
    h.build_all({{9, 4, 7, 4}}, keyed_value(2));
    const auto d = h.dump_node(0);
    CHECK(d.size() == 3);
    CHECK(d.begin()->first == 4 && d.at(9) == (std::vector<float>{9.0f, 9.0f}));
  }
}

// The fused batch path vs the oracle's train_reference, bit-exact.
static void fused_batch_case() {
  const std::uint64_t dims = 20000, B = 512, nnz = 20, nb = 3;
  std::vector<std::int64_t> off(B * nb + 1);
  std::vector<ParamKey> keys(B * nb * nnz);
  std::vector<std::uint8_t> lab(B * nb);
  hps_gpu::check(hps_gen_dataset(dims, B * nb, nnz, 1, 1.0, 5, 6.0, 0, off.data(), keys.data(),
                                 lab.data()));
  HbmTier::Options o;
  o.key_space = dims;
  o.max_batch_examples = B;
  o.max_batch_keys = B * nnz;
  HbmTier h(Topology(1, 1), 8, o);
  std::vector<float> store(dims * 8, 0.0f);
  h.attach_store(store.data(), dims, false);
  for (std::uint64_t b = 0; b < nb; ++b) {
    std::vector<std::int64_t> bo(B + 1);
    for (std::uint64_t i = 0; i <= B; ++i) bo[i] = off[b * B + i] - off[b * B];
    h.train_batch(B, bo.data(), keys.data() + off[b * B], lab.data() + b * B);
  }
  h.flush();  // deferred write-backs -> store
  const auto dense = h.dense();
  or_cfg c{};
  c.nodes = 1;
  c.devices = 1;
  c.embedding_dim = 8;
  c.num_layers = 3;
  c.layer_dims[0] = 8;
  c.layer_dims[1] = 16;
  c.layer_dims[2] = 1;
  c.learning_rate = 0.05f;
  c.seed = 42;
  c.minibatches = 4;
  c.deterministic = 1;
  c.inject_skip_sync = -1;
  std::vector<float> wd(dense.size());
  std::vector<std::uint64_t> wk(dims);
  std::vector<float> wr(dims * 8);
  std::uint64_t n = 0;
  CHECK(or_train_reference(&c, B, B * nb, off.data(), keys.data(), lab.data(), wd.data(), &n,
                           wk.data(), wr.data(), dims) == 0);
  CHECK(wd == dense);
  bool rows_equal = true;
  for (std::uint64_t i = 0; i < n; ++i)
    rows_equal &= std::memcmp(&store[wk[i] * 8], &wr[i * 8], 32) == 0;
  CHECK(rows_equal);
}

int main() {
  try {
    device_table_cases();
    hbm_cases();
    fused_batch_case();
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught: %s\n", e.what());
    ++g_fail;
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}

// hps_gpu/hbm_tier.hpp — C++ host side of the B200 HBM-PS tier, mirroring
// the reference parameter-server API (namespace hps, header-only C++20:
// /root/reference/proj/include/hps/hbm_ps.hpp:41-408,
// device_table.hpp:32-137, topology.hpp:28-65) on top of the C ABI in
// hps_gpu.h. Same names, argument meanings and error behaviour, for ONE rank
// (one GPU) of a PartitionPolicy::modulo tier:
//
//   reference                              here
//   HbmTier(topo, policy, width, tr)       HbmTier(topo, width, Options{rank, device, nccl_id})
//   build_node / build_all                 same (HostValue callback)
//   get(keys, requester)                   get(keys)          COLLECTIVE over ranks
//   push_deltas(deltas, src)               push_deltas(deltas) COLLECTIVE
//   drain_accums(me)                       drain_accums()
//   accumulate(deltas, src)                accumulate(deltas)  COLLECTIVE
//   table_at(g)->{capacity,...,get,...}    table_at(rank())    (a DeviceTableView)
//   dump_node(node)                        dump_node(node)     (this rank's slice)
//   SyncSession::run(g, buf)               synchronize(buf, deterministic) COLLECTIVE
//
// Errors throw hps_gpu::Error (a std::runtime_error, like hps::Error) carrying
// the library's message, which repeats the reference's texts ("device
// table: missing key K", "hbm: tables not built", ...).
//
// Differences a caller of the reference must know:
//   * one object per GPU/process (or per thread driving one GPU); the
//     reference's lockstep device-worker threads map 1:1 onto ranks;
//   * HostValue is called only for owned keys the previous table does not
//     hold (the device carries those over, hbm_ps.hpp:89-98);
//   * the in-process, all-devices form with the reference's own signatures
//     (HbmTier(topo, policy, width, Transport*), get(keys, Endpoint), ...) is
//     hps_gpu/hbm_ps.hpp (namespace hps);
//   * PartitionPolicy is always modulo (range_split exists in the reference
//     only for its Appendix-A unit test).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hps_gpu.h"

namespace hps_gpu {

using ParamKey = std::uint64_t;

class Error : public std::runtime_error {
 public:
  Error(hps_status s, const std::string& m) : std::runtime_error(m), status_(s) {}
  hps_status status() const { return status_; }

 private:
  hps_status status_;
};

inline void check(hps_status s) {
  if (s != HPS_OK) throw Error(s, hps_last_error());
}

// topology.hpp:28-55
struct Topology {
  int num_nodes = 1;
  int devices_per_node = 1;
  Topology() = default;
  Topology(int nodes, int devices) : num_nodes(nodes), devices_per_node(devices) {
    auto pow2 = [](int x) { return x >= 1 && (x & (x - 1)) == 0; };
    if (!pow2(nodes)) throw Error(HPS_ERR_ARG, "topology: num_nodes must be a power of two");
    if (!pow2(devices))
      throw Error(HPS_ERR_ARG, "topology: devices_per_node must be a power of two");
  }
  int total_devices() const { return num_nodes * devices_per_node; }
  int node_of(int g) const { return g % num_nodes; }
  int device_of(int g) const { return g / num_nodes; }
  int global_index(int node, int device) const { return device * num_nodes + node; }
  int owner_of(ParamKey k) const { return int(k % std::uint64_t(total_devices())); }
};

// The DeviceTable query API (device_table.hpp:47-101) over this rank's table.
class DeviceTableView {
 public:
  explicit DeviceTableView(hps_tier_t h) : h_(h) {}
  std::size_t capacity() const { return info().cap; }
  std::size_t occupancy() const { return info().occ; }
  std::size_t value_width() const { return info().width; }
  bool contains(ParamKey key) const {  // one device probe (hps_table_lookup)
    std::uint8_t f = 0;
    check(hps_table_lookup(h_, &key, 1, &f, nullptr));
    return f != 0;
  }
  std::vector<float> get(ParamKey key) const {
    std::uint64_t rw = 0;
    check(hps_row_width(h_, &rw));
    std::uint8_t f = 0;
    std::vector<float> row(rw);
    check(hps_table_lookup(h_, &key, 1, &f, row.data()));
    if (!f) throw Error(HPS_ERR_MISSING_KEY, "device table: missing key " + std::to_string(key));
    row.resize(info().width);  // the embedding (an optimizer state stays on the device)
    return row;
  }
  template <class Fn>  // Fn(ParamKey, const float*), slot order
  void for_each(Fn&& fn) const {
    const Info in = info();
    std::vector<ParamKey> slots(in.cap);
    std::vector<float> rows(in.cap * in.width);
    check(hps_table_slots(h_, slots.data(), rows.data()));
    for (std::size_t i = 0; i < in.cap; ++i)
      if (slots[i] != ~ParamKey{0}) fn(slots[i], rows.data() + i * in.width);
  }

 private:
  struct Info {
    std::size_t cap, occ, width;
  };
  Info info() const {
    std::uint64_t c = 0, o = 0, w = 0;
    check(hps_table_info(h_, &c, &o, &w));
    return Info{c, o, w};
  }
  hps_tier_t h_;
};

struct TierOptions {
  int rank = 0;                       // global device index g of this handle
  int cuda_device = 0;
  const std::uint8_t* nccl_id = nullptr;  // hps_get_unique_id() of rank 0, if N*D > 1
  std::vector<std::uint64_t> layer_dims{8, 16, 1};  // ModelConfig (model.hpp:35-40)
  float learning_rate = 0.05f;
  std::uint64_t seed = 42;
  int minibatches = 4;
  bool deterministic = true;
  std::int64_t inject_skip_sync = -1;
  std::uint64_t key_space = 0;
  std::uint64_t max_batch_examples = 1 << 16;
  std::uint64_t max_batch_keys = 1 << 20;
  std::uint64_t max_working_set = 0;
};

class HbmTier {
 public:
  using HostValue = std::function<std::vector<float>(ParamKey)>;

  using Options = TierOptions;

  HbmTier(const Topology& topo, std::size_t width, const Options& opt = Options{})
      : topo_(topo), width_(width), rank_(opt.rank) {
    hps_config c{};
    c.nodes = topo.num_nodes;
    c.devices_per_node = topo.devices_per_node;
    c.rank = opt.rank;
    c.cuda_device = opt.cuda_device;
    c.embedding_dim = int(width);
    if (opt.layer_dims.empty() || opt.layer_dims.size() > HPS_MAX_LAYERS)
      throw Error(HPS_ERR_ARG, "config: layer_dims must end in 1");
    c.num_layers = int(opt.layer_dims.size());
    for (std::size_t i = 0; i < opt.layer_dims.size(); ++i) c.layer_dims[i] = opt.layer_dims[i];
    c.learning_rate = opt.learning_rate;
    c.seed = opt.seed;
    c.minibatches = opt.minibatches;
    c.deterministic = opt.deterministic ? 1 : 0;
    c.inject_skip_sync = opt.inject_skip_sync;
    c.key_space = opt.key_space;
    c.max_batch_examples = opt.max_batch_examples;
    c.max_batch_keys = opt.max_batch_keys;
    c.max_working_set = opt.max_working_set;
    check(hps_create(&c, opt.nccl_id, &h_));
  }
  ~HbmTier() { hps_destroy(h_); }
  HbmTier(const HbmTier&) = delete;
  HbmTier& operator=(const HbmTier&) = delete;

  const Topology& topology() const { return topo_; }
  std::size_t value_width() const { return width_; }
  int rank() const { return rank_; }
  hps_tier_t handle() const { return h_; }

  // hbm_ps.hpp:65-102 (this rank's share of the node's build).
  void build_node(int node, const std::vector<std::vector<ParamKey>>& keys_per_node,
                  const HostValue& host_value) {
    if (topo_.node_of(rank_) != node) return;
    std::vector<ParamKey> merged;
    for (const auto& ks : keys_per_node) merged.insert(merged.end(), ks.begin(), ks.end());
    std::sort(merged.begin(), merged.end());
    merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
    std::vector<ParamKey> owned;
    for (ParamKey k : merged)
      if (topo_.owner_of(k) == rank_) owned.push_back(k);
    std::uint64_t rw = 0;
    check(hps_row_width(h_, &rw));
    std::vector<std::uint8_t> carried(owned.size(), 0);
    if (built_ && !owned.empty())  // keys the previous table holds: the device carries them
      check(hps_table_lookup(h_, owned.data(), owned.size(), carried.data(), nullptr));
    std::vector<float> rows(owned.size() * rw, 0.0f);
    for (std::size_t i = 0; i < owned.size(); ++i) {
      if (carried[i]) continue;
      const auto v = host_value(owned[i]);
      if (v.size() != width_ && v.size() != rw)
        throw Error(HPS_ERR_WIDTH, "hbm: host value width mismatch");
      std::copy(v.begin(), v.end(), rows.begin() + i * rw);
    }
    check(hps_build(h_, owned.data(), owned.size(), rows.data()));
    built_ = true;
  }

  void build_all(const std::vector<std::vector<ParamKey>>& keys_per_node,
                 const HostValue& host_value) {
    for (int n = 0; n < topo_.num_nodes; ++n) build_node(n, keys_per_node, host_value);
  }

  // hbm_ps.hpp:112-143: order-normalized view. COLLECTIVE.
  std::map<ParamKey, std::vector<float>> get(const std::vector<ParamKey>& keys) {
    std::vector<ParamKey> k(keys);
    std::sort(k.begin(), k.end());
    k.erase(std::unique(k.begin(), k.end()), k.end());
    std::vector<float> rows(k.size() * width_);
    check(hps_pull(h_, k.data(), k.size(), rows.data()));
    std::map<ParamKey, std::vector<float>> out;
    for (std::size_t i = 0; i < k.size(); ++i)
      out.emplace(k[i], std::vector<float>(rows.begin() + i * width_,
                                           rows.begin() + (i + 1) * width_));
    return out;
  }

  // hbm_ps.hpp:148-167. COLLECTIVE.
  void push_deltas(const std::map<ParamKey, std::vector<float>>& deltas) {
    std::vector<ParamKey> k;
    std::vector<float> d;
    k.reserve(deltas.size());
    d.reserve(deltas.size() * width_);
    for (const auto& [key, v] : deltas) {
      if (v.size() != width_) throw Error(HPS_ERR_WIDTH, "hbm: delta width mismatch");
      k.push_back(key);
      d.insert(d.end(), v.begin(), v.end());
    }
    check(hps_push(h_, k.data(), d.data(), k.size()));
  }

  // hbm_ps.hpp:172-195
  void drain_accums() { check(hps_drain(h_)); }

  // hbm_ps.hpp:197-204. COLLECTIVE.
  void accumulate(const std::map<ParamKey, std::vector<float>>& deltas) {
    push_deltas(deltas);
    drain_accums();
  }

  // hbm_ps.hpp:206-215
  DeviceTableView table_at(int g) const {
    if (!built_) throw Error(HPS_ERR_NOT_BUILT, "hbm: tables not built");
    if (g != rank_) throw Error(HPS_ERR_ARG, "table_at: only this rank's table is local");
    return DeviceTableView(h_);
  }
  bool built() const { return built_; }

  // hbm_ps.hpp:224-232 for this rank's slice of the node.
  std::map<ParamKey, std::vector<float>> dump_node(int node) const {
    std::map<ParamKey, std::vector<float>> out;
    if (topo_.node_of(rank_) != node) return out;
    std::uint64_t cap = 0, occ = 0, w = 0;
    check(hps_table_info(h_, &cap, &occ, &w));
    std::vector<ParamKey> k(occ);
    std::vector<float> rows(occ * width_);
    std::uint64_t n = 0;
    check(hps_dump(h_, k.data(), rows.data(), &n));
    for (std::size_t i = 0; i < n; ++i)
      out.emplace(k[i], std::vector<float>(rows.begin() + i * width_,
                                           rows.begin() + (i + 1) * width_));
    return out;
  }

  // dump_node written as reference parameter files pf_<first_id + i>.bin
  // (ssd_ps.hpp:50-56) that SsdStore recovers unchanged. Returns the count.
  std::uint64_t export_files(const std::string& dir, std::uint32_t file_capacity = 4096,
                             std::uint64_t first_id = 0) {
    std::uint64_t files = 0;
    check(hps_export(h_, dir.c_str(), file_capacity, first_id, &files));
    return files;
  }

  // SyncSession::run (hbm_ps.hpp:303-310). COLLECTIVE.
  void synchronize(std::vector<float>& buf, bool deterministic) {
    check(hps_dense_sync(h_, buf.data(), buf.size(), deterministic ? 1 : 0));
  }

  // The fused per-batch hot path (performance API, hps_gpu.h).
  hps_batch_stats train_batch(std::uint64_t num_examples, const std::int64_t* offsets,
                              const ParamKey* keys, const std::uint8_t* labels,
                              bool on_device = false) {
    hps_batch_stats st{};
    check(hps_train_batch(h_, num_examples, offsets, keys, labels, on_device ? 1 : 0, &st));
    return st;
  }
  // pipelined train_batch: submit returns once the batch is staged and
  // enqueued; wait returns results in submission order
  void submit_batch(std::uint64_t num_examples, const std::int64_t* offsets,
                    const ParamKey* keys, const std::uint8_t* labels, bool on_device = false) {
    check(hps_submit_batch(h_, num_examples, offsets, keys, labels, on_device ? 1 : 0));
  }
  hps_batch_stats wait_batch() {
    hps_batch_stats st{};
    check(hps_wait_batch(h_, &st));
    return st;
  }
  void attach_store(float* rows, std::uint64_t num_keys, bool on_device) {
    check(hps_attach_store(h_, rows, num_keys, on_device ? 1 : 0));
  }
  // collect stage barrier: every resident row has reached the store
  void flush() { check(hps_flush(h_)); }
  // (rows read from, rows written to) the value store since creation
  std::pair<std::uint64_t, std::uint64_t> store_traffic() const {
    std::uint64_t r = 0, w = 0;
    check(hps_store_traffic(h_, &r, &w));
    return {r, w};
  }
  // where the attached store trains: HPS_STORE_HOST_MIRRORED (copied to
  // HBM, exact on the host at every observation) or per-batch staging
  int store_mode() const {
    int m = 0;
    check(hps_store_mode(h_, &m));
    return m;
  }
  // (H2D, D2H) bytes the store has moved over PCIe
  std::pair<std::uint64_t, std::uint64_t> store_pcie_bytes() const {
    std::uint64_t h = 0, d = 0;
    check(hps_store_pcie_bytes(h_, &h, &d));
    return {h, d};
  }
  std::vector<float> dense() const {
    std::uint64_t n = 0;
    check(hps_dense_count(h_, &n));
    std::vector<float> w(n);
    check(hps_get_dense(h_, w.data()));
    return w;
  }

 private:
  Topology topo_;
  std::size_t width_;
  int rank_;
  hps_tier_t h_ = nullptr;
  bool built_ = false;
};

}  // namespace hps_gpu

// hps_gpu/hbm_ps.hpp — drop-in for the reference's <hps/hbm_ps.hpp> (B200 build).
//
// The reference HBM-PS API with the reference's own names and signatures
// (namespace hps; /root/reference/proj/include/hps/hbm_ps.hpp:41-408,
// device_table.hpp:32-137, topology.hpp:25-72, common.hpp:25-40), over the C
// ABI of hps_gpu.h, so the device-worker loop (pipeline.hpp:502-566) and the
// reference's tests compile against it unchanged:
//
//   HbmTier(const Topology&, PartitionPolicy, std::size_t width, Transport*)
//   build_node / build_all (HostValue called only for keys the device
//                           table does not carry over, hbm_ps.hpp:89-98)
//   get(keys, Endpoint requester)        order-normalised map, any thread
//   push_deltas(deltas, Endpoint src)    queued per owner (kAccum)
//   drain_accums(Endpoint me)            senders applied in canonical order
//   accumulate(deltas, Endpoint src)     push + drain of the owners
//   table_at(g) / table_at(node, device) -> shared_ptr<DeviceTable>
//   built(), dump_node(node)
//   SyncSession(const Topology&, Transport*, bool det).run(g, buf)  COLLECTIVE
//   synchronize(bufs, topo, transport, det), canonical_sum, average_by
//
// What differs is what the reference simulates: its Transport is an
// in-process message-channel stand-in for NVLink; here `hps::Transport` is
// the box's real fabric — one hps_tier_t per global device (one B200 each,
// all in this process), created together so their NVLink windows map each
// other (same-process peer access) and the dense sync runs over them. The
// only caller change is constructing the Transport. Every
// table lives in its device's HBM: get reads the owners' tables on device
// (hps_table_lookup), drain applies on device (hps_apply_local, the sparse
// optimizer in place), build_node stages the host rows with cudaMemcpyAsync.
//
// Threading follows the reference: get / push_deltas / drain_accums /
// table_at may be called from any thread (one mutex per device handle);
// SyncSession::run is a collective, one call per device, as in the reference.
// Placement follows the PartitionPolicy on the host (modulo or range_split,
// topology.hpp:58-72): build_node hands each device exactly its keys
// (hps_build_placed), get/push/drain route by the same policy.
#pragma once

#include <algorithm>
#include <compare>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "hps_gpu.h"

namespace hps {

using ParamKey = std::uint64_t;

// common.hpp:28-40
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class TransportError : public Error {
 public:
  using Error::Error;
};

inline void check(bool ok, const char* msg) {
  if (!ok) throw Error(msg);
}
inline void check_status(hps_status s) {
  if (s != HPS_OK) throw Error(hps_last_error());
}

// transport.hpp:42-46
struct Endpoint {
  int node = 0;
  int device = 0;
  auto operator<=>(const Endpoint&) const = default;
};

// topology.hpp:25-55
struct Topology {
  int num_nodes = 1;
  int devices_per_node = 1;
  Topology() = default;
  Topology(int nodes, int devices) : num_nodes(nodes), devices_per_node(devices) {
    auto pow2 = [](int x) { return x >= 1 && (x & (x - 1)) == 0; };
    check(pow2(nodes), "topology: num_nodes must be a power of two");
    check(pow2(devices), "topology: devices_per_node must be a power of two");
  }
  int total_devices() const { return num_nodes * devices_per_node; }
  int node_of(int g) const { return g % num_nodes; }
  int device_of(int g) const { return g / num_nodes; }
  int global_index(int node, int device) const { return device * num_nodes + node; }
  Endpoint endpoint_of(int g) const { return Endpoint{node_of(g), device_of(g)}; }
  Endpoint mem_endpoint(int node) const { return Endpoint{node, -1}; }
};

// topology.hpp:58-72
struct PartitionPolicy {
  std::function<int(ParamKey)> device_of_key;
  bool is_modulo = false;  // (B200 build) key % (N*D), the collective C-ABI path's placement

  static PartitionPolicy modulo(const Topology& topo) {
    const int total = topo.total_devices();
    return PartitionPolicy{[total](ParamKey key) { return int(key % std::uint64_t(total)); },
                           true};
  }
  static PartitionPolicy range_split(ParamKey threshold) {
    return PartitionPolicy{[threshold](ParamKey key) { return key <= threshold ? 0 : 1; }, false};
  }
  int operator()(ParamKey key) const { return device_of_key(key); }
};

// Construction knobs of the device handles (the model and buffer maxima of
// hps_config).
struct TransportOptions {
  std::vector<int> cuda_devices;  // CUDA ordinal of global device g (default: g)
  std::vector<std::uint64_t> layer_dims{8, 16, 1};  // ModelConfig (model.hpp:35-40)
  float learning_rate = 0.05f;
  std::uint64_t seed = 42;
  int minibatches = 4;
  bool deterministic = true;
  std::uint64_t key_space = 0;
  std::uint64_t max_batch_examples = 1 << 16;
  std::uint64_t max_batch_keys = 1 << 20;
  std::uint64_t max_working_set = 0;
  int optimizer = HPS_OPT_SGD;
  float adagrad_eps = 1e-8f;
};

// The box's NVLink fabric: one device-tier handle per global device, all in
// this process (the reference's Transport simulates these links).
class Transport {
 public:
  using Options = TransportOptions;

  Transport(const Topology& topo, std::size_t width, const Options& opt = Options{})
      : topo_(topo), handles_(topo.total_devices(), nullptr), mu_(topo.total_devices()) {
    const int G = topo.total_devices();
    std::uint8_t id[HPS_NCCL_ID_BYTES] = {};
    if (G > 1) check_status(hps_get_unique_id(id));
    std::vector<hps_status> st(G, HPS_OK);
    std::vector<std::string> msg(G);
    auto create = [&](int g) {
      hps_config c{};
      c.nodes = topo.num_nodes;
      c.devices_per_node = topo.devices_per_node;
      c.rank = g;
      c.cuda_device = g < int(opt.cuda_devices.size()) ? opt.cuda_devices[g] : g;
      c.embedding_dim = int(width);
      c.num_layers = int(opt.layer_dims.size());
      for (std::size_t i = 0; i < opt.layer_dims.size() && i < HPS_MAX_LAYERS; ++i)
        c.layer_dims[i] = opt.layer_dims[i];
      c.learning_rate = opt.learning_rate;
      c.seed = opt.seed;
      c.minibatches = opt.minibatches;
      c.deterministic = opt.deterministic ? 1 : 0;
      c.inject_skip_sync = -1;
      c.key_space = opt.key_space;
      c.max_batch_examples = opt.max_batch_examples;
      c.max_batch_keys = opt.max_batch_keys;
      c.max_working_set = opt.max_working_set;
      c.optimizer = opt.optimizer;
      c.adagrad_eps = opt.adagrad_eps;
      st[g] = hps_create(&c, G > 1 ? id : nullptr, &handles_[g]);
      if (st[g] != HPS_OK) msg[g] = hps_last_error();  // (the message is thread-local)
    };
    if (G == 1) {
      create(0);
    } else {  // the NCCL communicator of the handles is created collectively
      std::vector<std::thread> th;
      for (int g = 0; g < G; ++g) th.emplace_back(create, g);
      for (auto& t : th) t.join();
    }
    for (int g = 0; g < G; ++g)
      if (st[g] != HPS_OK) {
        close();
        throw Error(msg[g]);
      }
    width_ = width;
    std::uint64_t rw = 0;
    check_status(hps_row_width(handles_[0], &rw));
    row_width_ = std::size_t(rw);
  }
  ~Transport() { close(); }
  Transport(const Transport&) = delete;
  Transport& operator=(const Transport&) = delete;

  const Topology& topology() const { return topo_; }
  hps_tier_t handle(int g) const { return handles_.at(g); }
  std::mutex& lock(int g) const { return mu_.at(g); }
  std::size_t width() const { return width_; }
  std::size_t row_width() const { return row_width_; }

 private:
  void close() {
    for (auto& h : handles_)
      if (h) {
        hps_destroy(h);
        h = nullptr;
      }
  }
  Topology topo_;
  std::vector<hps_tier_t> handles_;
  mutable std::vector<std::mutex> mu_;
  std::size_t width_ = 0, row_width_ = 0;
};

// device_table.hpp:32-137: the query API over one device's HBM table.
class DeviceTable {
 public:
  DeviceTable(const Transport* tr, int g) : tr_(tr), g_(g) {}
  std::size_t capacity() const { return info().cap; }
  std::size_t occupancy() const { return info().occ; }
  std::size_t value_width() const { return info().width; }
  bool contains(ParamKey key) const {
    std::uint8_t f = 0;
    std::lock_guard lk(tr_->lock(g_));
    check_status(hps_table_lookup(tr_->handle(g_), &key, 1, &f, nullptr));
    return f != 0;
  }
  std::vector<float> get(ParamKey key) const {
    std::uint8_t f = 0;
    std::vector<float> row(tr_->row_width());
    {
      std::lock_guard lk(tr_->lock(g_));
      check_status(hps_table_lookup(tr_->handle(g_), &key, 1, &f, row.data()));
    }
    if (!f) throw Error("device table: missing key " + std::to_string(key));
    row.resize(value_width());  // the embedding (the optimizer state stays on device)
    return row;
  }
  template <class Fn>  // Fn(ParamKey, const float*), slot order (device_table.hpp:97-101)
  void for_each(Fn&& fn) const {
    const Info in = info();
    const std::size_t rw = tr_->row_width();
    std::vector<ParamKey> slots(in.cap);
    std::vector<float> rows(in.cap * rw);
    {
      std::lock_guard lk(tr_->lock(g_));
      check_status(hps_table_slots(tr_->handle(g_), slots.data(), rows.data()));
    }
    for (std::size_t i = 0; i < in.cap; ++i)
      if (slots[i] != ~ParamKey{0}) fn(slots[i], rows.data() + i * rw);
  }

 private:
  struct Info {
    std::size_t cap, occ, width;
  };
  Info info() const {
    std::uint64_t c = 0, o = 0, w = 0;
    std::lock_guard lk(tr_->lock(g_));
    check_status(hps_table_info(tr_->handle(g_), &c, &o, &w));
    return Info{c, o, w};
  }
  const Transport* tr_;
  int g_;
};

// hbm_ps.hpp:41-242
class HbmTier {
 public:
  using HostValue = std::function<std::vector<float>(ParamKey)>;

  HbmTier(const Topology& topo, PartitionPolicy policy, std::size_t width, Transport* transport)
      : topo_(topo), policy_(std::move(policy)), width_(width), tr_(transport),
        pending_(topo.total_devices()), built_(topo.total_devices(), false) {
    check(tr_ != nullptr, "hbm: the B200 tier needs its Transport (the device handles)");
    check(tr_->topology().total_devices() == topo.total_devices(),
          "hbm: transport topology mismatch");
    check(tr_->width() == width, "hbm: width mismatch");
    for (auto& p : pending_) p.resize(topo.total_devices());
  }

  const Topology& topology() const { return topo_; }
  std::size_t value_width() const { return width_; }

  // hbm_ps.hpp:65-102: per device of the node, its owned keys of the merged
  // working set; HostValue only for keys the previous table does not hold
  // (the device carries those over itself).
  void build_node(int node, const std::vector<std::vector<ParamKey>>& keys_per_node,
                  const HostValue& host_value) {
    std::vector<ParamKey> merged;
    for (const auto& ks : keys_per_node) merged.insert(merged.end(), ks.begin(), ks.end());
    std::sort(merged.begin(), merged.end());
    merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
    const std::size_t rw = tr_->row_width();
    for (int d = 0; d < topo_.devices_per_node; ++d) {
      const int g = topo_.global_index(node, d);
      std::vector<ParamKey> owned;
      for (ParamKey k : merged)
        if (owner_of(k) == g) owned.push_back(k);
      std::vector<std::uint8_t> carried(owned.size(), 0);
      std::lock_guard lk(tr_->lock(g));
      if (built_[g] && !owned.empty())
        check_status(hps_table_lookup(tr_->handle(g), owned.data(), owned.size(), carried.data(),
                                      nullptr));
      std::vector<float> rows(owned.size() * rw, 0.0f);
      for (std::size_t i = 0; i < owned.size(); ++i) {
        if (carried[i]) continue;  // the device copies the previous table's row
        const std::vector<float> v = host_value(owned[i]);
        if (v.size() != width_ && v.size() != rw) throw Error("hbm: host value width mismatch");
        std::copy(v.begin(), v.end(), rows.begin() + i * rw);
      }
      check_status(
          hps_build_placed(tr_->handle(g), owned.data(), owned.size(), rows.data()));
      built_[g] = true;
    }
  }

  void build_all(const std::vector<std::vector<ParamKey>>& keys_per_node,
                 const HostValue& host_value) {
    for (int n = 0; n < topo_.num_nodes; ++n) build_node(n, keys_per_node, host_value);
  }

  // hbm_ps.hpp:112-143: the requester's view, order-normalised by key; every
  // owner's rows read from its HBM table.
  std::map<ParamKey, std::vector<float>> get(const std::vector<ParamKey>& keys,
                                             Endpoint requester) {
    (void)requester;
    std::map<int, std::vector<ParamKey>> by_owner;
    for (ParamKey k : keys) by_owner[owner_of(k)].push_back(k);
    std::map<ParamKey, std::vector<float>> out;
    const std::size_t rw = tr_->row_width();
    for (auto& [g, ks] : by_owner) {
      require_built(g);
      std::sort(ks.begin(), ks.end());
      ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
      std::vector<std::uint8_t> found(ks.size());
      std::vector<float> rows(ks.size() * rw);
      {
        std::lock_guard lk(tr_->lock(g));
        check_status(hps_table_lookup(tr_->handle(g), ks.data(), ks.size(), found.data(),
                                      rows.data()));
      }
      for (std::size_t i = 0; i < ks.size(); ++i) {
        if (!found[i]) throw Error("device table: missing key " + std::to_string(ks[i]));
        out.emplace(ks[i], std::vector<float>(rows.begin() + i * rw,
                                              rows.begin() + i * rw + width_));
      }
    }
    return out;
  }

  // hbm_ps.hpp:148-167: each owner queues the sender's deltas.
  void push_deltas(const std::map<ParamKey, std::vector<float>>& deltas, Endpoint src) {
    const int s = topo_.global_index(src.node, src.device);
    std::map<int, std::vector<std::pair<ParamKey, const std::vector<float>*>>> parts;
    for (const auto& [k, v] : deltas) {
      if (v.size() != width_) throw Error("hbm: delta width mismatch");
      parts[owner_of(k)].emplace_back(k, &v);
    }
    std::lock_guard lk(mu_);
    for (auto& [g, kv] : parts) {  // one message per (owner, push), keys unique within it
      Message m;
      for (auto& [k, v] : kv) {
        m.keys.push_back(k);
        m.vals.insert(m.vals.end(), v->begin(), v->end());
      }
      pending_[g][s].push_back(std::move(m));
    }
  }

  // hbm_ps.hpp:172-195: senders in canonical (node, device) order.
  void drain_accums(Endpoint me) {
    const int g = topo_.global_index(me.node, me.device);
    require_built(g);
    std::vector<std::vector<Message>> mine(topo_.total_devices());
    {
      std::lock_guard lk(mu_);
      mine.swap(pending_[g]);
      pending_[g].resize(topo_.total_devices());
    }
    for (int sn = 0; sn < topo_.num_nodes; ++sn)
      for (int sd = 0; sd < topo_.devices_per_node; ++sd)
        for (const Message& m : mine[topo_.global_index(sn, sd)]) {  // in push order
          if (m.keys.empty()) continue;
          std::lock_guard lk(tr_->lock(g));
          check_status(
              hps_apply_local(tr_->handle(g), m.keys.data(), m.vals.data(), m.keys.size()));
        }
  }

  // hbm_ps.hpp:197-204
  void accumulate(const std::map<ParamKey, std::vector<float>>& deltas, Endpoint src) {
    push_deltas(deltas, src);
    std::vector<int> owners;
    for (const auto& kv : deltas) owners.push_back(owner_of(kv.first));
    std::sort(owners.begin(), owners.end());
    owners.erase(std::unique(owners.begin(), owners.end()), owners.end());
    for (int g : owners) drain_accums(topo_.endpoint_of(g));
  }

  // hbm_ps.hpp:206-222
  std::shared_ptr<DeviceTable> table_at(int global_device) const {
    check(global_device >= 0 && global_device < topo_.total_devices(), "hbm: bad device");
    std::lock_guard lk(mu_);
    if (!built_[global_device]) throw Error("hbm: tables not built");
    return std::make_shared<DeviceTable>(tr_, global_device);
  }
  std::shared_ptr<DeviceTable> table_at(int node, int device) const {
    return table_at(topo_.global_index(node, device));
  }
  bool built() const {
    std::lock_guard lk(mu_);
    return std::all_of(built_.begin(), built_.end(), [](bool b) { return b; });
  }

  // hbm_ps.hpp:224-232: every (key, row) of the node's tables, by key.
  std::map<ParamKey, std::vector<float>> dump_node(int node) const {
    std::map<ParamKey, std::vector<float>> out;
    const std::size_t rw = tr_->row_width();
    for (int d = 0; d < topo_.devices_per_node; ++d) {
      const int g = topo_.global_index(node, d);
      std::lock_guard lk(tr_->lock(g));
      std::uint64_t cap = 0, occ = 0, w = 0, n = 0;
      check_status(hps_table_info(tr_->handle(g), &cap, &occ, &w));
      std::vector<ParamKey> k(occ);
      std::vector<float> rows(occ * rw);
      check_status(hps_dump(tr_->handle(g), k.data(), rows.data(), &n));
      for (std::size_t i = 0; i < n; ++i)
        out.emplace(k[i], std::vector<float>(rows.begin() + i * rw,
                                             rows.begin() + i * rw + width_));
    }
    return out;
  }

 private:
  int owner_of(ParamKey k) const {
    const int g = policy_(k);
    if (g < 0 || g >= topo_.total_devices())
      throw Error("hbm: partition policy placed key " + std::to_string(k) + " on device " +
                  std::to_string(g) + " of " + std::to_string(topo_.total_devices()));
    return g;
  }

  struct Message {  // one push_deltas call's share for one owner (kAccum)
    std::vector<ParamKey> keys;
    std::vector<float> vals;
  };
  void require_built(int g) const {
    std::lock_guard lk(mu_);
    if (!built_[g]) throw Error("hbm: tables not built");
  }
  Topology topo_;
  PartitionPolicy policy_;
  std::size_t width_;
  Transport* tr_;
  mutable std::mutex mu_;
  std::vector<std::vector<std::vector<Message>>> pending_;  // [owner][sender]
  std::vector<bool> built_;
};

// hbm_ps.hpp:249-256
inline std::vector<float> average_by(const std::vector<float>& sum, int count) {
  std::vector<float> out(sum.size());
  for (std::size_t i = 0; i < sum.size(); ++i) out[i] = sum[i] / float(count);
  return out;
}

// hbm_ps.hpp:258-277 (host helper, as in the reference)
inline std::vector<float> canonical_sum(std::vector<std::pair<int, const std::vector<float>*>> parts,
                                        const Topology& topo) {
  check(!parts.empty(), "canonical_sum: no parts");
  std::sort(parts.begin(), parts.end(), [&](const auto& a, const auto& b) {
    return std::make_pair(topo.node_of(a.first), topo.device_of(a.first)) <
           std::make_pair(topo.node_of(b.first), topo.device_of(b.first));
  });
  const std::size_t len = parts[0].second->size();
  std::vector<float> out(len);
  for (std::size_t i = 0; i < len; ++i) {
    double acc = 0.0;
    for (const auto& [g, buf] : parts) acc += double((*buf)[i]);
    out[i] = static_cast<float>(acc);
  }
  return out;
}

// hbm_ps.hpp:285-401: the dense sync, one call per device (COLLECTIVE): every
// device's buffer becomes the canonical f64 sum of all devices' buffers, over
// NVLink (hps_dense_sync: the replicas all-gathered into the peers' windows).
class SyncSession {
 public:
  SyncSession(const Topology& topo, Transport* transport, bool deterministic)
      : topo_(topo), tr_(transport), det_(deterministic) {
    check(tr_ != nullptr, "sync: the B200 tier needs its Transport (the device handles)");
  }
  int rounds() const { return 1; }  // one all-gather over NVSwitch
  void run(int g, std::vector<float>& buf) {
    std::lock_guard lk(tr_->lock(g));  // (other threads may use device g's handle)
    check_status(hps_dense_sync(tr_->handle(g), buf.data(), buf.size(), det_ ? 1 : 0));
  }

 private:
  Topology topo_;
  Transport* tr_;
  bool det_;
};

// hbm_ps.hpp:403-408: all devices' buffers synchronised (one thread each).
inline void synchronize(std::vector<std::vector<float>>& bufs, const Topology& topo,
                        Transport* transport, bool deterministic) {
  SyncSession s(topo, transport, deterministic);
  std::vector<std::thread> th;
  std::vector<std::string> err(bufs.size());
  for (int g = 0; g < topo.total_devices(); ++g)
    th.emplace_back([&, g] {
      try {
        s.run(g, bufs[g]);
      } catch (const std::exception& e) {
        err[g] = e.what();
      }
    });
  for (auto& t : th) t.join();
  for (const auto& e : err)
    if (!e.empty()) throw Error(e);
}

}  // namespace hps

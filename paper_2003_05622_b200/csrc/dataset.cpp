// Synthetic CTR input generator (host side of the data loader).
//
// Restates the reference generator gen_dataset (dataset.hpp:180-227) so the
// GPU tier, the tests and the bench all see the exact example stream the
// reference CPU path trains on: one std::mt19937_64 stream per dataset,
// features drawn until `nnz` distinct keys exist (then ascending), labels
// Bernoulli(sigmoid(planted logit)). Two deliberate differences, neither
// observable in the output:
//   * the Zipf inverse-CDF table is built only for Zipf draws (the reference
//     builds it even for uniform keys, dataset.hpp:190-191, which costs
//     8 GB at 1e9 keys);
//   * per-example feature sets are a small sorted array instead of std::set.
// Byte-equality with the reference is pinned by tests/test_oracle_golden.py
// against fixtures produced by oracle/_ref (the unmodified reference).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "hps_gpu.h"
#include "tier_internal.h"

namespace hpsgpu {
namespace {

inline std::uint64_t splitmix(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// common.hpp:65-71
inline std::uint64_t stream_value(std::uint64_t seed, std::uint64_t n) {
  return splitmix(seed + 0x632be59bd9b4e019ULL * (n + 1));
}
inline double unit_of(std::uint64_t x) {
  return double(x >> 11) * 0x1.0p-53;
}

// Planted per-key Gaussian weight via Box-Muller (dataset.hpp:138-146).
struct PlantedModel {
  std::uint64_t clusters;
  std::uint64_t salt_a, salt_b;
  double scale;
  std::uint64_t nnz;

  double weight(std::uint64_t key) const {
    const std::uint64_t unit = clusters ? key % clusters : key;
    const double u1 = std::max(unit_of(splitmix(unit ^ salt_a)), 1e-300);
    const double u2 = unit_of(splitmix(unit ^ salt_b));
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }

  // dataset.hpp:148-155
  double logit(const std::uint64_t* f, std::size_t n) const {
    if (clusters) return scale * weight(f[0]);
    double z = 0.0;
    for (std::size_t i = 0; i < n; ++i) z += weight(f[i]);
    return z * scale / std::sqrt(double(nnz));
  }
};

// Inverse-CDF Zipf(s) over [0, n) (dataset.hpp:158-178).
class ZipfTable {
 public:
  ZipfTable(std::uint64_t n, double s) : cdf_(n) {
    double acc = 0.0;
    for (std::uint64_t r = 0; r < n; ++r) {
      acc += 1.0 / std::pow(double(r + 1), s);
      cdf_[r] = acc;
    }
    for (double& c : cdf_) c /= acc;
  }
  std::uint64_t draw(double u) const {
    auto it = std::lower_bound(cdf_.begin(), cdf_.end(), u);
    if (it == cdf_.end()) --it;
    return std::uint64_t(it - cdf_.begin());
  }

 private:
  std::vector<double> cdf_;
};

// Insert into a small ascending array if absent (std::set semantics).
inline bool insert_sorted(std::uint64_t* a, std::size_t& n, std::uint64_t k) {
  std::uint64_t* pos = std::lower_bound(a, a + n, k);
  if (pos != a + n && *pos == k) return false;
  std::move_backward(pos, a + n, a + n + 1);
  *pos = k;
  ++n;
  return true;
}

}  // namespace

// init_dense (model.hpp:42-53): uniform in +-0.05 from mt19937_64(seed).
void init_dense_host(const hps_config* cfg, float* out, std::uint64_t n) {
  std::mt19937_64 rng(cfg->seed);
  for (std::uint64_t i = 0; i < n; ++i)
    out[i] = static_cast<float>((unit_of(rng()) * 2.0 - 1.0) * 0.05);
}

}  // namespace hpsgpu

extern "C" hps_status hps_gen_dataset(uint64_t dims, uint64_t num_examples,
                                      uint64_t nnz, int zipf, double zipf_s,
                                      uint64_t seed, double signal_scale,
                                      uint64_t clusters, int64_t* offsets,
                                      uint64_t* keys, uint8_t* labels) {
  using namespace hpsgpu;
  if (!(dims >= nnz && nnz > 0))
    return set_error(HPS_ERR_ARG, "gen: need nnz <= dims");
  if (clusters != 0 && dims / clusters < nnz)
    return set_error(HPS_ERR_ARG, "gen: cluster key pools must hold nnz keys");
  if (!offsets || !keys || !labels)
    return set_error(HPS_ERR_ARG, "gen: null output buffer");
  std::mt19937_64 rng(seed);
  std::vector<ZipfTable> zt;
  if (zipf) zt.emplace_back(clusters ? clusters : dims, zipf_s);
  const PlantedModel pm{clusters, stream_value(seed, 100),
                        stream_value(seed, 101), signal_scale, nnz};
  const std::uint64_t pool = clusters ? dims / clusters : 0;
  for (std::uint64_t e = 0; e < num_examples; ++e) {
    std::uint64_t* f = keys + e * nnz;
    std::size_t have = 0;
    if (clusters) {
      const double uc = unit_of(rng());
      const std::uint64_t c =
          zipf ? zt[0].draw(uc)
               : std::min<std::uint64_t>(std::uint64_t(uc * double(clusters)),
                                         clusters - 1);
      while (have < nnz) {
        const std::uint64_t slot = std::min<std::uint64_t>(
            std::uint64_t(unit_of(rng()) * double(pool)), pool - 1);
        insert_sorted(f, have, slot * clusters + c);
      }
    } else {
      while (have < nnz) {
        const double u = unit_of(rng());
        const std::uint64_t k =
            zipf ? zt[0].draw(u)
                 : std::min<std::uint64_t>(std::uint64_t(u * double(dims)),
                                           dims - 1);
        insert_sorted(f, have, k);
      }
    }
    offsets[e] = int64_t(e * nnz);
    const double p = 1.0 / (1.0 + std::exp(-pm.logit(f, nnz)));
    labels[e] = (unit_of(rng()) < p) ? 1 : 0;
  }
  offsets[num_examples] = int64_t(num_examples * nnz);
  return HPS_OK;
}

// BASELINE config 4's multi-slot ads input (no reference generator exists;
// SURVEY 8(d) c4): every example draws T ~ U{1..max_keys} (slot, id) pairs,
// slot ~ U{0..slots-1}, id ~ Zipf(zipf_s) over ids_per_slot (a hot head per
// slot), key = slot * ids_per_slot + id, kept sorted and unique per example
// (so an example holds up to max_keys keys over up to `slots` fields,
// multi-hot within a field). Labels follow the planted logistic of
// gen_dataset over the example's keys. One mt19937_64 stream: deterministic.
extern "C" hps_status hps_gen_multislot(uint64_t slots, uint64_t ids_per_slot,
                                        uint64_t num_examples, uint64_t max_keys,
                                        double zipf_s, uint64_t seed, double signal_scale,
                                        int64_t* offsets, uint64_t* keys, uint8_t* labels,
                                        uint64_t* n_keys_out) {
  using namespace hpsgpu;
  if (!slots || !ids_per_slot || !max_keys)
    return set_error(HPS_ERR_ARG, "gen: slots, ids_per_slot and max_keys must be positive");
  if (slots > ~std::uint64_t(0) / ids_per_slot)
    return set_error(HPS_ERR_ARG, "gen: key space overflows 64 bits");
  if (!offsets || !keys || !labels || !n_keys_out)
    return set_error(HPS_ERR_ARG, "gen: null output buffer");
  std::mt19937_64 rng(seed);
  const ZipfTable zt(ids_per_slot, zipf_s);
  const PlantedModel pm{0, stream_value(seed, 100), stream_value(seed, 101), signal_scale, 1};
  std::uint64_t at = 0;
  for (std::uint64_t e = 0; e < num_examples; ++e) {
    offsets[e] = int64_t(at);
    std::uint64_t* f = keys + at;
    std::size_t have = 0;
    const std::uint64_t T =
        1 + std::min<std::uint64_t>(std::uint64_t(unit_of(rng()) * double(max_keys)), max_keys - 1);
    for (std::uint64_t t = 0; t < T; ++t) {
      const std::uint64_t s =
          std::min<std::uint64_t>(std::uint64_t(unit_of(rng()) * double(slots)), slots - 1);
      const std::uint64_t id = zt.draw(unit_of(rng()));
      insert_sorted(f, have, s * ids_per_slot + id);
    }
    at += have;
    double z = 0.0;
    for (std::size_t i = 0; i < have; ++i) z += pm.weight(f[i]);
    const double p = 1.0 / (1.0 + std::exp(-z * signal_scale / std::sqrt(double(have))));
    labels[e] = (unit_of(rng()) < p) ? 1 : 0;
  }
  offsets[num_examples] = int64_t(at);
  *n_keys_out = at;
  return HPS_OK;
}

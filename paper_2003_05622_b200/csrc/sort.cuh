// Stable LSD radix sort and tile scans whose element counts live in device
// memory, so a whole batch can run without host round-trips.
//
// Used for the working-set dedup (mem_ps.hpp:101-108, hbm_ps.hpp:69-74),
// the mini-batch dedup + inverse index (pipeline.hpp:523-528) and the stable
// partition of unique keys by owner (hbm_ps.hpp:75-79, 116-121). Keys are
// u64 but only their significant bits (< key_space) are sorted.
//
// Tile = 256 threads x 16 items. A pass is histogram -> single-CTA
// exclusive scan of the digit-major [digit][tile] counts -> stable scatter,
// ranked inside each warp with __match_any_sync (warps own contiguous
// 512-item sub-tiles, so warp order is input order).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hpsgpu {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kWarpTile = kSortTile / kSortWarps;      // 512
constexpr int kDigits = 256;

// An element count that is either known on the host or produced on the
// device by an earlier kernel (read at kernel start, no host round-trip).
struct Count {
  const std::uint64_t* p;
  std::uint64_t v;
  __device__ __forceinline__ std::uint64_t get() const { return p ? *p : v; }
};

struct ShiftDigit {
  int shift;
  __device__ __forceinline__ std::uint32_t operator()(std::uint64_t k) const {
    return std::uint32_t(k >> shift) & 0xFFu;
  }
};

// Owner bucket of the modulo policy (topology.hpp:61-65); digits < G <= 256.
struct ModDigit {
  std::uint32_t G;
  __device__ __forceinline__ std::uint32_t operator()(std::uint64_t k) const {
    return std::uint32_t(k % G);
  }
};

template <class Digit>
__global__ void __launch_bounds__(kSortThreads)
    radix_hist_kernel(const std::uint64_t* __restrict__ keys,
                      Count cnt_n, Digit dig,
                      std::uint32_t* __restrict__ hist, std::uint32_t nblocks) {
  __shared__ std::uint32_t cnt[kDigits];
  const std::uint64_t n = cnt_n.get();
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kSortTile;
  const unsigned lane = threadIdx.x & 31;
#pragma unroll 4
  for (int it = 0; it < kSortItems; ++it) {
    const std::uint64_t idx = base + std::uint64_t(it) * kSortThreads + threadIdx.x;
    const bool valid = idx < n;
    const std::uint32_t d = valid ? dig(keys[idx]) : kDigits;
    // warp-aggregated increments: one smem atomic per distinct digit
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    if (valid && lane == unsigned(__ffs(peers) - 1))
      atomicAdd(&cnt[d], unsigned(__popc(peers)));
  }
  __syncthreads();
  hist[std::uint64_t(threadIdx.x) * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// Exclusive scan of data[0..m) in place by one CTA of 1024 threads; the
// grand total goes to *total if non-null.
__global__ void __launch_bounds__(1024)
    scan_single_cta_kernel(std::uint32_t* __restrict__ data, std::uint64_t m,
                           std::uint64_t* __restrict__ total) {
  __shared__ std::uint32_t warp_sums[32];
  const std::uint64_t per = (m + 1023) / 1024;
  const std::uint64_t beg = per * threadIdx.x;
  const std::uint64_t end = beg + per < m ? beg + per : m;
  std::uint32_t s = 0;
  for (std::uint64_t i = beg; i < end; ++i) s += data[i];
  // block exclusive scan of s
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= unsigned(o)) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    std::uint32_t w = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= unsigned(o)) w += y;
    }
    warp_sums[lane] = w;  // inclusive
  }
  __syncthreads();
  std::uint32_t run = x - s + (warp ? warp_sums[warp - 1] : 0u);
  for (std::uint64_t i = beg; i < end; ++i) {
    const std::uint32_t v = data[i];
    data[i] = run;
    run += v;
  }
  if (total && threadIdx.x == 1023) *total = run;
}

template <class Digit, bool kValues>
__global__ void __launch_bounds__(kSortThreads)
    radix_scatter_kernel(const std::uint64_t* __restrict__ kin,
                         const std::uint32_t* __restrict__ vin,
                         Count cnt_n, Digit dig,
                         const std::uint32_t* __restrict__ hist_scanned,
                         std::uint32_t nblocks, std::uint64_t* __restrict__ kout,
                         std::uint32_t* __restrict__ vout) {
  __shared__ std::uint32_t wcnt[kSortWarps][kDigits];
  __shared__ std::uint32_t gbase[kDigits];
  const std::uint64_t n = cnt_n.get();
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kSortTile;
  if (base >= n) return;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kDigits / 32; ++i) wcnt[warp][lane + 32 * i] = 0;
  gbase[threadIdx.x] = hist_scanned[std::uint64_t(threadIdx.x) * nblocks + blockIdx.x];
  __syncwarp();
  const unsigned lt = lanemask_lt();
  const std::uint64_t wbase = base + std::uint64_t(warp) * kWarpTile;
  std::uint64_t k[kSortItems];
  std::uint32_t v[kSortItems];
  std::uint32_t r[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const std::uint64_t idx = wbase + std::uint64_t(it) * 32 + lane;
    const bool valid = idx < n;
    k[it] = valid ? kin[idx] : 0;
    if (kValues) v[it] = valid ? vin[idx] : 0;
    const std::uint32_t d = valid ? dig(k[it]) : kDigits;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    const std::uint32_t prior = valid ? wcnt[warp][d] : 0u;
    r[it] = prior + unsigned(__popc(peers & lt));
    __syncwarp();
    if (valid && lane == unsigned(__ffs(peers) - 1))
      wcnt[warp][d] = prior + unsigned(__popc(peers));
    __syncwarp();
  }
  __syncthreads();
  {
    const unsigned d = threadIdx.x;
    std::uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const std::uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const std::uint64_t idx = wbase + std::uint64_t(it) * 32 + lane;
    if (idx < n) {
      const std::uint32_t d = dig(k[it]);
      const std::uint64_t pos = std::uint64_t(gbase[d]) + wcnt[warp][d] + r[it];
      kout[pos] = k[it];
      if (kValues) vout[pos] = v[it];
    }
  }
}

// ---- three-kernel tile scan with a device-side element count -----------
//
// F  : __device__ std::uint32_t operator()(std::uint64_t i) const — item value
// Em : __device__ void operator()(std::uint64_t i, std::uint32_t v,
//                                  std::uint64_t exclusive_prefix) const

template <class F>
__global__ void __launch_bounds__(kSortThreads)
    tile_reduce_kernel(F f, Count cnt_n,
                       std::uint32_t* __restrict__ bsum) {
  __shared__ std::uint32_t ws[kSortWarps];
  const std::uint64_t n = cnt_n.get();
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kSortTile;
  std::uint32_t s = 0;
  for (int it = 0; it < kSortItems; ++it) {
    const std::uint64_t idx = base + std::uint64_t(it) * kSortThreads + threadIdx.x;
    if (idx < n) s += f(idx);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    std::uint32_t t = 0;
    for (int w = 0; w < kSortWarps; ++w) t += ws[w];
    bsum[blockIdx.x] = t;
  }
}

template <class F, class Em>
__global__ void __launch_bounds__(kSortThreads)
    tile_emit_kernel(F f, Em em, Count cnt_n,
                     const std::uint32_t* __restrict__ bsum_scanned) {
  __shared__ std::uint32_t ws[kSortWarps];
  const std::uint64_t n = cnt_n.get();
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kSortTile;
  if (base >= n) return;
  // blocked arrangement: thread t owns items base + t*16 .. +15
  const std::uint64_t tb = base + std::uint64_t(threadIdx.x) * kSortItems;
  std::uint32_t vals[kSortItems];
  std::uint32_t s = 0;
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const std::uint64_t idx = tb + it;
    vals[it] = idx < n ? f(idx) : 0u;
    s += vals[it];
  }
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= unsigned(o)) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  std::uint32_t wpre = 0;
  for (unsigned w = 0; w < warp; ++w) wpre += ws[w];
  std::uint64_t run = std::uint64_t(bsum_scanned[blockIdx.x]) + wpre + (x - s);
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const std::uint64_t idx = tb + it;
    if (idx < n) em(idx, vals[it], run);
    run += vals[it];
  }
}

inline std::uint32_t tiles_for(std::uint64_t n) {
  return std::uint32_t((n + kSortTile - 1) / kSortTile);
}

}  // namespace hpsgpu

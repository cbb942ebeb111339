// Stable LSD radix sort and prefix scans whose element counts may live in
// device memory, so a whole batch runs without host round-trips.
//
// Used for the working-set dedup (mem_ps.hpp:101-108, hbm_ps.hpp:69-74), the
// mini-batch dedup + inverse index (pipeline.hpp:523-528) and the stable
// owner partition of unique keys (hbm_ps.hpp:75-79, 116-121). Keys are u64;
// only their significant bits (< key_space) are sorted.
//
// Onesweep structure (8-bit digits):
//   * one histogram kernel counts the digits of every pass up front;
//   * one kernel per pass: a CTA takes the next tile ticket, ranks its tile
//     stably (warps own contiguous sub-tiles; __match_any_sync ranks within
//     a warp), publishes its per-digit count, resolves its exclusive prefix
//     per digit by decoupled look-back over the preceding tiles, and
//     scatters. Tickets are handed out in launch order, so a tile only ever
//     waits on tiles that are already running.
// Status words are 64-bit [epoch:32 | flag:2 | count:30]. A launch's epoch is
// (device context counter << 12) | launch index within the context, and the
// tile ticket counter is reset at the start of every context (a batch body or
// one API call): nothing baked into a launch depends on earlier launches, so
// a captured CUDA graph replays correctly, and the status arrays never need
// clearing (the host clears them once per 2^20 contexts, before a wrap).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hpsgpu {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kWarpTile = kSortTile / kSortWarps;      // 256
constexpr int kDigits = 256;
constexpr int kMaxPasses = 8;

constexpr std::uint64_t kFlagAgg = 1ull << 30;
constexpr std::uint64_t kFlagInc = 2ull << 30;
constexpr std::uint64_t kCountMask = (1ull << 30) - 1;

// An element count known on the host or produced on the device by an
// earlier kernel (read at kernel start, no host round-trip).
struct Count {
  const std::uint64_t* p;
  std::uint64_t v;
  __device__ __forceinline__ std::uint64_t get() const { return p ? *p : v; }
};

// Look-back context of one launch: ticket counter, the host-tracked number of
// tickets handed out before this launch, the launch's epoch, status words.
struct LookBack {
  unsigned long long* ticket;   // reset at the start of every context
  std::uint64_t base;           // tickets handed out earlier in this context
  std::uint32_t local;          // launch index within the context (< 4096)
  std::uint64_t* status;
  const std::uint32_t* context; // device context counter
  __device__ __forceinline__ std::uint32_t epoch() const { return (*context << 12) | local; }
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

__device__ __forceinline__ std::uint64_t ld_status(const std::uint64_t* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_status(std::uint64_t* p, std::uint64_t v) {
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ std::uint64_t status_word(std::uint32_t epoch, std::uint64_t flag,
                                                     std::uint64_t count) {
  return (std::uint64_t(epoch) << 32) | flag | count;
}

// Exclusive prefix of `tile` for one lane (digit) by decoupled look-back.
// Eight predecessors' status words are loaded per step (independent loads),
// then consumed newest-first until an inclusive prefix ends the walk; a
// not-yet-published predecessor is re-polled from where the walk stopped.
__device__ __forceinline__ std::uint64_t look_back(const LookBack& lb, std::uint32_t epoch,
                                                   std::uint64_t tile, int stride, int lane_idx) {
  constexpr int kAhead = 8;
  std::uint64_t excl = 0;
  std::int64_t j = std::int64_t(tile) - 1;
  while (j >= 0) {
    std::uint64_t w[kAhead];
#pragma unroll
    for (int q = 0; q < kAhead; ++q)
      w[q] = (j - q >= 0) ? ld_status(lb.status + std::uint64_t(j - q) * stride + lane_idx) : 0;
    // consume newest-first (fully unrolled: w stays in registers)
    int consumed = 0;
    bool stop = false, done = false;
#pragma unroll
    for (int q = 0; q < kAhead; ++q) {
      if (!stop) {
        const std::uint64_t x = w[q];
        if (j - q < 0 || std::uint32_t(x >> 32) != epoch || (x & (kFlagAgg | kFlagInc)) == 0) {
          stop = true;
        } else {
          excl += x & kCountMask;
          ++consumed;
          if (x & kFlagInc) {
            done = true;
            stop = true;
          }
        }
      }
    }
    if (done) return excl;
    j -= consumed;  // re-poll the first unready predecessor (if any)
  }
  return excl;
}

// ------------------------------------------------------------ histogram --

// Digit counts of every pass: hist[p * 256 + d] (p < passes), plus the count
// of a ModDigit when passes == 0 (mod_G > 0).
__global__ void __launch_bounds__(kSortThreads)
    onesweep_hist_kernel(const std::uint64_t* __restrict__ keys, Count cnt_n, int passes,
                         std::uint32_t mod_G, std::uint32_t* __restrict__ hist) {
  pdl_wait();
  __shared__ std::uint32_t h[kMaxPasses * kDigits];
  const int np = passes ? passes : 1;
  for (int i = threadIdx.x; i < np * kDigits; i += kSortThreads) h[i] = 0;
  __syncthreads();
  const std::uint64_t n = cnt_n.get();
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t stride = std::uint64_t(gridDim.x) * kSortThreads;
  for (std::uint64_t base = std::uint64_t(blockIdx.x) * kSortThreads; base < n; base += stride) {
    const std::uint64_t i = base + threadIdx.x;
    const bool valid = i < n;
    const std::uint64_t k = valid ? keys[i] : 0;
    for (int p = 0; p < np; ++p) {
      const std::uint32_t d = !valid ? kDigits
                                     : (passes ? std::uint32_t(k >> (8 * p)) & 0xFFu
                                               : std::uint32_t(k % mod_G));
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
      if (valid && lane == unsigned(__ffs(peers) - 1))
        atomicAdd(&h[p * kDigits + d], unsigned(__popc(peers)));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < np * kDigits; i += kSortThreads)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// In-place exclusive scan of each pass's 256 counts (one CTA per pass).
__global__ void __launch_bounds__(kDigits) onesweep_scan_kernel(std::uint32_t* __restrict__ hist) {
  pdl_wait();
  __shared__ std::uint32_t ws[kDigits / 32];
  std::uint32_t* h = hist + blockIdx.x * kDigits;
  const std::uint32_t v = h[threadIdx.x];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= unsigned(o)) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  std::uint32_t pre = 0;
  for (unsigned w = 0; w < warp; ++w) pre += ws[w];
  h[threadIdx.x] = pre + x - v;
}

// ------------------------------------------------------------ one pass --

template <class Digit, bool kValues>
__global__ void __launch_bounds__(kSortThreads)
    onesweep_pass_kernel(const std::uint64_t* __restrict__ kin,
                         const std::uint32_t* __restrict__ vin, Count cnt_n, Digit dig,
                         const std::uint32_t* __restrict__ digit_base, LookBack lb,
                         std::uint64_t* __restrict__ kout, std::uint32_t* __restrict__ vout) {
  pdl_wait();
  __shared__ std::uint32_t wcnt[kSortWarps][kDigits];
  __shared__ std::uint32_t gbase[kDigits];
  __shared__ std::uint64_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(lb.ticket, 1ull) - lb.base;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kDigits / 32; ++i) wcnt[warp][lane + 32 * i] = 0;
  __syncthreads();
  const std::uint64_t tile = s_tile;
  const std::uint64_t n = cnt_n.get();
  const std::uint64_t base = tile * kSortTile;
  if (base >= n) return;  // trailing tiles of an upper-bound grid: nobody waits on them
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
    if (valid && lane == unsigned(__ffs(peers) - 1)) wcnt[warp][d] = prior + unsigned(__popc(peers));
    __syncwarp();
  }
  __syncthreads();
  {
    const unsigned d = threadIdx.x;  // one thread per digit
    std::uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const std::uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    std::uint64_t* my = lb.status + tile * kDigits + d;
    const std::uint32_t ep = lb.epoch();
    if (tile == 0) {
      st_status(my, status_word(ep, kFlagInc, run));
      gbase[d] = digit_base[d];
    } else {
      st_status(my, status_word(ep, kFlagAgg, run));
      const std::uint64_t excl = look_back(lb, ep, tile, kDigits, d);
      st_status(my, status_word(ep, kFlagInc, excl + run));
      gbase[d] = digit_base[d] + std::uint32_t(excl);
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

// ---------------------------------------------------------- tile scan ----
//
// Single-pass exclusive scan with decoupled look-back.
//   F  : __device__ std::uint32_t operator()(std::uint64_t i) const — item value
//   Em : __device__ void operator()(std::uint64_t i, std::uint32_t v,
//                                    std::uint64_t exclusive_prefix) const
// The grand total goes to *total (written by the tile holding item n-1).

constexpr int kScanItems = 16;
constexpr int kScanTile = kSortThreads * kScanItems;  // 4096

template <class F, class Em>
__global__ void __launch_bounds__(kSortThreads)
    scan_lookback_kernel(F f, Em em, Count cnt_n, LookBack lb, std::uint64_t* __restrict__ total) {
  pdl_wait();
  __shared__ std::uint32_t ws[kSortWarps];
  __shared__ std::uint64_t s_tile, s_pre;
  if (threadIdx.x == 0) s_tile = atomicAdd(lb.ticket, 1ull) - lb.base;
  __syncthreads();
  const std::uint64_t tile = s_tile;
  const std::uint64_t n = cnt_n.get();
  const std::uint64_t base = tile * kScanTile;
  if (base >= n) {
    if (tile == 0 && total) *total = 0;
    return;
  }
  // warp-striped arrangement: warp w owns items base + w*512 .. +511, and in
  // round it its lane handles item + it*32 + lane (coalesced loads; the
  // emits see exactly the same exclusive prefixes as a blocked walk)
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint64_t wb = base + std::uint64_t(warp) * (32 * kScanItems);
  std::uint32_t vals[kScanItems];
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const std::uint64_t idx = wb + it * 32 + lane;
    vals[it] = idx < n ? f(idx) : 0u;
  }
  // per round: inclusive scan across the lanes; rounds chain in order
  std::uint32_t incl[kScanItems];
  std::uint32_t wtot = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    std::uint32_t x = vals[it];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= unsigned(o)) x += y;
    }
    incl[it] = wtot + x;  // within the warp's 512 items
    wtot += __shfl_sync(0xFFFFFFFFu, x, 31);
  }
  if (lane == 0) ws[warp] = wtot;
  __syncthreads();
  if (threadIdx.x == 0) {
    std::uint32_t agg = 0;
    for (int w = 0; w < kSortWarps; ++w) agg += ws[w];
    std::uint64_t* my = lb.status + tile;
    std::uint64_t pre = 0;
    const std::uint32_t ep = lb.epoch();
    if (tile == 0) {
      st_status(my, status_word(ep, kFlagInc, agg));
    } else {
      st_status(my, status_word(ep, kFlagAgg, agg));
      pre = look_back(lb, ep, tile, 1, 0);
      st_status(my, status_word(ep, kFlagInc, pre + agg));
    }
    s_pre = pre;
    if (total && base + kScanTile >= n) *total = pre + agg;
  }
  __syncthreads();
  std::uint32_t wpre = 0;
  for (unsigned w = 0; w < warp; ++w) wpre += ws[w];
  const std::uint64_t run = s_pre + wpre;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const std::uint64_t idx = wb + it * 32 + lane;
    if (idx < n) em(idx, vals[it], run + incl[it] - vals[it]);
  }
}

inline std::uint32_t sort_tiles(std::uint64_t n) {
  return std::uint32_t((n + kSortTile - 1) / kSortTile);
}
inline std::uint32_t scan_tiles(std::uint64_t n) {
  return std::uint32_t((n + kScanTile - 1) / kScanTile);
}

}  // namespace hpsgpu

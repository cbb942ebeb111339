// Mini-batch dedup without sorting (G == 1): group the occurrences of a shard
// by their slot in the batch's HBM table (every key of the batch is there),
// producing exactly what the sort-based dedup produces for the consumers —
// per unique key u: its occurrences' example ids exs[seg[u] .. seg[u+1]) in
// occurrence order (the reference's per-key order of backward's sparse
// accumulation, model.hpp:182-187), and per occurrence q its key's uid
// inv[q] — but with uids in claim order and the table slot of every uid known
// (uid_slot), so the pull is the table row itself (hbm_ps.hpp:112-143 at a
// single device: get() copies the very rows the table holds).
//
//   group_probe_kernel  position-major: lane = shard example, loop over
//                       feature positions; probe the slot, __match_any_sync
//                       over the warp (sorted features put a hot key at the
//                       same position in most examples), one atomicAdd per
//                       distinct slot per warp returns the lanes' tickets;
//                       the first touch of a slot claims its uid.
//   (tile scan)         seg = exclusive scan of the uid counts.
//   group_compact_kernel dense uids from the partitioned claims.
//   group_place_kernel  occurrence q -> position seg[uid] + ticket.
// Occurrence ids are batch key indices (off[ex] + position): unique, and in
// the shard's occurrence order.
//   group_order_kernel  segments <= kGroupShort: one thread sorts its few
//                       occurrence ids (insertion) and writes exs; longer
//                       ones are queued.
//   group_warp_kernel / group_cta_kernel
//                       longer segments, a warp / a CTA each: a shared-memory
//                       bitmap over the shard's examples ranks every
//                       occurrence in O(n + examples/32), no comparison sort;
//                       group_dup_kernel handles inputs that repeat a key
//                       inside an example.
#pragma once

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace hpsgpu {

constexpr int kGroupShort = 8;      // segments ordered in registers by one thread
constexpr int kGroupThreads = 1024;
constexpr int kGroupPosGroups = 64;  // warps sharing one 32-example group
constexpr int kGroupWarpThreads = 256;  // group_warp_kernel: one warp per segment
constexpr int kGroupSortThreads = 512;  // group_sort_kernel (a block per huge segment)
constexpr int kGroupWarpMax = 256;      // longer segments: one CTA each (group_cta_kernel)
constexpr int kGroupParts = 32;         // uid claim counters (contention / kGroupParts)
constexpr int kGroupPartStride = 32;    // u32 words between counters (one 128-B line each)
constexpr std::size_t kGroupSmemMax = 200 * 1024;

// Request table (G > 1): every key of this rank's shards once, so grouping
// has a slot per key whoever owns it. Unordered CAS insert (the table is
// internal, its layout free), read-first for hot keys. Warp per example.
__global__ void rq_insert_kernel(const std::int64_t* __restrict__ off,
                                 const std::uint64_t* __restrict__ keys, std::uint64_t B, int G,
                                 int g, int J, std::uint64_t* __restrict__ rq,
                                 const std::uint64_t* __restrict__ cap_ptr) {
  pdl_wait();
  const std::uint64_t cap = *cap_ptr, GJ = std::uint64_t(G) * J;
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t nw = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (std::uint64_t i = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5; i < B;
       i += nw) {
    if ((i % GJ) / J != std::uint64_t(g)) continue;
    const std::int64_t b = off[i], e = off[i + 1];
    for (std::int64_t p = b + lane; p < e; p += 32) {
      const std::uint64_t k = keys[p];
      std::uint64_t idx = mix64(k) & (cap - 1);
      for (;;) {
        const std::uint64_t seen = *reinterpret_cast<volatile const std::uint64_t*>(rq + idx);
        if (seen == k) break;
        if (seen == kEmptyKey) {
          const unsigned long long old =
              atomicCAS(reinterpret_cast<unsigned long long*>(rq + idx), kEmptyKey, k);
          if (old == kEmptyKey || old == k) break;
        }
        idx = (idx + 1) & (cap - 1);
      }
    }
  }
}

// Warp w: examples 32*(w / kGroupPosGroups) + lane, feature positions
// p = w % kGroupPosGroups (mod kGroupPosGroups), in lock-step across the
// lanes. Writes occ_slot[q], tick[q], ex_of[q]; counts per slot in cnt (zero
// on entry); uid claim: slot_uid[slot], uid_slot[uid], *n_uid.
__global__ void group_probe_kernel(ShardMap sm, const std::int64_t* __restrict__ off,
                                   const std::uint64_t* __restrict__ keys,
                                   const std::uint64_t* __restrict__ tkeys,
                                   const std::uint64_t* __restrict__ cap_ptr,
                                   std::uint32_t* __restrict__ cnt,
                                   std::uint32_t* __restrict__ slot_uid,
                                   std::uint32_t* __restrict__ part_slot,
                                   std::uint32_t part_cap,
                                   std::uint32_t* __restrict__ part_n,
                                   std::uint32_t* __restrict__ occ_slot,
                                   std::uint32_t* __restrict__ tick,
                                   std::uint32_t* __restrict__ ex_of, DevError* err,
                                   bool ordered) {
  pdl_wait();
  const std::uint64_t cap = *cap_ptr;
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const std::uint64_t nw = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (std::uint64_t w = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5;
       (w / kGroupPosGroups) * 32 < sm.count; w += nw) {
    const int pg = int(w % kGroupPosGroups);
    const std::uint64_t k = (w / kGroupPosGroups) * 32 + lane;
    const bool has = k < sm.count;
    std::int64_t b = 0, len = 0;
    if (has) {
      const std::uint64_t ex = sm.first + k * sm.stride;
      b = off[ex];
      len = off[ex + 1] - b;
    }
    std::int64_t maxlen = len;
    for (int o = 16; o > 0; o >>= 1) {
      const std::int64_t y = __shfl_xor_sync(0xFFFFFFFFu, maxlen, o);
      maxlen = y > maxlen ? y : maxlen;
    }
    for (std::int64_t p = pg; p < maxlen; p += kGroupPosGroups) {
      const bool act = p < len;
      std::uint32_t slot = kNoSlot;
      if (act) {
        slot = ordered ? probe_slot_ordered(tkeys, cap, keys[b + p])  // the batch table
                       : probe_slot(tkeys, cap, keys[b + p]);         // G > 1: request table
        if (slot == kNoSlot) raise_error(err, 1, keys[b + p]);
      }
      const unsigned am = __ballot_sync(0xFFFFFFFFu, act && slot != kNoSlot);
      unsigned match = 0;
      if (act && slot != kNoSlot) match = __match_any_sync(am, slot);
      const bool leader = match && lane == unsigned(__ffs(match) - 1);
      std::uint32_t base = 0;
      bool fresh = false;
      if (leader) {
        base = atomicAdd(&cnt[slot], std::uint32_t(__popc(match)));
        fresh = base == 0;
      }
      // first touch of a slot: claim an id in this block's partition
      // (warp-aggregated; group_compact_kernel makes the ids dense)
      const unsigned fm = __ballot_sync(0xFFFFFFFFu, fresh);
      if (fm) {
        const unsigned part = blockIdx.x % kGroupParts;
        std::uint32_t u0 = 0;
        if (lane == unsigned(__ffs(fm) - 1))
          u0 = atomicAdd(&part_n[part * kGroupPartStride], std::uint32_t(__popc(fm)));
        u0 = __shfl_sync(0xFFFFFFFFu, u0, __ffs(fm) - 1);
        if (fresh) {
          const std::uint32_t i = u0 + std::uint32_t(__popc(fm & lt));
          slot_uid[slot] = part * part_cap + i;  // partition-local id, made dense later
          part_slot[std::size_t(part) * part_cap + i] = slot;
        }
      }
      const std::uint32_t lb = __shfl_sync(0xFFFFFFFFu, base, match ? __ffs(match) - 1 : lane);
      if (match) {
        const std::uint32_t q = std::uint32_t(b + p);  // occurrence id = batch key index
        occ_slot[q] = slot;
        tick[q] = lb + std::uint32_t(__popc(match & lt));
        ex_of[q] = std::uint32_t(k);
      }
    }
  }
}

// Dense uids: partition p's ids follow the ids of partitions < p. Every
// block derives the bases itself; block 0 publishes them and *n_uid; the
// grid fills uid_slot (dense). (group_order_kernel resets the counters.)
__global__ void group_compact_kernel(const std::uint32_t* __restrict__ part_n,
                                     const std::uint32_t* __restrict__ part_slot,
                                     std::uint32_t part_cap, std::uint32_t* __restrict__ part_base,
                                     std::uint32_t* __restrict__ uid_slot,
                                     unsigned long long* __restrict__ n_uid) {
  pdl_wait();
  __shared__ std::uint32_t base[kGroupParts + 1];
  if (threadIdx.x == 0) {
    std::uint32_t run = 0;
    for (int p = 0; p < kGroupParts; ++p) {
      base[p] = run;
      run += part_n[p * kGroupPartStride];
    }
    base[kGroupParts] = run;
    if (blockIdx.x == 0) *n_uid = run;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < kGroupParts) part_base[threadIdx.x] = base[threadIdx.x];
  const std::uint32_t U = base[kGroupParts];
  for (std::uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < U;
       u += gridDim.x * blockDim.x) {
    int lo = 0, hi = kGroupParts;  // last partition with base <= u
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (base[mid] <= u) lo = mid; else hi = mid;
    }
    uid_slot[u] = part_slot[std::size_t(lo) * part_cap + (u - base[lo])];
  }
}

__device__ __forceinline__ std::uint32_t dense_uid(std::uint32_t packed, std::uint32_t part_cap,
                                                   const std::uint32_t* part_base) {
  const std::uint32_t p = packed / part_cap;
  return part_base[p] + (packed - p * part_cap);
}

// G > 1: the unique keys of a grouped mini-batch in uid order (the exchange
// sends them to their owners), from the request table.
__global__ void uid_keys_kernel(const std::uint32_t* __restrict__ uid_slot,
                                const std::uint64_t* __restrict__ rq,
                                const unsigned long long* __restrict__ n_uid,
                                std::uint64_t* __restrict__ ukeys,
                                unsigned long long* __restrict__ u_out) {
  pdl_wait();
  const std::uint64_t U = *n_uid;
  if (blockIdx.x == 0 && threadIdx.x == 0) *u_out = U;  // the exchange's key count
  for (std::uint64_t u = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; u < U;
       u += std::uint64_t(gridDim.x) * blockDim.x)
    ukeys[u] = rq[uid_slot[u]];
}

struct UidCount {  // count of uid u's occurrences (for the segment scan)
  const std::uint32_t* uid_slot;
  const std::uint32_t* cnt;
  __device__ std::uint32_t operator()(std::uint64_t u) const { return cnt[uid_slot[u]]; }
};
struct SegEmit {
  std::uint32_t* seg;
  Count n;
  __device__ void operator()(std::uint64_t u, std::uint32_t v, std::uint64_t pre) const {
    seg[u] = std::uint32_t(pre);
    if (u + 1 == n.get()) seg[u + 1] = std::uint32_t(pre + v);
  }
};

// Occurrence q (a batch key index of this shard) -> its position in the
// segment (unordered for now), and (G > 1, rows arrive in uid order) its uid
// inv[q]. One warp per example, lanes over its positions.
__global__ void group_place_kernel(ShardMap sm, const std::int64_t* __restrict__ off,
                                   const std::uint32_t* __restrict__ occ_slot,
                                   const std::uint32_t* __restrict__ tick,
                                   const std::uint32_t* __restrict__ slot_uid,
                                   std::uint32_t part_cap,
                                   const std::uint32_t* __restrict__ part_base,
                                   const std::uint32_t* __restrict__ seg,
                                   std::uint32_t* __restrict__ seg_occ,
                                   std::uint32_t* __restrict__ inv,
                                   std::uint32_t* __restrict__ cnt,
                                   std::uint32_t* __restrict__ part_n,
                                   std::uint32_t* __restrict__ long_list,
                                   unsigned long long* __restrict__ n_long,
                                   std::uint32_t* __restrict__ huge_list,
                                   unsigned long long* __restrict__ n_huge) {
  pdl_wait();
  __shared__ std::uint32_t pb[kGroupParts];
  if (threadIdx.x < kGroupParts) pb[threadIdx.x] = part_base[threadIdx.x];
  __syncthreads();
  // the claim counters are read (group_compact) and free again
  if (cnt && blockIdx.x == 0 && threadIdx.x < kGroupParts)
    part_n[threadIdx.x * kGroupPartStride] = 0;
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t nw = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (std::uint64_t k = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5;
       k < sm.count; k += nw) {
    const std::uint64_t ex = sm.first + k * sm.stride;
    const std::int64_t b = off[ex], e = off[ex + 1];
    for (std::int64_t q = b + lane; q < e; q += 32) {
      const std::uint32_t sl = occ_slot[q];
      const std::uint32_t u = dense_uid(slot_uid[sl], part_cap, pb);
      const std::uint32_t t = tick[q];
      seg_occ[seg[u] + t] = std::uint32_t(q);
      if (inv) inv[q] = u;
      if (cnt && t == 0) {  // one occurrence per key: its counter and its list
        cnt[sl] = 0;        // (the segment scan has read it)
        const std::uint32_t n = seg[u + 1] - seg[u];
        if (n > std::uint32_t(kGroupWarpMax)) huge_list[atomicAdd(n_huge, 1ull)] = u;
        else if (n > std::uint32_t(kGroupShort)) long_list[atomicAdd(n_long, 1ull)] = u;
      }
    }
  }
}

// Short segments (<= kGroupShort): one thread sorts the occurrence ids in
// registers (insertion) and writes exs; longer ones go to long_list. Also
// clears the uid's slot counter.
__global__ void group_order_kernel(const unsigned long long* __restrict__ n_uid,
                                   const std::uint32_t* __restrict__ seg,
                                   std::uint32_t* __restrict__ seg_occ,
                                   const std::uint32_t* __restrict__ ex_of,
                                   const std::uint32_t* __restrict__ uid_slot,
                                   std::uint32_t* __restrict__ cnt,
                                   std::uint32_t* __restrict__ exs,
                                   std::uint32_t* __restrict__ long_list,
                                   unsigned long long* __restrict__ n_long,
                                   std::uint32_t* __restrict__ huge_list,
                                   unsigned long long* __restrict__ n_huge,
                                   std::uint32_t* __restrict__ part_n) {
  pdl_wait();
  const std::uint64_t U = *n_uid;
  if (blockIdx.x == 0 && threadIdx.x < kGroupParts) part_n[threadIdx.x * kGroupPartStride] = 0;
  for (std::uint64_t u = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; u < U;
       u += std::uint64_t(gridDim.x) * blockDim.x) {
    cnt[uid_slot[u]] = 0;
    const std::uint32_t p0 = seg[u];
    const int n = int(seg[u + 1] - p0);
    if (n > kGroupWarpMax) {
      huge_list[atomicAdd(n_huge, 1ull)] = std::uint32_t(u);
      continue;
    }
    if (n > kGroupShort) {
      long_list[atomicAdd(n_long, 1ull)] = std::uint32_t(u);
      continue;
    }
    std::uint32_t v[kGroupShort];
#pragma unroll
    for (int i = 0; i < kGroupShort; ++i) v[i] = i < n ? seg_occ[p0 + i] : 0xFFFFFFFFu;
    // sorting network on kGroupShort registers (padding sorts last)
#pragma unroll
    for (int i = 1; i < kGroupShort; ++i)
#pragma unroll
      for (int j = i; j > 0; --j) {
        const std::uint32_t a = v[j - 1], b = v[j];
        v[j - 1] = min(a, b);
        v[j] = max(a, b);
      }
#pragma unroll
    for (int i = 0; i < kGroupShort; ++i)
      if (i < n) exs[p0 + i] = ex_of[v[i]];
  }
}

// Sets bit e of bm for every active lane; lanes sharing a word combine their
// bits first (one write per word). True if a bit was already set (a repeat).
__device__ __forceinline__ bool set_bits(std::uint32_t* bm, std::uint32_t e, bool act) {
  const unsigned am = __ballot_sync(0xFFFFFFFFu, act);
  bool dup = false;
  if (act) {
    const unsigned grp = __match_any_sync(am, e >> 5);
    const std::uint32_t bit = 1u << (e & 31);
    const std::uint32_t all = __reduce_or_sync(grp, bit);
    if (threadIdx.x % 32 == unsigned(__ffs(grp) - 1)) {
      const std::uint32_t old = atomicOr(&bm[e >> 5], all);
      dup = (old & all) != 0 || __popc(all) != __popc(grp);
    }
  }
  return dup;
}

// Longer segments (<= kGroupWarpMax), one warp each: rank by shard example
// id through a bitmap over the shard's examples in shared memory (an example
// holds a key at most once unless the input repeats it, so example order is
// occurrence order). Each lane stages its <= kGroupWarpMax/32 ids in
// registers (two rounds of independent loads). A repeat (a bit already set)
// sends the segment to group_dup_kernel.
__global__ void __launch_bounds__(kGroupWarpThreads)
    group_warp_kernel(const unsigned long long* __restrict__ n_long,
                      const std::uint32_t* __restrict__ long_list,
                      const std::uint32_t* __restrict__ seg,
                      const std::uint32_t* __restrict__ seg_occ,
                      const std::uint32_t* __restrict__ ex_of, std::uint32_t words,
                      std::uint32_t* __restrict__ exs, std::uint32_t* __restrict__ dup_list,
                      unsigned long long* __restrict__ n_dup) {
  pdl_wait();
  constexpr int R = kGroupWarpMax / 32;
  extern __shared__ std::uint32_t wsm[];  // per warp: bitmap[words], prefix[words]
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  std::uint32_t* bm = wsm + std::size_t(warp) * 2 * words;
  std::uint32_t* pre = bm + words;
  const std::uint64_t NL = *n_long;
  const std::uint64_t nwarps = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (std::uint64_t li = std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + warp; li < NL;
       li += nwarps) {
    const std::uint32_t u = long_list[li];
    const std::uint32_t p0 = seg[u], p1 = seg[u + 1];
    std::uint32_t ev[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const std::uint32_t p = p0 + r * 32 + lane;
      ev[r] = p < p1 ? seg_occ[p] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) ev[r] = ev[r] != 0xFFFFFFFFu ? ex_of[ev[r]] : 0xFFFFFFFFu;
    for (std::uint32_t i = lane; i < words; i += 32) bm[i] = 0;
    __syncwarp();
    bool dup = false;
#pragma unroll
    for (int r = 0; r < R; ++r) dup |= set_bits(bm, ev[r], ev[r] != 0xFFFFFFFFu);
    if (__any_sync(0xFFFFFFFFu, dup)) {
      if (lane == 0) dup_list[atomicAdd(n_dup, 1ull)] = u;
      continue;
    }
    __syncwarp();
    // exclusive prefix of popcounts, each lane a contiguous run of words
    const std::uint32_t per = (words + 31) / 32;
    const std::uint32_t w0 = lane * per, w1 = min(words, w0 + per);
    std::uint32_t mine = 0;
    for (std::uint32_t i = w0; i < w1; ++i) mine += __popc(bm[i]);
    std::uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= unsigned(o)) x += y;
    }
    std::uint32_t run = x - mine;
    for (std::uint32_t i = w0; i < w1; ++i) {
      pre[i] = run;
      run += __popc(bm[i]);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const std::uint32_t e = ev[r];
      if (e == 0xFFFFFFFFu) continue;
      const std::uint32_t rk = pre[e >> 5] + __popc(bm[e >> 5] & ((1u << (e & 31)) - 1u));
      exs[p0 + rk] = e;
    }
    __syncwarp();
  }
}

// Segments longer than kGroupWarpMax, one CTA each: the same example bitmap
// (words = ceil(shard examples / 32)), block-wide prefix.
__global__ void __launch_bounds__(kGroupThreads)
    group_cta_kernel(const unsigned long long* __restrict__ n_huge,
                     const std::uint32_t* __restrict__ huge_list,
                     const std::uint32_t* __restrict__ seg,
                     const std::uint32_t* __restrict__ seg_occ,
                     const std::uint32_t* __restrict__ ex_of, std::uint32_t words,
                     std::uint32_t* __restrict__ exs, std::uint32_t* __restrict__ dup_list,
                     unsigned long long* __restrict__ n_dup) {
  pdl_wait();
  extern __shared__ std::uint32_t cbm[];  // bitmap[words], prefix[words]
  __shared__ std::uint32_t wsum[kGroupThreads / 32];
  __shared__ int s_dup;
  std::uint32_t* pre = cbm + words;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const std::uint64_t NH = *n_huge;
  for (std::uint64_t li = blockIdx.x; li < NH; li += gridDim.x) {
    const std::uint32_t u = huge_list[li];
    const std::uint32_t p0 = seg[u], p1 = seg[u + 1];
    for (std::uint32_t i = threadIdx.x; i < words; i += blockDim.x) cbm[i] = 0;
    if (threadIdx.x == 0) s_dup = 0;
    __syncthreads();
    constexpr int R = 4;  // independent loads in flight per thread
    for (std::uint32_t b0 = p0 + warp * 32; b0 < p1; b0 += blockDim.x * R) {  // warp-uniform
      std::uint32_t ev[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const std::uint32_t p = b0 + r * blockDim.x + lane;
        ev[r] = p < p1 ? seg_occ[p] : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) ev[r] = ev[r] != 0xFFFFFFFFu ? ex_of[ev[r]] : 0xFFFFFFFFu;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (set_bits(cbm, ev[r], ev[r] != 0xFFFFFFFFu)) s_dup = 1;
    }
    __syncthreads();
    if (s_dup) {
      if (threadIdx.x == 0) dup_list[atomicAdd(n_dup, 1ull)] = u;
      __syncthreads();
      continue;
    }
    const std::uint32_t per = (words + blockDim.x - 1) / blockDim.x;
    const std::uint32_t w0 = threadIdx.x * per, w1 = min(words, w0 + per);
    std::uint32_t mine = 0;
    for (std::uint32_t i = w0; i < w1; ++i) mine += __popc(cbm[i]);
    std::uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= unsigned(o)) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    std::uint32_t run = x - mine;
    for (unsigned w = 0; w < warp; ++w) run += wsum[w];
    for (std::uint32_t i = w0; i < w1; ++i) {
      pre[i] = run;
      run += __popc(cbm[i]);
    }
    __syncthreads();
    for (std::uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
      const std::uint32_t e = ex_of[seg_occ[p]];
      const std::uint32_t r = pre[e >> 5] + __popc(cbm[e >> 5] & ((1u << (e & 31)) - 1u));
      exs[p0 + r] = e;
    }
    __syncthreads();
  }
}

// Segments whose examples repeat the key (only when the input repeats a
// feature inside an example): rank of each occurrence id by counting the
// smaller ids of the segment (O(n^2) over the CTA; a correctness path).
__global__ void __launch_bounds__(kGroupThreads)
    group_dup_kernel(const unsigned long long* __restrict__ n_dup,
                     const std::uint32_t* __restrict__ dup_list,
                     const std::uint32_t* __restrict__ seg,
                     const std::uint32_t* __restrict__ seg_occ,
                     const std::uint32_t* __restrict__ ex_of, std::uint32_t* __restrict__ exs) {
  pdl_wait();
  const std::uint64_t ND = *n_dup;
  for (std::uint64_t li = blockIdx.x; li < ND; li += gridDim.x) {
    const std::uint32_t u = dup_list[li];
    const std::uint32_t p0 = seg[u], p1 = seg[u + 1];
    for (std::uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
      const std::uint32_t q = seg_occ[p];
      std::uint32_t r = 0;
      for (std::uint32_t i = p0; i < p1; ++i) r += seg_occ[i] < q;
      exs[p0 + r] = ex_of[q];
    }
  }
}

// The whole segment ordering in ONE launch (HPS_GROUP_FUSED=1, the
// default; group_order + group_warp + group_cta + group_dup otherwise), after
// group_place has listed the longer segments: every block first orders the
// short segments (<= kGroupShort) of its share of the uids in registers, then
// takes the huge segments (> kGroupWarpMax) one per block, then its warps take
// the long ones one per warp — the same example-bitmap ranks as above. A
// segment whose examples repeat its key (the input repeats a feature inside
// an example) is ranked in place by counting smaller occurrence ids.
__device__ __forceinline__ void rank_by_count(std::uint32_t p0, std::uint32_t p1,
                                              const std::uint32_t* __restrict__ seg_occ,
                                              const std::uint32_t* __restrict__ ex_of,
                                              std::uint32_t* __restrict__ exs, unsigned t,
                                              unsigned nt) {
  for (std::uint32_t p = p0 + t; p < p1; p += nt) {
    const std::uint32_t q = seg_occ[p];
    std::uint32_t r = 0;
    for (std::uint32_t i = p0; i < p1; ++i) r += seg_occ[i] < q;
    exs[p0 + r] = ex_of[q];
  }
}

__global__ void __launch_bounds__(kGroupSortThreads)
    group_sort_kernel(const unsigned long long* __restrict__ n_uid,
                      const std::uint32_t* __restrict__ seg,
                      const std::uint32_t* __restrict__ seg_occ,
                      const std::uint32_t* __restrict__ ex_of, std::uint32_t words,
                      std::uint32_t* __restrict__ exs,
                      const unsigned long long* __restrict__ n_long,
                      const std::uint32_t* __restrict__ long_list,
                      const unsigned long long* __restrict__ n_huge,
                      const std::uint32_t* __restrict__ huge_list) {
  pdl_wait();
  extern __shared__ std::uint32_t gsort_sm[];  // per warp: bitmap[words], prefix[words]
  __shared__ std::uint32_t wsum[kGroupSortThreads / 32];
  __shared__ int s_dup;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr unsigned kWarps = kGroupSortThreads / 32;
  // ---- short segments: one thread each, in registers
  const std::uint64_t U = *n_uid;
  for (std::uint64_t u = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; u < U;
       u += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint32_t p0 = seg[u];
    const int n = int(seg[u + 1] - p0);
    if (n > kGroupShort) continue;
    std::uint32_t v[kGroupShort];
#pragma unroll
    for (int i = 0; i < kGroupShort; ++i) v[i] = i < n ? seg_occ[p0 + i] : 0xFFFFFFFFu;
#pragma unroll
    for (int i = 1; i < kGroupShort; ++i)
#pragma unroll
      for (int j = i; j > 0; --j) {
        const std::uint32_t a = v[j - 1], b = v[j];
        v[j - 1] = min(a, b);
        v[j] = max(a, b);
      }
#pragma unroll
    for (int i = 0; i < kGroupShort; ++i)
      if (i < n) exs[p0 + i] = ex_of[v[i]];
  }
  // ---- huge segments: one block each (bitmap over the block's smem)
  {
    std::uint32_t* cbm = gsort_sm;
    std::uint32_t* pre = gsort_sm + words;
    const std::uint64_t NH = *n_huge;
    for (std::uint64_t li = blockIdx.x; li < NH; li += gridDim.x) {
      const std::uint32_t u = huge_list[li];
      const std::uint32_t p0 = seg[u], p1 = seg[u + 1];
      for (std::uint32_t i = threadIdx.x; i < words; i += blockDim.x) cbm[i] = 0;
      if (threadIdx.x == 0) s_dup = 0;
      __syncthreads();
      constexpr int R = 4;
      for (std::uint32_t b0 = p0 + warp * 32; b0 < p1; b0 += blockDim.x * R) {
        std::uint32_t ev[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const std::uint32_t p = b0 + r * blockDim.x + lane;
          ev[r] = p < p1 ? seg_occ[p] : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) ev[r] = ev[r] != 0xFFFFFFFFu ? ex_of[ev[r]] : 0xFFFFFFFFu;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (set_bits(cbm, ev[r], ev[r] != 0xFFFFFFFFu)) s_dup = 1;
      }
      __syncthreads();
      if (s_dup) {
        rank_by_count(p0, p1, seg_occ, ex_of, exs, threadIdx.x, blockDim.x);
        __syncthreads();
        continue;
      }
      const std::uint32_t per = (words + blockDim.x - 1) / blockDim.x;
      const std::uint32_t w0 = threadIdx.x * per, w1 = min(words, w0 + per);
      std::uint32_t mine = 0;
      for (std::uint32_t i = w0; i < w1; ++i) mine += __popc(cbm[i]);
      std::uint32_t x = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= unsigned(o)) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      std::uint32_t run = x - mine;
      for (unsigned w = 0; w < warp; ++w) run += wsum[w];
      for (std::uint32_t i = w0; i < w1; ++i) {
        pre[i] = run;
        run += __popc(cbm[i]);
      }
      __syncthreads();
      for (std::uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const std::uint32_t e = ex_of[seg_occ[p]];
        const std::uint32_t r = pre[e >> 5] + __popc(cbm[e >> 5] & ((1u << (e & 31)) - 1u));
        exs[p0 + r] = e;
      }
      __syncthreads();
    }
  }
  // ---- long segments: one warp each
  {
    constexpr int R = kGroupWarpMax / 32;
    std::uint32_t* bm = gsort_sm + std::size_t(warp) * 2 * words;
    std::uint32_t* pre = bm + words;
    // the blocks that ordered a huge segment take no long ones (they are the
    // grid's tail); the rest share them
    const std::uint64_t NL = *n_long;
    const std::uint64_t NH0 = *n_huge, gl = std::uint64_t(gridDim.x) - 1;
    const std::uint64_t NHb = NH0 < gl ? NH0 : gl;
    if (blockIdx.x < NHb) return;
    const std::uint64_t nwarps = (std::uint64_t(gridDim.x) - NHb) * kWarps;
    for (std::uint64_t li = (std::uint64_t(blockIdx.x) - NHb) * kWarps + warp; li < NL;
         li += nwarps) {
      const std::uint32_t u = long_list[li];
      const std::uint32_t p0 = seg[u], p1 = seg[u + 1];
      std::uint32_t ev[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const std::uint32_t p = p0 + r * 32 + lane;
        ev[r] = p < p1 ? seg_occ[p] : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) ev[r] = ev[r] != 0xFFFFFFFFu ? ex_of[ev[r]] : 0xFFFFFFFFu;
      for (std::uint32_t i = lane; i < words; i += 32) bm[i] = 0;
      __syncwarp();
      bool dup = false;
#pragma unroll
      for (int r = 0; r < R; ++r) dup |= set_bits(bm, ev[r], ev[r] != 0xFFFFFFFFu);
      if (__any_sync(0xFFFFFFFFu, dup)) {
        rank_by_count(p0, p1, seg_occ, ex_of, exs, lane, 32);
        __syncwarp();
        continue;
      }
      __syncwarp();
      const std::uint32_t per = (words + 31) / 32;
      const std::uint32_t w0 = lane * per, w1 = min(words, w0 + per);
      std::uint32_t mine = 0;
      for (std::uint32_t i = w0; i < w1; ++i) mine += __popc(bm[i]);
      std::uint32_t x = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= unsigned(o)) x += y;
      }
      std::uint32_t run = x - mine;
      for (std::uint32_t i = w0; i < w1; ++i) {
        pre[i] = run;
        run += __popc(bm[i]);
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const std::uint32_t e = ev[r];
        if (e == 0xFFFFFFFFu) continue;
        const std::uint32_t rk = pre[e >> 5] + __popc(bm[e >> 5] & ((1u << (e & 31)) - 1u));
        exs[p0 + rk] = e;
      }
      __syncwarp();
    }
  }
}

}  // namespace hpsgpu

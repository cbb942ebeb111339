// HBM-resident open-addressing table of one rank (the DeviceTable of
// device_table.hpp:32-137, rebuilt per batch by HbmTier::build_node,
// hbm_ps.hpp:65-102).
//
// Layout: keys u64[cap] (EMPTY = ~0) and rows f32[cap][E] (row-major, E
// contiguous, 16-B aligned when E % 4 == 0). The capacity lives in device
// memory (it depends on the working-set size the GPU just computed).
//
// Build is history-independent "ordered linear probing": each key walks its
// probe sequence doing 64-bit atomicMin; a smaller key takes the slot and
// the displaced larger key continues from the next slot. The fixpoint is
// the layout the reference produces by inserting keys in ascending order
// (hbm_ps.hpp:89-98): every key ends at the first slot of its probe
// sequence not held by a smaller key. Rows are filled afterwards (atomics
// cannot carry the value).
#pragma once

#include <cstdint>
#include <type_traits>

#include "common.cuh"

namespace hpsgpu {

__global__ void table_clear_kernel(std::uint64_t* __restrict__ keys,
                                   const std::uint64_t* __restrict__ cap_ptr,
                                   const unsigned* __restrict__ only_if = nullptr) {
  pdl_wait();
  if (only_if && *only_if == 0u) return;  // conditional pass (graph-stable)
  const std::uint64_t cap = *cap_ptr;
  for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       i < cap; i += std::uint64_t(gridDim.x) * blockDim.x)
    keys[i] = kEmptyKey;
}

__global__ void table_capacity_kernel(const std::uint64_t* __restrict__ n_ptr,
                                      std::uint64_t* __restrict__ cap_ptr) {
  pdl_wait();
  *cap_ptr = table_capacity(*n_ptr);
}

// device_table.hpp:51-73 semantics (duplicate / overflow are errors).
__global__ void table_insert_kernel(const std::uint64_t* __restrict__ ws,
                                    const std::uint64_t* __restrict__ n_ptr,
                                    std::uint64_t* __restrict__ keys,
                                    const std::uint64_t* __restrict__ cap_ptr,
                                    DevError* err) {
  pdl_wait();
  const std::uint64_t n = *n_ptr, cap = *cap_ptr;
  for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       i < n; i += std::uint64_t(gridDim.x) * blockDim.x) {
    std::uint64_t cur = ws[i];
    if (cur == kEmptyKey) {
      raise_error(err, 1 /*HPS_ERR_ARG: reserved key*/, cur);
      continue;
    }
    std::uint64_t idx = mix64(cur) & (cap - 1);
    std::uint64_t probes = 0;
    for (;;) {
      const std::uint64_t old = atomicMin(
          reinterpret_cast<unsigned long long*>(keys + idx),
          static_cast<unsigned long long>(cur));
      if (old == kEmptyKey) break;
      if (old == cur) {
        raise_error(err, 3 /*HPS_ERR_DUPLICATE*/, cur);
        break;
      }
      if (old > cur) cur = old;  // displaced: carry the larger key onward
      idx = (idx + 1) & (cap - 1);
      if (++probes > cap) {
        raise_error(err, 4 /*HPS_ERR_OVERFLOW*/, cur);
        break;
      }
    }
  }
}

// ---- sort-free build from the raw batch keys (hps_train_batch) ---------
//
// 1. table_insert_dedup_kernel, speculative: at the previous table's
//    capacity, counting the distinct keys as they claim empty slots;
//    table_spec_check_kernel redoes the build at the counted capacity when it
//    differs (the layout depends on the capacity, hence on the count).
// 2. table_insert_dedup_kernel: ordered linear probing of every owned
//    occurrence; a thread that meets its own key stops. Ordered probing is
//    history-independent for sets, so the layout equals ascending insertion
//    of the sorted unique keys (hbm_ps.hpp:69-98) without sorting them.
// 3. the live slots are compacted and sorted by key; rows are then filled in
//    key order (table_prefetch_probe / store_gather / table_carry) and
//    written back in key order (table_writeback_sorted).

// Ordered insert of one key (atomicMin, the larger key carried on); true if
// it claimed an EMPTY slot. A table that fills up sets *spec_fail
// (speculative pass) or raises.
constexpr std::uint64_t kSpecProbeLimit = 4096;
__device__ __forceinline__ bool insert_ordered(std::uint64_t cur, std::uint64_t* tkeys,
                                               std::uint64_t cap, unsigned* spec_fail,
                                               DevError* err) {
  const std::uint64_t key = cur;
  std::uint64_t idx = mix64(cur) & (cap - 1);
  for (std::uint64_t probes = 0;; ++probes) {
    // slots only ever decrease: a read that shows cur (present) or a smaller
    // key (advance) decides exactly what the atomic would; hot keys then
    // cost plain cached loads instead of serialised atomics
    const std::uint64_t seen = *reinterpret_cast<volatile const std::uint64_t*>(tkeys + idx);
    if (seen == cur) return false;
    if (seen > cur) {
      const std::uint64_t old = atomicMin(reinterpret_cast<unsigned long long*>(tkeys + idx),
                                          static_cast<unsigned long long>(cur));
      if (old == kEmptyKey) return true;  // placed
      if (old == cur) return false;       // already present
      if (old > cur) cur = old;           // displaced: carry the larger key
    }
    idx = (idx + 1) & (cap - 1);
    // a speculative pass gives up early: at a load factor <= 0.75 probe runs
    // stay far below kSpecProbeLimit, so a run this long means the guessed
    // capacity is too small (or the table is full) and the pass is redone
    if (probes > cap || (spec_fail && probes > kSpecProbeLimit)) {
      if (spec_fail) *spec_fail = 1u;
      else raise_error(err, 4, key);
      return false;
    }
  }
}

// Counts the distinct keys as it goes (every occupied slot is claimed from
// EMPTY exactly once, duplicates and displaced keys included) into *n_new.
// Speculative pass (spec_fail non-null): a table that fills up sets
// *spec_fail instead of raising. only_if non-null: run only if *only_if.
//
// Position-major, like group_probe_kernel: warp w takes examples
// 32*(w / kInsertPosGroups) + lane at feature positions w % kInsertPosGroups
// (mod kInsertPosGroups). Sorted features put a hot key at the same position
// in most examples, so __match_any_sync leaves one lane per distinct key of
// the warp to insert it (a set insert is idempotent) instead of a burst of
// same-address atomics.
constexpr int kInsertPosGroups = 32;
__global__ void table_insert_dedup_kernel(const std::int64_t* __restrict__ off, std::uint64_t B,
                                          const std::uint64_t* __restrict__ keys,
                                          std::uint64_t G, std::uint64_t g,
                                          std::uint64_t* __restrict__ tkeys,
                                          const std::uint64_t* __restrict__ cap_ptr,
                                          DevError* err, unsigned long long* __restrict__ n_new,
                                          unsigned* __restrict__ spec_fail,
                                          const unsigned* __restrict__ only_if) {
  pdl_wait();
  if (only_if && *only_if == 0u) return;
  const std::uint64_t cap = *cap_ptr;
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const std::uint64_t nw = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long placed = 0;
  for (std::uint64_t w = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5;
       (w / kInsertPosGroups) * 32 < B; w += nw) {
    const int pg = int(w % kInsertPosGroups);
    const std::uint64_t ex = (w / kInsertPosGroups) * 32 + lane;
    std::int64_t b = 0, len = 0;
    if (ex < B) {
      b = off[ex];
      len = off[ex + 1] - b;
    }
    std::int64_t maxlen = len;
    for (int o = 16; o > 0; o >>= 1) {
      const std::int64_t y = __shfl_xor_sync(0xFFFFFFFFu, maxlen, o);
      maxlen = y > maxlen ? y : maxlen;
    }
    for (std::int64_t p = pg; p < maxlen; p += kInsertPosGroups) {
      std::uint64_t cur = kEmptyKey;
      bool act = p < len;
      if (act) {
        cur = keys[b + p];
        if (G > 1 && cur % G != g) {  // another rank's key (no 64-bit division at G == 1)
          act = false;
          cur = kEmptyKey;
        } else if (cur == kEmptyKey) {
          raise_error(err, 1, cur);
          act = false;
        }
      }
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, static_cast<unsigned long long>(cur));
      if (act && (peers & lt) == 0u && insert_ordered(cur, tkeys, cap, spec_fail, err)) ++placed;
    }
  }
  for (int o = 16; o > 0; o >>= 1) placed += __shfl_xor_sync(0xFFFFFFFFu, placed, o);
  if (lane == 0 && placed && n_new) atomicAdd(n_new, placed);
}

// After a speculative insert pass (run twice: after the guess, after the
// first redo). The pass's distinct count is exact unless the table filled up
// (or a probe run hit kSpecProbeLimit): then the count stopped early, so the
// redo runs at `fallback` (the capacity of the batch's owned-occurrence bound,
// which holds every distinct key) to get an exact count, and the second check
// redoes once more at the counted capacity if that differs. Otherwise: redo at
// the counted capacity if it differs from the one built, else no redo.
// *redo tells the next clear + insert pass whether to run.
__global__ void table_spec_check_kernel(unsigned long long* __restrict__ n,
                                        std::uint64_t* __restrict__ cap,
                                        unsigned* __restrict__ spec_fail,
                                        unsigned* __restrict__ redo, std::uint64_t fallback) {
  pdl_wait();
  if (*spec_fail) {
    *redo = 1u;
    *cap = fallback;
    *n = 0;
    *spec_fail = 0u;
    return;
  }
  const std::uint64_t needed = table_capacity(*n);
  if (needed != *cap) {
    *redo = 1u;
    *cap = needed;
    *n = 0;
  } else {
    *redo = 0u;
  }
}

// The capacity guess of the speculative build: the previous table's.
__global__ void table_guess_kernel(const std::uint64_t* __restrict__ prev_cap,
                                   std::uint64_t fallback, std::uint64_t* __restrict__ cap) {
  pdl_wait();
  *cap = prev_cap ? *prev_cap : fallback;
}

// Row-source tags in the top bits of csrc (slots stay below 2^30).
constexpr std::uint32_t kSrcMask = 0xC0000000u;
constexpr std::uint32_t kSrcProxy1 = 0x40000000u;  // the table two builds back
constexpr std::uint32_t kSrcProxy2 = 0x80000000u;  // three builds back

// Pipelined build, prep half (runs beside the previous batch's body), in two
// kernels so that PCIe latency never sits behind HBM probes:
// table_prefetch_probe_kernel (full grid, HBM only), one thread per
// working-set entry i (sorted key ws[i], slot wslot[i] in the fresh table):
// csrc[i] = the key's slot in the previous table (copied by
// table_carry_kernel once the previous batch is done, hbm_ps.hpp:86-98), else
// the row comes from the table two (then three) builds back when that holds
// the key (its final rows are exactly what its write-back puts into the store,
// and the newer batches never touched the key), else the key joins the store list
// (warp-contiguous, so in key order within a warp), else the row is zeros.
__global__ void table_prefetch_probe_kernel(
    const std::uint64_t* __restrict__ ws, const std::uint32_t* __restrict__ wslot,
    const std::uint64_t* __restrict__ n_ptr, float* __restrict__ vals,
    std::uint32_t* __restrict__ csrc, const std::uint64_t* __restrict__ prev_keys,
    const std::uint64_t* __restrict__ prev_cap_ptr, const std::uint64_t* __restrict__ old_keys,
    const std::uint64_t* __restrict__ old_cap_ptr, const std::uint64_t* __restrict__ old2_keys,
    const std::uint64_t* __restrict__ old2_cap_ptr, bool from_store, std::uint64_t store_keys, int E, std::uint64_t* __restrict__ need_key,
    std::uint32_t* __restrict__ need_slot, unsigned long long* __restrict__ n_need,
    unsigned long long* carried) {
  pdl_wait();
  const std::uint64_t n = *n_ptr;
  const std::uint64_t pcap = prev_cap_ptr ? *prev_cap_ptr : 0;
  const std::uint64_t ocap = old_cap_ptr ? *old_cap_ptr : 0;
  const std::uint64_t o2cap = old2_cap_ptr ? *old2_cap_ptr : 0;
  const unsigned lane = threadIdx.x & 31;
  unsigned long long n_car = 0;
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  // warp-uniform trip count (the ballots below need the whole warp)
  for (std::uint64_t base = blockIdx.x * std::uint64_t(blockDim.x) + (threadIdx.x & ~31u);
       base < n; base += stride) {
    const std::uint64_t i = base + lane;
    const bool live = i < n;
    const std::uint64_t key = live ? ws[i] : 0;
    const std::uint32_t slot = live ? wslot[i] : 0;
    // the three resident tables probed at once (their home slots load
    // together); ordered tables: a miss stops at the first larger key
    std::uint32_t ps = kNoSlot, os = kNoSlot, o2 = kNoSlot;
    if (live) probe3_ordered(key, prev_keys, pcap, old_keys, ocap, old2_keys, o2cap, &ps, &os, &o2);
    bool need = false;
    if (live && ps == kNoSlot) {
      // newest proxy first: its row is the key's latest. The copy itself is
      // table_carry_kernel's (in the body, when the source rows are final),
      // so this prep never waits for the batches still training.
      std::uint32_t src = kNoSlot;
      if (os != kNoSlot) {
        src = kSrcProxy1 | os;
      } else if (o2 != kNoSlot) {
        src = kSrcProxy2 | o2;
      }
      csrc[i] = src;
      if (src != kNoSlot) {
      } else if (from_store && key < store_keys) {
        need = true;
      } else {
        float* dst = vals + std::uint64_t(slot) * E;
        for (int d = 0; d < E; ++d) dst[d] = 0.0f;
      }
    } else if (live) {
      csrc[i] = ps;  // carry-over from the previous table (tag 0)
    }
    n_car += (live && ps != kNoSlot);
    const unsigned m = __ballot_sync(0xFFFFFFFFu, need);
    if (m) {
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(n_need, (unsigned long long)__popc(m));
      at = __shfl_sync(0xFFFFFFFFu, at, 0);
      if (need) {
        const unsigned r = __popc(m & ((1u << lane) - 1u));
        need_key[at + r] = key;
        need_slot[at + r] = slot;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) n_car += __shfl_xor_sync(0xFFFFFFFFu, n_car, o);
  if (lane == 0 && n_car) atomicAdd(carried, n_car);
}

// The store rows of the list: a streaming gather (zero-copy over PCIe for a
// host store), ILP independent loads per thread before their stores so a few
// CTAs keep the link busy.
template <int VEC, int ILP>
__global__ void store_gather_kernel(const std::uint64_t* __restrict__ need_key,
                                    const std::uint32_t* __restrict__ need_slot,
                                    const unsigned long long* __restrict__ n_need,
                                    const float* __restrict__ store, float* __restrict__ vals,
                                    int E) {
  pdl_wait();
  using V = typename std::conditional<VEC == 4, float4, float>::type;
  const int tpk = E / VEC;
  const std::uint64_t total = std::uint64_t(*n_need) * tpk;
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  for (std::uint64_t t0 = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t0 < total;
       t0 += stride * ILP) {
    V v[ILP];
    std::uint64_t dst[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const std::uint64_t t = t0 + u * stride;
      if (t < total) {
        const std::uint64_t i = t / tpk;
        const int part = int(t - i * tpk);
        v[u] = reinterpret_cast<const V*>(store + need_key[i] * E)[part];
        dst[u] = std::uint64_t(need_slot[i]) * E + std::uint64_t(part) * VEC;
      }
    }
#pragma unroll
    for (int u = 0; u < ILP; ++u)
      if (t0 + u * stride < total) *reinterpret_cast<V*>(vals + dst[u]) = v[u];
  }
}

// DMA staging (Tier::dma): staged row i -> its table slot, and the reverse
// compaction of evicted rows for the D2H copy. *n_ptr rows, RW floats each.
template <int VEC>
__global__ void staged_rows_to_slots_kernel(const float* __restrict__ staged,
                                            const std::uint32_t* __restrict__ slots,
                                            const unsigned long long* __restrict__ n_ptr,
                                            float* __restrict__ vals, int RW) {
  pdl_wait();
  const int tpk = RW / VEC;
  const std::uint64_t total = std::uint64_t(*n_ptr) * tpk;
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const int part = int(t - i * tpk);
    const float* src = staged + i * RW + part * VEC;
    float* dst = vals + std::uint64_t(slots[i]) * RW + part * VEC;
    if (VEC == 4) {
      st_f4(dst, ld_f4(src));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) dst[q] = src[q];
    }
  }
}
template <int VEC>
__global__ void slots_to_staged_rows_kernel(const std::uint32_t* __restrict__ slots,
                                            const unsigned long long* __restrict__ n_ptr,
                                            const float* __restrict__ vals,
                                            float* __restrict__ staged, int RW) {
  pdl_wait();
  const int tpk = RW / VEC;
  const std::uint64_t total = std::uint64_t(*n_ptr) * tpk;
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const int part = int(t - i * tpk);
    const float* src = vals + std::uint64_t(slots[i]) * RW + part * VEC;
    float* dst = staged + i * RW + part * VEC;
    if (VEC == 4) {
      st_f4(dst, ld_f4(src));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) dst[q] = src[q];
    }
  }
}

// Pipelined build, body half: the rows from the resident tables (the
// previous table's carry-over, or a proxy's), once those batches are done.
template <int VEC>
__global__ void table_carry_kernel(const std::uint32_t* __restrict__ csrc,
                                   const std::uint32_t* __restrict__ wslot,
                                   const std::uint64_t* __restrict__ n_ptr,
                                   const float* __restrict__ prev_vals,
                                   const float* __restrict__ p1_vals,
                                   const float* __restrict__ p2_vals, float* __restrict__ vals,
                                   int E) {
  pdl_wait();
  const int tpk = E / VEC;
  const std::uint64_t n = *n_ptr;
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < n * std::uint64_t(tpk); t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const std::uint32_t ps = csrc[i];
    if (ps == kNoSlot) continue;
    const int part = int(t - i * tpk);
    const std::uint32_t tag = ps & kSrcMask;
    const float* base = tag == kSrcProxy1 ? p1_vals : (tag == kSrcProxy2 ? p2_vals : prev_vals);
    const float* src = base + std::uint64_t(ps & ~kSrcMask) * E + part * VEC;
    float* dst = vals + std::uint64_t(wslot[i]) * E + part * VEC;
    if (VEC == 4) {
      st_f4(dst, ld_f4(src));
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) dst[v] = src[v];
    }
  }
}


// Eviction filter of a table's working set (sorted keys ws, slots wslot):
// rows whose key a newer resident table also holds are skipped (that table
// has the fresher row and writes it back itself later); the rest join a
// warp-contiguous, hence key-ordered, list for the zero-copy writer.
__global__ void table_evict_filter_kernel(const std::uint64_t* __restrict__ ws,
                                          const std::uint32_t* __restrict__ wslot,
                                          const std::uint64_t* __restrict__ n_ptr,
                                          const std::uint64_t* __restrict__ k1,
                                          const std::uint64_t* __restrict__ c1,
                                          const std::uint64_t* __restrict__ k2,
                                          const std::uint64_t* __restrict__ c2,
                                          const std::uint64_t* __restrict__ k3,
                                          const std::uint64_t* __restrict__ c3,
                                          std::uint64_t store_keys,
                                          std::uint64_t* __restrict__ out_key,
                                          std::uint32_t* __restrict__ out_slot,
                                          unsigned long long* __restrict__ n_out,
                                          unsigned long long* __restrict__ total) {
  pdl_wait();
  const std::uint64_t n = *n_ptr;
  const std::uint64_t cap1 = c1 ? *c1 : 0, cap2 = c2 ? *c2 : 0, cap3 = c3 ? *c3 : 0;
  const unsigned lane = threadIdx.x & 31;
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  for (std::uint64_t base = blockIdx.x * std::uint64_t(blockDim.x) + (threadIdx.x & ~31u);
       base < n; base += stride) {
    const std::uint64_t i = base + lane;
    bool keep = false;
    std::uint64_t key = 0;
    if (i < n) {
      key = ws[i];
      std::uint32_t s1 = kNoSlot, s2 = kNoSlot, s3 = kNoSlot;
      if (key < store_keys) probe3_ordered(key, k1, cap1, k2, cap2, k3, cap3, &s1, &s2, &s3);
      keep = key < store_keys && s1 == kNoSlot && s2 == kNoSlot && s3 == kNoSlot;
    }
    const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
    if (m) {
      unsigned long long at = 0;
      if (lane == 0) {
        at = atomicAdd(n_out, (unsigned long long)__popc(m));
        atomicAdd(total, (unsigned long long)__popc(m));
      }
      at = __shfl_sync(0xFFFFFFFFu, at, 0);
      if (keep) {
        const unsigned r = __popc(m & ((1u << lane) - 1u));
        out_key[at + r] = key;
        out_slot[at + r] = wslot[i];
      }
    }
  }
}

// The evicted rows of the list to the value store (zero-copy for a host
// store): ILP independent row loads per thread before their posted stores.
constexpr int kMirrorPageShift = 10;  // 1024 rows per dirty page of a mirrored store
template <int VEC, int ILP>
__global__ void store_scatter_kernel(const std::uint64_t* __restrict__ keys,
                                     const std::uint32_t* __restrict__ slots,
                                     const unsigned long long* __restrict__ n_ptr,
                                     const float* __restrict__ vals, float* __restrict__ store,
                                     int E, std::uint8_t* __restrict__ dirty) {
  pdl_wait();
  using V = typename std::conditional<VEC == 4, float4, float>::type;
  const int tpk = E / VEC;
  const std::uint64_t total = std::uint64_t(*n_ptr) * tpk;
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  for (std::uint64_t t0 = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t0 < total;
       t0 += stride * ILP) {
    V v[ILP];
    std::uint64_t dst[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const std::uint64_t t = t0 + u * stride;
      if (t < total) {
        const std::uint64_t i = t / tpk;
        const int part = int(t - i * tpk);
        v[u] = reinterpret_cast<const V*>(vals + std::uint64_t(slots[i]) * E)[part];
        dst[u] = keys[i] * E + std::uint64_t(part) * VEC;
        // a mirrored host store: the key's page is copied back at the next quiesce
        if (dirty && part == 0) dirty[keys[i] >> kMirrorPageShift] = 1;
      }
    }
#pragma unroll
    for (int u = 0; u < ILP; ++u)
      if (t0 + u * stride < total) *reinterpret_cast<V*>(store + dst[u]) = v[u];
  }
}

// Row fill for the fresh table (hbm_ps.hpp:86-98): carry-over from the
// previous table when the key was resident, else the staged host row
// (HostValue), else the attached value store, else zeros. VEC floats per
// thread, E/VEC threads per key; every thread of a key's group probes (the
// loads coalesce into one transaction).
template <int VEC>
__global__ void table_fill_kernel(
    const std::uint64_t* __restrict__ ws, const std::uint64_t* __restrict__ n_ptr,
    const std::uint64_t* __restrict__ keys, float* __restrict__ vals,
    const std::uint64_t* __restrict__ cap_ptr,
    const std::uint64_t* __restrict__ prev_keys,
    const float* __restrict__ prev_vals,
    const std::uint64_t* __restrict__ prev_cap_ptr,  // null: no previous table
    const std::uint32_t* __restrict__ staged_idx,    // null: no staged rows
    const float* __restrict__ staged_rows,
    const float* __restrict__ store, std::uint64_t store_keys, int E,
    unsigned long long* carried, DevError* err) {
  pdl_wait();
  const int tpk = E / VEC;
  const std::uint64_t n = *n_ptr, cap = *cap_ptr;
  const std::uint64_t pcap = prev_cap_ptr ? *prev_cap_ptr : 0;
  const std::uint64_t total = n * std::uint64_t(tpk);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < total; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const int part = int(t - i * tpk);
    const std::uint64_t key = ws[i];
    const std::uint32_t slot = probe_slot_ordered(keys, cap, key);
    if (slot == kNoSlot) {
      raise_error(err, 2, key);
      continue;
    }
    const float* src = nullptr;
    if (pcap) {
      const std::uint32_t ps = probe_slot_ordered(prev_keys, pcap, key);
      if (ps != kNoSlot) src = prev_vals + std::uint64_t(ps) * E;
    }
    if (carried) {  // warp-aggregated count of carry-over rows
      const unsigned hit = __ballot_sync(__activemask(), src != nullptr && part == 0);
      if (hit && (threadIdx.x & 31) == unsigned(__ffs(__activemask()) - 1))
        atomicAdd(carried, (unsigned long long)__popc(hit));
    }
    if (!src && staged_rows) src = staged_rows + std::uint64_t(staged_idx[i]) * E;
    if (!src && store && key < store_keys) src = store + key * std::uint64_t(E);
    float* dst = vals + std::uint64_t(slot) * E + part * VEC;
    if (VEC == 4) {
      st_f4(dst, src ? ld_f4(src + part * 4) : make_float4(0.f, 0.f, 0.f, 0.f));
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) dst[v] = src ? src[part * VEC + v] : 0.0f;
    }
  }
}

// Pull gather (DeviceTable::get, device_table.hpp:78-85): probe each query
// key, cache its slot for the push, copy the row. Missing key -> error.
template <int VEC>
__global__ void table_gather_kernel(const std::uint64_t* __restrict__ qkeys,
                                    const std::uint64_t* __restrict__ n_ptr,
                                    std::uint64_t n_host, const std::uint64_t* __restrict__ keys,
                                    const float* __restrict__ vals,
                                    const std::uint64_t* __restrict__ cap_ptr,
                                    float* __restrict__ out_rows,
                                    std::uint32_t* __restrict__ out_slots,
                                    int E, int stride, DevError* err) {
  // (E floats of each stride-float table row: the embedding, not its state)
  pdl_wait();
  const int tpk = E / VEC;
  const std::uint64_t n = n_ptr ? *n_ptr : n_host;
  const std::uint64_t cap = *cap_ptr;
  const std::uint64_t total = n * std::uint64_t(tpk);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < total; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const int part = int(t - i * tpk);
    const std::uint64_t key = qkeys[i];
    const std::uint32_t slot = probe_slot_ordered(keys, cap, key);
    if (slot == kNoSlot) {
      raise_error(err, 2, key);
      continue;
    }
    if (out_slots && part == 0) out_slots[i] = slot;
    const float* src = vals + std::uint64_t(slot) * stride + part * VEC;
    float* dst = out_rows + i * E + part * VEC;
    if (VEC == 4) {
      st_f4(dst, ld_f4(src));
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) dst[v] = src[v];
    }
  }
}

// Local lookups (DeviceTable::contains / get, device_table.hpp:76-85) without
// the missing-key error: found[i] = 1 and the key's RW-float row (when rows
// is non-null), else found[i] = 0. One thread per key.
__global__ void table_lookup_kernel(const std::uint64_t* __restrict__ qkeys, std::uint64_t n,
                                    const std::uint64_t* __restrict__ keys,
                                    const float* __restrict__ vals,
                                    const std::uint64_t* __restrict__ cap_ptr, int RW,
                                    std::uint8_t* __restrict__ found, float* __restrict__ rows) {
  pdl_wait();
  const std::uint64_t cap = *cap_ptr;
  for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t key = qkeys[i];
    const std::uint32_t slot = key == kEmptyKey ? kNoSlot : probe_slot_ordered(keys, cap, key);
    found[i] = slot != kNoSlot;
    if (rows)
      for (int d = 0; d < RW; ++d)
        rows[i * RW + d] = slot != kNoSlot ? vals[std::uint64_t(slot) * RW + d] : 0.0f;
  }
}

// Owner apply of one sender's segment (device_table.hpp:88-95): v += d in
// f32, no contraction (or the Adagrad step, Optim). Keys inside one segment
// are unique, so no atomics; segments are launched in canonical sender order
// (hbm_ps.hpp:172-195). slots == null: probe `qkeys` instead of using cached
// slots.
template <int VEC>
__global__ void table_apply_kernel(const std::uint32_t* __restrict__ slots,
                                   const std::uint64_t* __restrict__ qkeys,
                                   const std::uint64_t* __restrict__ tkeys,
                                   const std::uint64_t* __restrict__ cap_ptr,
                                   const float* __restrict__ deltas,
                                   const std::uint64_t* __restrict__ n_ptr,
                                   std::uint64_t n_host, float* __restrict__ vals,
                                   Optim opt, DevError* err) {
  pdl_wait();
  const int E = opt.E;
  const int tpk = E / VEC;
  const std::uint64_t n = n_ptr ? *n_ptr : n_host;
  const std::uint64_t total = n * std::uint64_t(tpk);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < total; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const int part = int(t - i * tpk);
    std::uint32_t slot;
    if (slots) {
      slot = slots[i];
    } else {
      slot = probe_slot_ordered(tkeys, *cap_ptr, qkeys[i]);
      if (slot == kNoSlot) {
        raise_error(err, 2, qkeys[i]);
        continue;
      }
    }
    float* row = vals + std::uint64_t(slot) * opt.RW;
    const float* d = deltas + i * E + part * VEC;
    if (VEC == 4) {
      opt.apply4(row, part * 4, ld_f4(d));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) opt.apply(row, part * VEC + q, d[q]);
    }
  }
}

// Write-back of the batch's rows to the value store (dump_node ->
// collect_updates, hbm_ps.hpp:224-232, mem_ps.hpp:210-245) and/or to a
// dense (keys, rows) dump in working-set (= ascending key) order.
template <int VEC>
__global__ void table_dump_kernel(const std::uint64_t* __restrict__ ws,
                                  const std::uint64_t* __restrict__ n_ptr,
                                  const std::uint64_t* __restrict__ keys,
                                  const float* __restrict__ vals,
                                  const std::uint64_t* __restrict__ cap_ptr,
                                  float* __restrict__ store, std::uint64_t store_keys,
                                  float* __restrict__ out_rows, int E,
                                  DevError* err) {
  pdl_wait();
  const int tpk = E / VEC;
  const std::uint64_t n = *n_ptr, cap = *cap_ptr;
  const std::uint64_t total = n * std::uint64_t(tpk);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < total; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const int part = int(t - i * tpk);
    const std::uint64_t key = ws[i];
    const std::uint32_t slot = probe_slot_ordered(keys, cap, key);
    if (slot == kNoSlot) {
      raise_error(err, 2, key);
      continue;
    }
    const float* src = vals + std::uint64_t(slot) * E + part * VEC;
    if (VEC == 4) {
      const float4 r = ld_f4(src);
      if (store && key < store_keys) st_f4(store + key * E + part * 4, r);
      if (out_rows) st_f4(out_rows + i * E + part * 4, r);
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        if (store && key < store_keys) store[key * E + part * VEC + q] = src[q];
        if (out_rows) out_rows[i * E + part * VEC + q] = src[q];
      }
    }
  }
}

}  // namespace hpsgpu

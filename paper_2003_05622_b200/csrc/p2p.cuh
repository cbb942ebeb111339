// In-kernel NVLink/NVSwitch all-to-all between the ranks of one box.
//
// Every rank exports one HBM window through CUDA IPC (or, for ranks living in
// one process, plain peer pointers):
//   keys   u64 [G][slot]     pull requests from each source rank
//   hdr    u64 [G][2]        per source: {count, source's send offset}
//   deltas f32 [G][slot][E]  pushed deltas, same order as the keys
//   dense  f32 [G][nw]       dense-gradient replicas for the canonical sum
//   flags  u64 [G][kPhases]  arrival flags per source and phase
// plus the requester-side row buffer, written directly by the owners.
//
// A phase is: writer kernel (P2P stores straight into the peers' windows) ->
// its last CTA fences at system scope and raises flags[me][phase] = epoch in
// every peer -> the consumer's wait kernel spins (bounded) until every
// source's flag reached the epoch. Windows are reused every mini-batch; the
// phase order (keys -> rows -> deltas -> dense) guarantees a window is never
// overwritten before its owner consumed it.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "sort.cuh"

namespace hpsgpu {

constexpr int kMaxRanks = 8;
// kPhKeys..kPhDense: the four-phase exchange of the parity API and the sort
// path; kPhX / kPhY: the fused two-phase round of the batch body (below).
enum P2PPhase {
  kPhKeys = 0, kPhRows = 1, kPhDeltas = 2, kPhDense = 3, kPhX = 4, kPhY = 5, kPhases = 6
};

struct PeerWindows {
  std::uint64_t* keys[kMaxRanks];    // peer's keys window base
  std::uint32_t* uids[kMaxRanks];    // requester-side uid of each requested key
  std::uint64_t* hdr[kMaxRanks];     // peer's header base
  float* deltas[kMaxRanks];          // peer's delta window base
  float* dense[kMaxRanks];           // peer's dense window base
  float* rows[kMaxRanks];            // peer's requester row buffer
  std::uint64_t* flags[kMaxRanks];   // peer's flag array
  int cta_sys_fence;                 // 1: every CTA fences at system scope (HPS_CTA_FENCE=sys)
};

// Both parity copies of every rank's windows plus the device-resident round
// counter: kernels pick the parity from the counter, so a captured CUDA graph
// stays valid across replays (nothing round-dependent is baked into it).
struct P2PCtx {
  PeerWindows par[2];
  const unsigned long long* epoch;
  __device__ __forceinline__ std::uint64_t round() const { return *epoch; }
  __device__ __forceinline__ const PeerWindows& cur(std::uint64_t e) const { return par[e & 1]; }
};

__global__ void epoch_inc_kernel(unsigned long long* epoch) {
  pdl_wait(); *epoch += 1; }

__device__ __forceinline__ void st_release_sys(std::uint64_t* p, std::uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ std::uint64_t ld_acquire_sys(const std::uint64_t* p) {
  std::uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Called by every CTA after its P2P stores; the last CTA to finish raises
// this rank's flag for `phase` in every peer. After the CTA barrier, thread
// 0's acq_rel add on the done counter releases the CTA's stores at GPU scope
// and, in the last CTA, acquires every earlier CTA's (the adds form one
// release sequence); its st.release.sys flag then publishes all of them to
// the peers. A system fence in every CTA (HPS_CTA_FENCE=sys, the earlier
// scheme) costs ≈ 6 µs more per phase (tools/p2p_phase_probe.cu: 3.2 MB at
// the G = 2 interleave, 22.2 -> 16.4 µs per round).
__device__ __forceinline__ void signal_peers(const PeerWindows& pw, int G, int me, int phase,
                                             std::uint64_t epoch, unsigned* done_ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (pw.cta_sys_fence) __threadfence_system();
    const unsigned prev = atom_add_acq_rel_gpu(done_ctr, 1u);
    if (prev == gridDim.x * gridDim.y - 1) {
      *done_ctr = 0;
      if (pw.cta_sys_fence) __threadfence_system();
      for (int p = 0; p < G; ++p) st_release_sys(pw.flags[p] + me * kPhases + phase, epoch);
    }
  }
}

// Waits until every source raised `phase` to the current round in this
// rank's flags: threads < G poll one source each (bounded: a dead peer
// raises an error instead of hanging), then the whole CTA proceeds. Every
// thread of the block must call it.
__device__ __forceinline__ void wait_sources(const P2PCtx& ctx, int G, int me, int phase,
                                             DevError* err) {
  if (threadIdx.x < unsigned(G)) {
    const std::uint64_t epoch = ctx.round();
    const std::uint64_t* f = ctx.par[0].flags[me] + threadIdx.x * kPhases + phase;
    long long spins = 0;
    while (ld_acquire_sys(f) < epoch) {
      if (++spins > (1ll << 27)) {  // ~10 s: a peer died; fail instead of hanging
        raise_error(err, 10 /*HPS_ERR_NCCL*/, std::uint64_t(threadIdx.x));
        break;
      }
      __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void p2p_wait_kernel(P2PCtx ctx, int G, int me, int phase, DevError* err) {
  pdl_wait();
  wait_sources(ctx, G, me, phase, err);
}

// Owner ranks of the sorted unique keys: orank[u] = number of earlier unique
// keys with the same owner (key % G), i.e. the key's index in its owner's
// request region; otot[o] = keys per owner. One decoupled look-back pass
// (G <= 8 counters per tile). Thread 0 of tile 0 also opens the exchange
// round (device round counter) and clears the segment queues of the sparse
// reduce, saving two graph nodes.
constexpr int kRankThreads = 256;
constexpr int kRankItems = 8;
constexpr int kRankTile = kRankThreads * kRankItems;

__global__ void __launch_bounds__(kRankThreads)
    owner_rank_kernel(const std::uint64_t* __restrict__ ukeys,
                      const std::uint64_t* __restrict__ u_ptr, int G, LookBack lb,
                      std::uint32_t* __restrict__ orank, std::uint64_t* __restrict__ otot,
                      unsigned long long* epoch, unsigned long long* clear2) {
  pdl_wait();
  __shared__ std::uint32_t wcnt[kRankThreads / 32][kMaxRanks];
  __shared__ std::uint32_t base[kMaxRanks];
  __shared__ std::uint64_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(lb.ticket, 1ull) - lb.base;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < kMaxRanks) wcnt[warp][lane] = 0;
  __syncthreads();
  const std::uint64_t tile = s_tile;
  const std::uint64_t U = *u_ptr;
  if (tile == 0 && threadIdx.x == 0) {
    *epoch += 1;
    clear2[0] = 0;
    clear2[1] = 0;
  }
  const std::uint64_t b0 = tile * kRankTile;
  if (b0 >= U && !(tile == 0)) return;
  const unsigned lt = lanemask_lt();
  const std::uint64_t wb = b0 + std::uint64_t(warp) * (kRankTile / (kRankThreads / 32));
  std::uint32_t r[kRankItems], dg[kRankItems];
#pragma unroll
  for (int it = 0; it < kRankItems; ++it) {
    const std::uint64_t idx = wb + std::uint64_t(it) * 32 + lane;
    const bool valid = idx < U;
    const std::uint32_t d = valid ? std::uint32_t(ukeys[idx] % std::uint64_t(G)) : kMaxRanks;
    dg[it] = d;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    const std::uint32_t prior = valid ? wcnt[warp][d] : 0u;
    r[it] = prior + unsigned(__popc(peers & lt));
    __syncwarp();
    if (valid && lane == unsigned(__ffs(peers) - 1)) wcnt[warp][d] = prior + unsigned(__popc(peers));
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < unsigned(G)) {
    const int d = threadIdx.x;
    std::uint32_t run = 0;
    for (int w = 0; w < kRankThreads / 32; ++w) {
      const std::uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    std::uint64_t* my = lb.status + tile * kMaxRanks + d;
    std::uint64_t excl = 0;
    const std::uint32_t ep = lb.epoch();
    if (tile == 0) {
      st_status(my, status_word(ep, kFlagInc, run));
    } else {
      st_status(my, status_word(ep, kFlagAgg, run));
      excl = look_back(lb, ep, tile, kMaxRanks, d);
      st_status(my, status_word(ep, kFlagInc, excl + run));
    }
    base[d] = std::uint32_t(excl);
    if (b0 + kRankTile >= U) otot[d] = excl + run;  // the last tile knows the totals
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kRankItems; ++it) {
    const std::uint64_t idx = wb + std::uint64_t(it) * 32 + lane;
    if (idx < U) orank[idx] = base[dg[it]] + wcnt[warp][dg[it]] + r[it];
  }
}

// Requester -> owners: every unique key u goes to its owner's keys window,
// region `me`, at its owner rank, with u (the requester's row index).
// Thread o < G of block 0 writes the per-owner request counts.
__global__ void p2p_send_keys_kernel(P2PCtx ctx, int G, int me, std::uint64_t slot,
                                     const std::uint64_t* __restrict__ ukeys,
                                     const std::uint64_t* __restrict__ u_ptr,
                                     const std::uint32_t* __restrict__ orank,
                                     const std::uint64_t* __restrict__ otot,
                                     unsigned* done_ctr) {
  pdl_wait();
  const std::uint64_t epoch = ctx.round();
  const PeerWindows& pw = ctx.cur(epoch);
  const std::uint64_t U = *u_ptr;
  if (blockIdx.x == 0 && threadIdx.x < unsigned(G)) {
    const int o = threadIdx.x;
    pw.hdr[o][me * 2] = U ? otot[o] : 0;
  }
  for (std::uint64_t u = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; u < U;
       u += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t k = ukeys[u];
    const int o = int(k % std::uint64_t(G));
    const std::uint64_t at = me * slot + orank[u];
    pw.keys[o][at] = k;
    pw.uids[o][at] = std::uint32_t(u);
  }
  signal_peers(pw, G, me, kPhKeys, epoch, done_ctr);
}

// Owner: for every source s and request i (G <= 8 segments, decoded from the
// headers): probe, cache the slot, store the row straight into requester s's
// row buffer at its send position. VEC floats per thread.
template <int VEC>
__global__ void p2p_serve_rows_kernel(P2PCtx ctx, int G, int me, std::uint64_t slot,
                                      const std::uint64_t* __restrict__ tkeys,
                                      const float* __restrict__ tvals,
                                      const std::uint64_t* __restrict__ cap_ptr,
                                      std::uint32_t* __restrict__ rslots, int E, int stride,
                                      unsigned* done_ctr, unsigned long long* served,
                                      DevError* err, int wait_phase, int sig_phase) {
  pdl_wait();
  if (wait_phase >= 0) wait_sources(ctx, G, me, wait_phase, err);  // the requests arrived
  const std::uint64_t epoch = ctx.round();
  const PeerWindows& pw = ctx.cur(epoch);
  const std::uint64_t* my_keys = pw.keys[me];
  const std::uint32_t* my_uids = pw.uids[me];
  const std::uint64_t* my_hdr = pw.hdr[me];
  const int tpk = E / VEC;
  const std::uint64_t cap = *cap_ptr;
  std::uint64_t cnt[kMaxRanks], base[kMaxRanks];
  std::uint64_t total = 0;
  for (int s = 0; s < G; ++s) {
    cnt[s] = my_hdr[s * 2];
    base[s] = total;
    total += cnt[s];
  }
  if (served && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(served, total);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < total * tpk; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t r = t / tpk;
    const int part = int(t - r * tpk);
    int s = 0;
    while (s + 1 < G && r >= base[s + 1]) ++s;
    const std::uint64_t i = r - base[s];
    const std::uint64_t key = my_keys[s * slot + i];
    const std::uint32_t sl = probe_slot_ordered(tkeys, cap, key);
    if (sl == kNoSlot) {
      raise_error(err, 2, key);
      continue;
    }
    if (part == 0) rslots[s * slot + i] = sl;
    const float* src = tvals + std::uint64_t(sl) * stride + part * VEC;  // the embedding
    float* dst = pw.rows[s] + std::uint64_t(my_uids[s * slot + i]) * E + part * VEC;
    if (VEC == 4) {
      st_f4(dst, ld_f4(src));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) dst[q] = src[q];
    }
  }
  signal_peers(pw, G, me, sig_phase, epoch, done_ctr);
}

// Requester -> owners: delta rows (send order) into the owner's deltas
// window, region `me`, at the request's index.
template <int VEC>
__global__ void p2p_send_deltas_kernel(P2PCtx ctx, int G, int me, std::uint64_t slot,
                                       const std::uint64_t* __restrict__ ukeys,
                                       const std::uint64_t* __restrict__ u_ptr,
                                       const std::uint32_t* __restrict__ orank,
                                       const float* __restrict__ deltas, int E,
                                       unsigned* done_ctr) {
  pdl_wait();
  const std::uint64_t epoch = ctx.round();
  const PeerWindows& pw = ctx.cur(epoch);
  const int tpk = E / VEC;
  const std::uint64_t U = *u_ptr;
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t < U * tpk;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t u = t / tpk;
    const int part = int(t - u * tpk);
    const int o = int(ukeys[u] % std::uint64_t(G));
    const float* src = deltas + u * E + part * VEC;
    float* dst = pw.deltas[o] + (me * slot + orank[u]) * E + part * VEC;
    if (VEC == 4) {
      st_f4(dst, ld_f4(src));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) dst[q] = src[q];
    }
  }
  signal_peers(pw, G, me, kPhDeltas, epoch, done_ctr);
}

// Owner apply of one source's deltas; sources are applied in canonical
// sender order (keys shared between sources would race inside one grid, so
// the host enqueues one small grid per source, in order).
template <int VEC>
__global__ void p2p_apply_kernel(P2PCtx ctx, int me, int s, std::uint64_t slot,
                                 const std::uint32_t* __restrict__ rslots,
                                 float* __restrict__ tvals, Optim opt, int G, int wait_phase,
                                 DevError* err, int cnt_field) {
  pdl_wait();
  if (wait_phase >= 0) wait_sources(ctx, G, me, wait_phase, err);  // the deltas arrived
  const PeerWindows& pw = ctx.cur(ctx.round());
  const std::uint64_t* my_hdr = pw.hdr[me];
  const float* my_deltas = pw.deltas[me];
  const int E = opt.E;
  const int tpk = E / VEC;
  const std::uint64_t n = my_hdr[s * 2 + cnt_field];
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t < n * tpk;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t i = t / tpk;
    const int part = int(t - i * tpk);
    float* row = tvals + std::uint64_t(rslots[s * slot + i]) * opt.RW;
    const float* d = my_deltas + (s * slot + i) * E + part * VEC;
    if (VEC == 4) {
      opt.apply4(row, part * 4, ld_f4(d));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) opt.apply(row, part * VEC + q, d[q]);
    }
  }
}

// Wait for every source's dense replica, then the canonical f64 sum, /G
// and the SGD update (hbm_ps.hpp:258-277, 249-256, model.hpp:205-212) in the
// same launch. One CTA.
__global__ void p2p_dense_update_kernel(P2PCtx ctx, int G, int me, int nodes, int devices,
                                        std::uint64_t nw, float* __restrict__ w, float lr,
                                        int apply, float* __restrict__ sum_out, DevError* err,
                                        int wait_phase) {
  pdl_wait();
  __shared__ int ok;
  const std::uint64_t epoch = ctx.round();
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  if (threadIdx.x < unsigned(G) && wait_phase >= 0) {
    const std::uint64_t* f = ctx.par[0].flags[me] + threadIdx.x * kPhases + wait_phase;
    long long spins = 0;
    while (ld_acquire_sys(f) < epoch) {
      if (++spins > (1ll << 27)) {
        raise_error(err, 10, std::uint64_t(threadIdx.x));
        ok = 0;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (!ok) return;
  const float* bufs = ctx.cur(epoch).dense[me];
  for (std::uint64_t i = threadIdx.x; i < nw; i += blockDim.x) {
    double acc = 0.0;
    for (int nn = 0; nn < nodes; ++nn)
      for (int d = 0; d < devices; ++d)
        acc = __dadd_rn(acc, double(bufs[std::uint64_t(d * nodes + nn) * nw + i]));
    const float s = __double2float_rn(acc);
    if (sum_out) sum_out[i] = s;
    if (apply) {
      const float g = __fdiv_rn(s, float(nodes * devices));
      const float nwv = __fsub_rn(w[i], __fmul_rn(lr, g));
      if (!isfinite(nwv)) raise_error(err, 5, i);
      w[i] = nwv;
    }
  }
}

// Dense replica all-gather: this rank's gradient into every peer's dense
// window, region `me`.
__global__ void p2p_send_dense_kernel(P2PCtx ctx, int G, int me, std::uint64_t nw,
                                      const float* __restrict__ grad, unsigned* done_ctr) {
  pdl_wait();
  const std::uint64_t epoch = ctx.round();
  const PeerWindows& pw = ctx.cur(epoch);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t < nw * G;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    const int p = int(t / nw);
    const std::uint64_t i = t - std::uint64_t(p) * nw;
    pw.dense[p][me * nw + i] = grad[i];
  }
  signal_peers(pw, G, me, kPhDense, epoch, done_ctr);
}

// ---- the fused round of the batch body (two phases per mini-batch) -------
//
// Round r of a batch carries, in ONE signalled phase X from every rank to
// every owner: the sparse deltas of mini-batch j (in the owner's request
// order of j, counted in hdr[.][2s+1]), the dense replica of j, and the keys
// of mini-batch j+1 (hdr[.][2s]). Each owner then waits X, applies the
// senders' deltas in canonical order (p2p_apply_kernel, the rows cached when
// it served j), does the canonical dense sum + update, and only then serves
// j+1's rows (phase Y) — so j+1 reads every row after j's apply, the
// reference's read-after-apply order (oracle.hpp:85-112), with two lockstep
// points per mini-batch instead of four (keys, rows, deltas, dense). Windows
// alternate parity by round, and every round but a batch's last ends in Y,
// so no rank is ever more than one round ahead of a peer.
template <int VEC>
__global__ void p2p_send_x_kernel(P2PCtx ctx, int G, int me, std::uint64_t slot, int E,
                                  const std::uint64_t* __restrict__ dkeys,
                                  const std::uint64_t* __restrict__ du_ptr,
                                  const std::uint32_t* __restrict__ dorank,
                                  const std::uint64_t* __restrict__ dotot,
                                  const float* __restrict__ deltas, std::uint64_t nw,
                                  const float* __restrict__ grad,
                                  const std::uint64_t* __restrict__ nkeys,
                                  const std::uint64_t* __restrict__ nu_ptr,
                                  const std::uint32_t* __restrict__ norank,
                                  const std::uint64_t* __restrict__ notot, unsigned* done_ctr) {
  pdl_wait();
  const std::uint64_t epoch = ctx.round();
  const PeerWindows& pw = ctx.cur(epoch);
  const std::uint64_t DU = deltas ? *du_ptr : 0, NU = nkeys ? *nu_ptr : 0;
  if (blockIdx.x == 0 && threadIdx.x < unsigned(G)) {
    const int o = threadIdx.x;
    pw.hdr[o][me * 2] = NU ? notot[o] : 0;      // keys of j+1 (served in Y)
    pw.hdr[o][me * 2 + 1] = DU ? dotot[o] : 0;  // deltas of j (applied after X)
  }
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  const std::uint64_t t0 = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
  const int tpk = E / VEC;
  for (std::uint64_t t = t0; t < DU * tpk; t += stride) {  // deltas -> owners' windows
    const std::uint64_t u = t / tpk;
    const int part = int(t - u * tpk);
    const int o = int(dkeys[u] % std::uint64_t(G));
    const float* src = deltas + u * E + part * VEC;
    float* dst = pw.deltas[o] + (me * slot + dorank[u]) * E + part * VEC;
    if (VEC == 4) {
      st_f4(dst, ld_f4(src));
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) dst[q] = src[q];
    }
  }
  if (grad)  // dense replica -> every peer (all-gather)
    for (std::uint64_t t = t0; t < nw * G; t += stride) {
      const int p = int(t / nw);
      const std::uint64_t i = t - std::uint64_t(p) * nw;
      pw.dense[p][me * nw + i] = grad[i];
    }
  for (std::uint64_t u = t0; u < NU; u += stride) {  // next keys -> owners
    const std::uint64_t k = nkeys[u];
    const int o = int(k % std::uint64_t(G));
    const std::uint64_t at = me * slot + norank[u];
    pw.keys[o][at] = k;
    pw.uids[o][at] = std::uint32_t(u);
  }
  signal_peers(pw, G, me, kPhX, epoch, done_ctr);
}

}  // namespace hpsgpu

namespace hpsgpu {
// The dense replicas this rank received in the current round's parity.
__device__ __forceinline__ const float* dense_window(const P2PCtx& ctx, int me) {
  return ctx.cur(ctx.round()).dense[me];
}
}  // namespace hpsgpu

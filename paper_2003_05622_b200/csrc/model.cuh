// CTR model math of one mini-batch shard on the GPU (model.hpp:57-230).
//
// Numerics follow the reference exactly: parameters/gradients f32, every
// intermediate in f64 with explicit _rn intrinsics (no FMA contraction, IEEE
// division), sums in the reference's order:
//   * embed_sum: features in example order (model.hpp:84-95);
//   * each pre-activation: bias then inputs in index order (model.hpp:65-71);
//   * dprev[i]: outputs in index order (model.hpp:167-172);
//   * dense grads: examples in shard order (model.hpp:161-175) — one thread
//     per weight walks the examples sequentially;
//   * sparse grads: per key, examples in shard order (model.hpp:182-187) —
//     the CSR segment of a key lists its occurrences in example order
//     because the radix sort is stable.
// sigmoid uses CUDA's double exp (<= 1 ulp, glibc's is correctly rounded in
// practice); the parity tests show the f32 results agree bit-for-bit.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hpsgpu {

constexpr int kMaxLayers = 8;
constexpr int kMaxHidden = 64;  // per-layer width supported by this kernel

struct ModelDims {
  int E, L, nw;
  int hw, dw;  // per-example record widths of H (inputs) and DL (deltas)
  int maxw;
  int dims[kMaxLayers];
  int ins[kMaxLayers];
  int offs[kMaxLayers];
  int hoff[kMaxLayers];
  int doff[kMaxLayers];
};

// Shard-local example k of mini-batch shard s is batch example s + k*GJ
// (sharding.hpp:36-40).
struct ShardMap {
  std::uint64_t first;   // s
  std::uint64_t stride;  // G*J
  std::uint64_t count;   // n
};

// Forward + per-example backward. LPE lanes per example (power of two
// <= 32); each example's scratch lives in shared memory. Writes the H and DL
// records (for the dense-gradient reduction), DX = dL/dx (for the sparse
// segment reduction) and accumulates the log loss (model.hpp:232-242).
template <int LPE>
__global__ void __launch_bounds__(128)
    fwd_bwd_kernel(ModelDims md, ShardMap sm, const float* __restrict__ dense,
                   const std::uint32_t* __restrict__ occ_off,
                   const std::uint32_t* __restrict__ occ_row,  // row of each occurrence
                   const float* __restrict__ rows,
                   const std::uint8_t* __restrict__ labels,
                   double* __restrict__ H, double* __restrict__ DL,
                   double* __restrict__ DX, double* __restrict__ loss,
                   DevError* err) {
  extern __shared__ double smem[];
  constexpr int kEPB = 128 / LPE;  // examples per block
  float* W = reinterpret_cast<float*>(smem);
  const int wfl = (md.nw + 1) & ~1;  // keep doubles 8-B aligned
  double* scratch = smem + wfl / 2;
  const int per_ex = md.hw + md.dw + md.maxw;  // h records, z/dl, dprev
  for (int i = threadIdx.x; i < md.nw; i += blockDim.x) W[i] = dense[i];
  __syncthreads();

  const int sub = threadIdx.x % LPE;
  const int slot = threadIdx.x / LPE;
  const unsigned gmask =
      LPE == 32 ? 0xFFFFFFFFu
                : (((1u << LPE) - 1u) << ((threadIdx.x & 31) / LPE * LPE));
  double* hrec = scratch + slot * per_ex;     // [hw]: x | h1 | h2 ...
  double* zrec = hrec + md.hw;                // [dw]: z per layer, then dl
  double* dprev = zrec + md.dw;               // [maxw]
  const int E = md.E;
  double loss_acc = 0.0;

  for (std::uint64_t k0 = std::uint64_t(blockIdx.x) * kEPB; k0 < sm.count;
       k0 += std::uint64_t(gridDim.x) * kEPB) {
    const std::uint64_t k = k0 + slot;
    const bool active = k < sm.count;
    // --- embed_sum: x[d] = sum over features in order
    if (active) {
      const std::uint32_t o0 = occ_off[k], o1 = occ_off[k + 1];
      for (int d = sub; d < E; d += LPE) {
        double acc = 0.0;
        for (std::uint32_t o = o0; o < o1; ++o)
          acc = __dadd_rn(acc, double(rows[std::uint64_t(occ_row[o]) * E + d]));
        hrec[d] = acc;
      }
    }
    __syncwarp();
    // --- run_stack
    double z_out = 0.0;
    for (int l = 0; l < md.L; ++l) {
      const int out = md.dims[l], in = md.ins[l], off = md.offs[l];
      const double* h = hrec + md.hoff[l];
      double* z = zrec + md.doff[l];
      if (active) {
        for (int o = sub; o < out; o += LPE) {
          double acc = double(W[off + in * out + o]);
          const float* row = W + off + o * in;
          for (int i = 0; i < in; ++i)
            acc = __dadd_rn(acc, __dmul_rn(double(row[i]), h[i]));
          if (!isfinite(acc)) raise_error(err, 5, 0);
          z[o] = acc;
          if (l + 1 < md.L) hrec[md.hoff[l + 1] + o] = acc > 0.0 ? acc : 0.0;
        }
      }
      __syncwarp();
    }
    if (active) z_out = zrec[md.doff[md.L - 1]];
    // --- sigmoid, loss, output delta (model.hpp:157-159)
    if (active) {
      const std::uint64_t ex = sm.first + k * sm.stride;
      const double p = 1.0 / (1.0 + exp(-z_out));
      const double y = double(labels[ex]);
      if (sub == 0) {
        const double pc = fmin(fmax(p, 1e-12), 1.0 - 1e-12);
        loss_acc += labels[ex] ? -log(pc) : -log(1.0 - pc);
      }
      __syncwarp(gmask);
      // the output layer has width 1: its delta overwrites z (z no longer needed)
      if (sub == 0) zrec[md.doff[md.L - 1]] = p - y;
    }
    __syncwarp();
    // --- backprop, layer by layer (model.hpp:161-180). zrec[doff[l]..] holds
    // z of layer l until its delta is written; dl of layer l-1 is derived
    // from dprev gated by z of layer l-1.
    for (int li = md.L - 1; li >= 0; --li) {
      const int out = md.dims[li], in = md.ins[li], off = md.offs[li];
      const double* dl = zrec + md.doff[li];  // deltas of layer li
      if (active) {
        for (int i = sub; i < in; i += LPE) {
          double acc = 0.0;
          for (int o = 0; o < out; ++o)
            acc = __dadd_rn(acc, __dmul_rn(double(W[off + o * in + i]), dl[o]));
          dprev[i] = acc;
        }
      }
      __syncwarp();
      if (active) {
        if (li > 0) {
          double* dlp = zrec + md.doff[li - 1];  // holds z of layer li-1
          for (int i = sub; i < in; i += LPE) {
            const double zz = dlp[i];
            dlp[i] = zz <= 0.0 ? 0.0 : dprev[i];
          }
        } else {
          for (int i = sub; i < in; i += LPE) DX[k * E + i] = dprev[i];
        }
      }
      __syncwarp();
    }
    // --- persist records for the reductions
    if (active) {
      for (int i = sub; i < md.hw; i += LPE) H[k * md.hw + i] = hrec[i];
      for (int i = sub; i < md.dw; i += LPE) DL[k * md.dw + i] = zrec[i];
    }
    __syncwarp();
  }
  if (sub == 0 && loss_acc != 0.0) atomicAdd(loss, loss_acc);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- TMA bulk copy + mbarrier helpers (sm_90+/sm_100a async proxy) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// Dense gradient of the shard: one thread per weight walks the examples in
// order (model.hpp:161-175), then *1/n and the f32 cast (model.hpp:189-193).
// 128 threads = one warp per SM sub-partition, so each weight's f64 chain
// issues at the DADD latency. The per-example H/DL records (contiguous per
// chunk of examples) arrive through a kGradStages-deep ring of TMA bulk
// copies (one elected thread, mbarrier completion), off the consumers' issue
// slots. H/DL are padded by 2 doubles so chunk sizes round up to 16 B.
constexpr int kGradStages = 4;
constexpr int kGradThreads = 128;

inline int grad_chunk(const ModelDims& md) {
  int ch = 64;
  while (ch > 8 && size_t(kGradStages) * ch * (md.hw + md.dw) * 8 + 64 > 200 * 1024) ch >>= 1;
  return ch;
}
inline size_t dense_grad_smem(const ModelDims& md) {
  return size_t(kGradStages) * grad_chunk(md) * (md.hw + md.dw) * sizeof(double) + 64;
}

__global__ void __launch_bounds__(kGradThreads)
    dense_grad_kernel(ModelDims md, std::uint64_t n, int chunk,
                      const double* __restrict__ H, const double* __restrict__ DL,
                      float* __restrict__ grad) {
  extern __shared__ __align__(128) double sm[];
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(sm);  // kGradStages barriers
  double* ring = sm + 8;                                          // 64 B header
  const int hw = md.hw, dw = md.dw;
  const std::size_t stage_elems = std::size_t(chunk) * (hw + dw);
  const int w = blockIdx.x * kGradThreads + threadIdx.x;
  const bool live = w < md.nw;
  int hi = 0, di = 0;
  bool bias = false;
  if (live) {
    int l = md.L - 1;
    while (w < md.offs[l]) --l;
    const int in = md.ins[l], out = md.dims[l], rel = w - md.offs[l];
    bias = rel >= in * out;
    const int o = bias ? rel - in * out : rel / in;
    di = md.doff[l] + o;
    hi = md.hoff[l] + (bias ? 0 : rel % in);
  }
  const std::uint64_t nchunks = (n + chunk - 1) / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGradStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](std::uint64_t c) {  // thread 0 only
    double* sH = ring + (c % kGradStages) * stage_elems;
    double* sD = sH + std::size_t(chunk) * hw;
    const std::uint64_t k0 = c * chunk;
    const unsigned cnt = unsigned(n - k0 < std::uint64_t(chunk) ? n - k0 : chunk);
    const unsigned bh = (cnt * hw * 8u + 15u) & ~15u, bd = (cnt * dw * 8u + 15u) & ~15u;
    std::uint64_t* bar = &full[c % kGradStages];
    mbar_expect_tx(bar, bh + bd);
    bulk_g2s(sH, H + k0 * hw, bh, bar);
    bulk_g2s(sD, DL + k0 * dw, bd, bar);
  };
  if (threadIdx.x == 0)
    for (std::uint64_t c = 0; c < nchunks && c < std::uint64_t(kGradStages); ++c) issue(c);
  double acc = 0.0;
  for (std::uint64_t c = 0; c < nchunks; ++c) {
    mbar_wait(&full[c % kGradStages], unsigned((c / kGradStages) & 1));
    if (live) {
      const double* sH = ring + (c % kGradStages) * stage_elems + hi;
      const double* sD = ring + (c % kGradStages) * stage_elems + std::size_t(chunk) * hw + di;
      const std::uint64_t k0 = c * chunk;
      const int cnt = int(n - k0 < std::uint64_t(chunk) ? n - k0 : chunk);
      if (bias) {
#pragma unroll 8
        for (int k = 0; k < cnt; ++k, sD += dw) acc = __dadd_rn(acc, *sD);
      } else {
#pragma unroll 8
        for (int k = 0; k < cnt; ++k, sD += dw, sH += hw)
          acc = __dadd_rn(acc, __dmul_rn(*sD, *sH));
      }
    }
    __syncthreads();  // every consumer is done with this stage
    if (threadIdx.x == 0 && c + kGradStages < nchunks) issue(c + kGradStages);
  }
  if (live) {
    const double inv_n = n == 0 ? 0.0 : 1.0 / double(n);
    grad[w] = __double2float_rn(__dmul_rn(acc, inv_n));
  }
}

// Sparse gradient segment-reduce + sgd_delta (model.hpp:182-200, 226-230).
// Per unique key u: sum over its occurrences, in example order, of the
// example's dL/dx (the CSR segment [seg[u], seg[u+1]) of the stably sorted
// occurrences; exs[p] = shard example of sorted occurrence p), *1/n, f32,
// then -(lr * g) into the push row of the key (pos[u], its position in the
// owner-partitioned send order; identity when pos is null).
//
// Short segments (<= kLongSeg): LPK lanes per key; each round the group loads
// up to 8 example ids, every lane issues its 8 independent DX loads into
// registers, then adds them in order. Longer segments (hot Zipf keys: up to
// the whole shard) are queued for sparse_delta_long_kernel.
constexpr int kLongSeg = 64;
constexpr int kStageDepth = 8;

__device__ __forceinline__ void write_delta(float* out, std::uint64_t row, int E, int d,
                                            double acc, double inv_n, float lr) {
  const float g = __double2float_rn(__dmul_rn(acc, inv_n));
  out[row * E + d] = -__fmul_rn(lr, g);
}

template <int LPK, int kDPL>
__global__ void __launch_bounds__(256)
    sparse_delta_kernel(int E, float lr, std::uint64_t n,
                        const std::uint64_t* __restrict__ u_ptr,
                        const std::uint32_t* __restrict__ seg,
                        const std::uint32_t* __restrict__ exs,
                        const std::uint32_t* __restrict__ pos,
                        const double* __restrict__ DX, float* __restrict__ out,
                        unsigned long long* __restrict__ pulled,
                        std::uint32_t* __restrict__ long_list,
                        unsigned long long* __restrict__ n_long) {
  const std::uint64_t U = *u_ptr;
  if (pulled && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(pulled, (unsigned long long)U);
  const double inv_n = n == 0 ? 0.0 : 1.0 / double(n);
  const int sub = threadIdx.x % LPK;
  const unsigned lane = threadIdx.x & 31;
  const unsigned gmask =
      LPK == 32 ? 0xFFFFFFFFu : (((1u << LPK) - 1u) << (lane / LPK * LPK));
  constexpr int SD = LPK < kStageDepth ? LPK : kStageDepth;  // ids come from SD lanes
  const std::uint64_t groups = (std::uint64_t(gridDim.x) * blockDim.x) / LPK;
  for (std::uint64_t u = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) / LPK; u < U;
       u += groups) {
    const std::uint32_t p0 = seg[u], p1 = seg[u + 1];
    if (p1 - p0 > std::uint32_t(kLongSeg)) {
      if (sub == 0) long_list[atomicAdd(n_long, 1ull)] = std::uint32_t(u);
      continue;
    }
    double acc[kDPL];
#pragma unroll
    for (int q = 0; q < kDPL; ++q) acc[q] = 0.0;
    for (std::uint32_t c = p0; c < p1; c += SD) {
      const int len = int(p1 - c < std::uint32_t(SD) ? p1 - c : SD);
      const std::uint32_t my_ex = sub < len ? exs[c + sub] : 0u;
      double v[SD][kDPL];
#pragma unroll
      for (int r = 0; r < SD; ++r) {
        const std::uint64_t ex = __shfl_sync(gmask, my_ex, r, LPK);
        const double* row = DX + ex * std::uint64_t(E);
#pragma unroll
        for (int q = 0; q < kDPL; ++q) {
          const int d = sub + q * LPK;
          v[r][q] = (r < len && d < E) ? row[d] : 0.0;
        }
      }
#pragma unroll
      for (int r = 0; r < SD; ++r)
        if (r < len) {
#pragma unroll
          for (int q = 0; q < kDPL; ++q) acc[q] = __dadd_rn(acc[q], v[r][q]);
        }
    }
    const std::uint64_t orow = pos ? pos[u] : u;
#pragma unroll
    for (int q = 0; q < kDPL; ++q) {
      const int d = sub + q * LPK;
      if (d < E) write_delta(out, orow, E, d, acc[q], inv_n, lr);
    }
  }
}

// Long segments: one CTA per key. Warps that own no dimension (and do not
// share sub-partition 0 with warp 0) gather the segment's DX rows into a
// double-buffered shared ring with 16-B cp.async; thread d < E runs the
// sequential f64 sum of dimension d from shared memory, alone on its issue
// slot, so the chain proceeds at the DADD latency.
constexpr int kLongThreads = 256;

inline int long_chunk(int E) {
  int ch = 512;
  while (ch > 32 && size_t(2) * ch * E * 8 > 160 * 1024) ch >>= 1;
  return ch;
}

__global__ void __launch_bounds__(kLongThreads)
    sparse_delta_long_kernel(int E, float lr, std::uint64_t n, int chunk,
                             const std::uint32_t* __restrict__ long_list,
                             const unsigned long long* __restrict__ n_long,
                             const std::uint32_t* __restrict__ seg,
                             const std::uint32_t* __restrict__ exs,
                             const std::uint32_t* __restrict__ pos,
                             const double* __restrict__ DX, float* __restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  const unsigned long long NL = *n_long;
  const double inv_n = n == 0 ? 0.0 : 1.0 / double(n);
  const int warp = threadIdx.x >> 5;
  const int cw = (E + 31) / 32;  // consumer warps 0..cw-1
  // producers: warps >= cw that do not share a sub-partition with a consumer
  const bool producer = warp >= cw && (warp % 4) >= cw;
  int prank = 0, nprod = 0;
  for (int w = 0; w < kLongThreads / 32; ++w) {
    const bool pw = w >= cw && (w % 4) >= cw;
    if (pw) {
      if (w < warp) prank += 32;
      nprod += 32;
    }
  }
  prank += threadIdx.x & 31;
  const bool even = (E & 1) == 0;
  const int pieces_per_row = even ? E / 2 : E;  // 16-B or 8-B pieces
  for (unsigned long long li = blockIdx.x; li < NL; li += gridDim.x) {
    const std::uint32_t u = long_list[li];
    const std::uint32_t p0 = seg[u], p1 = seg[u + 1];
    const std::uint32_t nch = (p1 - p0 + chunk - 1) / chunk;
    auto issue = [&](std::uint32_t c) {
      if (producer && c < nch) {
        double* buf = sm + std::size_t(c & 1) * chunk * E;
        const std::uint32_t b = p0 + c * chunk;
        const int cnt = int(p1 - b < std::uint32_t(chunk) ? p1 - b : chunk);
        for (int t = prank; t < cnt * pieces_per_row; t += nprod) {
          const int r = t / pieces_per_row, q = t - r * pieces_per_row;
          const double* src = DX + std::uint64_t(exs[b + r]) * E;
          if (even) {
            const unsigned s = smem_u32(buf + r * E + 2 * q);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + 2 * q));
          } else {
            cp_async8(buf + r * E + q, src + q);
          }
        }
      }
      cp_async_commit();
    };
    issue(0);
    double acc = 0.0;
    for (std::uint32_t c = 0; c < nch; ++c) {
      issue(c + 1);
      cp_async_wait<1>();
      __syncthreads();
      if (int(threadIdx.x) < E) {
        const double* buf = sm + std::size_t(c & 1) * chunk * E + threadIdx.x;
        const std::uint32_t b = p0 + c * chunk;
        const int cnt = int(p1 - b < std::uint32_t(chunk) ? p1 - b : chunk);
#pragma unroll 8
        for (int r = 0; r < cnt; ++r, buf += E) acc = __dadd_rn(acc, *buf);
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    if (int(threadIdx.x) < E)
      write_delta(out, pos ? pos[u] : u, E, threadIdx.x, acc, inv_n, lr);
    __syncthreads();
  }
}

// Dense sync finalize + update: canonical f64 sum of the G replica buffers
// in node-major/device-major order (hbm_ps.hpp:258-277), sum/float(G)
// (249-256), w -= lr*g with the non-finite check (model.hpp:205-212).
// nodes == 0 marks "already summed" (f32 all-reduce result in bufs[0]).
__global__ void dense_update_kernel(float* __restrict__ w,
                                    const float* __restrict__ bufs,
                                    std::uint64_t len, int nodes, int devices,
                                    float lr, int apply, float* __restrict__ sum_out,
                                    DevError* err) {
  for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       i < len; i += std::uint64_t(gridDim.x) * blockDim.x) {
    float s;
    if (nodes == 0) {
      s = bufs[i];
    } else {
      double acc = 0.0;
      for (int nn = 0; nn < nodes; ++nn)
        for (int d = 0; d < devices; ++d)
          acc = __dadd_rn(acc, double(bufs[std::uint64_t(d * nodes + nn) * len + i]));
      s = __double2float_rn(acc);
    }
    if (sum_out) sum_out[i] = s;
    if (apply) {
      const float g = __fdiv_rn(s, float(nodes == 0 ? devices : nodes * devices));
      const float nw = __fsub_rn(w[i], __fmul_rn(lr, g));
      if (!isfinite(nw)) raise_error(err, 5, i);
      w[i] = nw;
    }
  }
}

}  // namespace hpsgpu

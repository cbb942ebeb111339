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

// Dense gradient of the shard: one thread per weight, examples in order,
// then *1/n and the f32 cast (model.hpp:189-193).
__global__ void dense_grad_kernel(ModelDims md, std::uint64_t n,
                                  const double* __restrict__ H,
                                  const double* __restrict__ DL,
                                  float* __restrict__ grad) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= md.nw) return;
  int l = md.L - 1;
  while (w < md.offs[l]) --l;
  const int in = md.ins[l], out = md.dims[l], rel = w - md.offs[l];
  const bool bias = rel >= in * out;
  const int o = bias ? rel - in * out : rel / in;
  const int i = bias ? 0 : rel % in;
  const double* dl = DL + md.doff[l] + o;
  const double* h = H + md.hoff[l] + i;
  double acc = 0.0;
  if (bias) {
    for (std::uint64_t k = 0; k < n; ++k) acc = __dadd_rn(acc, dl[k * md.dw]);
  } else {
    for (std::uint64_t k = 0; k < n; ++k)
      acc = __dadd_rn(acc, __dmul_rn(dl[k * md.dw], h[k * md.hw]));
  }
  const double inv_n = n == 0 ? 0.0 : 1.0 / double(n);
  grad[w] = __double2float_rn(__dmul_rn(acc, inv_n));
}

// Sparse gradient segment-reduce + sgd_delta (model.hpp:182-200, 226-230):
// thread per (unique key, dim); the key's CSR segment lists its
// occurrences in example order. Writes -(lr * g) into the push buffer row
// of the key (its position in the owner-partitioned send order).
__global__ void sparse_delta_kernel(int E, float lr, std::uint64_t n,
                                    const std::uint64_t* __restrict__ u_ptr,
                                    const std::uint32_t* __restrict__ seg,
                                    const std::uint32_t* __restrict__ sorted_occ,
                                    const std::uint32_t* __restrict__ ex_of_occ,
                                    const std::uint32_t* __restrict__ pos,  // null: identity
                                    const double* __restrict__ DX,
                                    float* __restrict__ out) {
  const std::uint64_t U = *u_ptr;
  const double inv_n = n == 0 ? 0.0 : 1.0 / double(n);
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
       t < U * E; t += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t u = t / E;
    const int d = int(t - u * E);
    double acc = 0.0;
    for (std::uint32_t p = seg[u], pe = seg[u + 1]; p < pe; ++p)
      acc = __dadd_rn(acc, DX[std::uint64_t(ex_of_occ[sorted_occ[p]]) * E + d]);
    const float g = __double2float_rn(__dmul_rn(acc, inv_n));
    const std::uint64_t row = pos ? pos[u] : u;
    out[row * E + d] = -__fmul_rn(lr, g);
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

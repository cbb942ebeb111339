// Wide dense MLP of one mini-batch shard on the 5th-generation tensor cores
// (BASELINE config 4: layers {512, 256, 128, 1}, 173k weights; the reference
// stack is model.hpp:57-202, generic in depth and width).
//
// The narrow configs (every layer <= kMaxHidden) keep fwd_bwd_kernel: f64,
// the reference's exact order, bit-exact. A wide stack does not fit that
// kernel's per-example shared-memory scheme, and its GEMM-shaped work belongs
// on tcgen05: examples are the M dimension of every layer's GEMM,
//   forward   Z_l   = H_{l-1} W_l^T + b_l,  H_l = relu(Z_l)        (M=n, N=out, K=in)
//   backward  dZ_l-1 = (dZ_l W_l) .* [H_{l-1} > 0]                (M=n, N=in,  K=out)
//             [dW_l | db_l] = dZ_l^T [H_{l-1} | 1] / n           (M=out, N=in+1, K=n)
//             dX    = dZ_0 W_0  (f64 out, feeds the sparse segment-reduce)
// with FP32 accumulation in TMEM (kind::tf32) and "3xTF32" operands: each
// fp32 value x is split into hi = tf32_rna(x) and lo = x - hi, and
// hi*hi + hi*lo + lo*hi (three MMAs into one accumulator) recovers ~fp32
// products (plain TF32 keeps 10 mantissa bits; measured on c4 it left
// embedding rows 3.7% off the f64 reference after 8 steps, 3xTF32 ~1e-5).
// Results match the f64 reference to a stated tolerance, not bit for bit
// (tests/test_gpu_wide_mlp.py). The output layer (width 1), the sigmoid /
// loss / output delta and its gradient are CUDA-core kernels.
//
// GEMM kernel (umma_gemm_kernel): one CTA per 128 x BN output tile (and per
// K slice: split-K writes fp32 partials reduced in a fixed order, so results
// are deterministic), 128 threads. K is walked in 32-element stages, double
// buffered: all threads stage A and B (any strides: the loaders transpose on
// the fly) into shared memory in the canonical K-major no-swizzle UMMA layout
// (8-row x 16-byte core matrices; LBO = 128 B between K core matrices, SBO =
// 1024 B between 8-row groups), one elected thread issues 4 tcgen05.mma
// (M=128, N=BN, K=8; 12 with the 3xTF32 split) and commits them to the
// stage's mbarrier, which gates
// the reuse of that buffer. The accumulator (128 lanes x BN fp32 columns of
// TMEM) is drained by tcgen05.ld (32x32b: warp w owns lanes 32w..32w+31, one
// output row per thread) into the fused epilogue.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hpsgpu {

constexpr int kGemmBM = 128;      // UMMA M (cta_group::1)
constexpr int kGemmBK = 32;       // K per stage (4 x UMMA K=8 for tf32)
constexpr int kGemmThreads = 128;

enum GemmEpi : int {
  kEpiStore = 0,     // D = acc (split-K partial slice z at D + z * M * ldd)
  kEpiBiasRelu = 1,  // D = max(acc + bias[n], 0)
  kEpiMask = 2,      // D = mask(m, n) > 0 ? acc : 0
  kEpiF64 = 3,       // Dd = double(acc)
};

struct GemmArgs {
  int M, N, K;
  const float* A;
  std::int64_t a_m, a_k;  // A(m, k) = A[m * a_m + k * a_k]
  const float* B;
  std::int64_t b_n, b_k;  // B(n, k) = B[n * b_n + k * b_k]
  int b_ones_col;         // B(N-1, k) = 1 (bias column of the weight-gradient GEMM)
  int epi;
  float* D;
  std::int64_t ldd;       // D(m, n) = D[m * ldd + n]
  double* Dd;             // kEpiF64 output (ldd too)
  const float* bias;      // kEpiBiasRelu: [N]
  const float* mask;      // kEpiMask: mask(m, n) = mask[m * ldm + n]
  std::int64_t ldm;
  int k_per_split;        // K range of grid.z slice z: [z * k_per_split, ...)
  int split3;             // 1: 3xTF32 (hi/lo operand split), 0: plain TF32
};

// ---- tcgen05 / TMEM primitives (PTX ISA 8.6+, sm_100a) --------------------

__device__ __forceinline__ std::uint32_t smem_u32_addr(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no-swizzle shared-memory matrix descriptor (tcgen05 "version 1").
__device__ __forceinline__ std::uint64_t umma_smem_desc(std::uint32_t saddr, std::uint32_t lbo,
                                                        std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFFu);
  d |= std::uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= std::uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= std::uint64_t(1) << 46;  // descriptor version (Blackwell)
  return d;                     // base offset 0, legacy LBO mode, SWIZZLE_NONE
}

// Instruction descriptor of kind::tf32: D f32, A/B tf32, both K-major.
__host__ __device__ constexpr std::uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                          // c_format F32
         | (2u << 7)                        // a_format TF32
         | (2u << 10)                       // b_format TF32
         | (std::uint32_t(N >> 3) << 17)    // n_dim
         | (std::uint32_t(M >> 4) << 24);   // m_dim
}

__device__ __forceinline__ void umma_tf32(std::uint32_t tmem_d, std::uint64_t adesc,
                                          std::uint64_t bdesc, std::uint32_t idesc,
                                          std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::
                   "r"(smem_u32_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_init1(std::uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32_addr(bar)));
}
__device__ __forceinline__ void mbar_wait_parity(std::uint64_t* bar, std::uint32_t parity) {
  std::uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32_addr(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// 32 lanes x 32 bit x 16 columns: thread t gets lane (base lane + t), columns
// col..col+15 of the TMEM address.
__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, float* v) {
  std::uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// x = hi + lo with hi = x rounded to TF32 (10 mantissa bits, low 13 bits
// zero) and lo = x - hi (exact in fp32; the MMA reads its top 10 bits).
__device__ __forceinline__ float tf32_hi(float x) {
  std::uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void put_split(char* dst, std::size_t lo_off, std::size_t at, float v,
                                          bool split) {
  if (split) {
    const float hi = tf32_hi(v);
    *reinterpret_cast<float*>(dst + at) = hi;
    *reinterpret_cast<float*>(dst + lo_off + at) = __fsub_rn(v, hi);
  } else {
    *reinterpret_cast<float*>(dst + at) = v;
  }
}

__device__ __forceinline__ void cp_async4_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(valid ? 4 : 0));
}

// Issue the cp.async copies of a rows x kGemmBK tile of X(r, k) (r in
// [r0, r0+rows), k in [k0, k0+32), zero outside [0, R) x [0, klim)) into the
// canonical layout at dst: byte (r/8)*1024 + (k/4)*128 + (r%8)*16 + (k%4)*4.
// No registers are held while the copies are in flight. The ones row (the
// bias column of the weight-gradient GEMM) is written directly.
__device__ __forceinline__ void stage_tile_async(float* dst, int rows, const float* X,
                                                 std::int64_t x_r, std::int64_t x_k, int r0,
                                                 int R, int k0, int klim, int ones_row) {
  const int tid = threadIdx.x;
  char* base = reinterpret_cast<char*>(dst);
  if (x_k == 1 && (x_r & 3) == 0 && (reinterpret_cast<std::uintptr_t>(X) & 15) == 0 &&
      (klim & 3) == 0) {
    // K contiguous: one 16-byte copy per core-matrix row; thread -> (row % 8)
    // fastest, then the K chunk
    const int chunks = rows * (kGemmBK / 4);
    for (int c = tid; c < chunks; c += kGemmThreads) {
      const int r8 = c & 7, kc = (c >> 3) & 7, rg = c >> 6;
      const int r = rg * 8 + r8, gr = r0 + r, gk = k0 + kc * 4;
      char* at = base + rg * 1024 + kc * 128 + r8 * 16;
      if (gr == ones_row) {
        *reinterpret_cast<float4*>(at) =
            gk < klim ? make_float4(1.f, 1.f, 1.f, 1.f) : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        const bool ok = gr < R && gk < klim;
        cp_async16_zfill(at, ok ? X + gr * x_r + gk : X, ok);
      }
    }
  } else {
    // general strides (transposed operands): 4-byte copies, row fastest
    const int elems = rows * kGemmBK;
    for (int e = tid; e < elems; e += kGemmThreads) {
      const int r = e % rows, k = e / rows;
      const int gr = r0 + r, gk = k0 + k;
      char* at = base + (r >> 3) * 1024 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
      if (gr == ones_row) {
        *reinterpret_cast<float*>(at) = gk < klim ? 1.f : 0.f;
      } else {
        const bool ok = gr < R && gk < klim;
        cp_async4_zfill(at, ok ? X + gr * x_r + std::int64_t(gk) * x_k : X, ok);
      }
    }
  }
}

// 3xTF32: split a landed stage in place, hi = tf32_rna(x) over x, lo = x - hi
// at + lo_off (same layout). Each thread converts 16-byte chunks.
__device__ __forceinline__ void split_stage(char* base, std::size_t bytes, std::size_t lo_off) {
  for (std::size_t o = std::size_t(threadIdx.x) * 16; o < bytes; o += kGemmThreads * 16) {
    const float4 v = *reinterpret_cast<const float4*>(base + o);
    const float4 hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    *reinterpret_cast<float4*>(base + o) = hi;
    *reinterpret_cast<float4*>(base + lo_off + o) =
        make_float4(__fsub_rn(v.x, hi.x), __fsub_rn(v.y, hi.y), __fsub_rn(v.z, hi.z),
                    __fsub_rn(v.w, hi.w));
  }
}

// Stages in the shared-memory ring of umma_gemm_kernel<BN>: as many as fit in
// ~200 KB, 3..4 (BN <= 128). A stage is the A and B tiles (twice that with the
// split).
__host__ __device__ constexpr int gemm_stages(int bn, bool split) {
  return (200 * 1024) / int(std::size_t(kGemmBM + bn) * kGemmBK * 4 * (split ? 2 : 1)) < 3
             ? 3
             : ((200 * 1024) / int(std::size_t(kGemmBM + bn) * kGemmBK * 4 * (split ? 2 : 1)) > 4
                    ? 4
                    : (200 * 1024) / int(std::size_t(kGemmBM + bn) * kGemmBK * 4 * (split ? 2 : 1)));
}
__host__ __device__ constexpr std::size_t gemm_smem(int bn, bool split) {
  return std::size_t(gemm_stages(bn, split)) * (kGemmBM + bn) * kGemmBK * 4 * (split ? 2 : 1);
}

// D(m, n) = sum_k A(m, k) B(n, k) (+ epilogue), (3x)TF32 -> FP32 on tcgen05.
// grid (ceil(M/128), ceil(N/BN), k slices); dynamic smem gemm_smem(BN, split3).
// K walks a ring of gemm_stages() stages: the copies of stage it + S - 1 are
// issued (cp.async) before stage it is consumed, so global latency overlaps
// the MMAs; a stage's buffer is refilled once the MMAs that read it committed.
template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1) umma_gemm_kernel(GemmArgs g) {
  pdl_wait();
  extern __shared__ __align__(1024) std::uint8_t gsm[];
  const bool split = g.split3 != 0;
  const int S = gemm_stages(BN, split);
  // per stage: A hi, B hi (, A lo, B lo)
  constexpr std::size_t kA = std::size_t(kGemmBM) * kGemmBK * 4, kB = std::size_t(BN) * kGemmBK * 4;
  const std::size_t stage_bytes = (kA + kB) * (split ? 2 : 1);
  const std::size_t lo_off = kA + kB;  // lo parts follow the stage's hi tiles
  __shared__ __align__(8) std::uint64_t bar[4];
  __shared__ std::uint32_t tmem_base_sh;
  constexpr int kCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kGemmBM, n0 = blockIdx.y * BN;
  const int kb = blockIdx.z * g.k_per_split;
  const int ke = min(g.K, kb + g.k_per_split);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32_addr(&tmem_base_sh)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) mbar_init1(&bar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_sh;
  const std::uint32_t idesc = umma_idesc_tf32(kGemmBM, BN);
  const int nk = (ke - kb + kGemmBK - 1) / kGemmBK;
  const int ones_row = g.b_ones_col ? g.N - 1 - n0 : -1;  // tile-local row of the ones column
  const int RB = g.b_ones_col ? g.N - 1 - n0 : g.N - n0;
  const float* Bt = g.B + std::int64_t(n0) * g.b_n;
  auto stage_ptr = [&](int i) { return gsm + std::size_t(i % S) * stage_bytes; };
  auto issue = [&](int i) {  // copies of k-stage i (an empty group past the end)
    if (i < nk) {
      const int k0 = kb + i * kGemmBK;
      std::uint8_t* sp = stage_ptr(i);
      stage_tile_async(reinterpret_cast<float*>(sp), kGemmBM, g.A, g.a_m, g.a_k, m0, g.M, k0, ke,
                       -1);
      stage_tile_async(reinterpret_cast<float*>(sp + kA), BN, Bt, g.b_n, g.b_k, 0, RB, k0, ke,
                       ones_row);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  for (int i = 0; i < S - 1; ++i) issue(i);
  for (int it = 0; it < nk; ++it) {
    // this thread's copies of stage it landed (stages it+1 .. it+S-2 may pend)
    if (S == 4) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    std::uint8_t* sp = stage_ptr(it);
    if (split) split_stage(reinterpret_cast<char*>(sp), kA + kB, lo_off);
    fence_async_smem();  // generic-proxy smem writes -> the tensor core's async proxy
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const std::uint32_t a0 = smem_u32_addr(sp), b0 = smem_u32_addr(sp + kA);
      const std::uint32_t lo = std::uint32_t(lo_off);
#pragma unroll
      for (int kk = 0; kk < kGemmBK / 8; ++kk) {
        const std::uint64_t ah = umma_smem_desc(a0 + kk * 256, 128, 1024);
        const std::uint64_t bh = umma_smem_desc(b0 + kk * 256, 128, 1024);
        if (split) {  // small terms first, then hi*hi
          umma_tf32(tmem, umma_smem_desc(a0 + lo + kk * 256, 128, 1024), bh, idesc,
                    (it | kk) != 0);
          umma_tf32(tmem, ah, umma_smem_desc(b0 + lo + kk * 256, 128, 1024), idesc, 1u);
          umma_tf32(tmem, ah, bh, idesc, 1u);
        } else {
          umma_tf32(tmem, ah, bh, idesc, (it | kk) != 0);
        }
      }
      umma_commit(&bar[it % S]);
    }
    // while stage it's MMAs run: refill the buffer stage it-1 used, once its
    // MMAs committed, with stage it + S - 1 (then convert stage it + 1)
    if (it >= 1) mbar_wait_parity(&bar[(it - 1) % S], std::uint32_t(((it - 1) / S) & 1));
    issue(it + S - 1);
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  if (nk > 0) mbar_wait_parity(&bar[(nk - 1) % S], std::uint32_t(((nk - 1) / S) & 1));
  tc_fence_after();
  // epilogue: TMEM lane = output row; a thread loads its row's 16 columns at a
  // time, the warp transposes them through shared memory (the drained stage
  // ring) and stores / reads row segments: 16 lanes cover one row's 64 bytes
  // (a thread-per-row store would touch 32 rows per instruction)
  float* tile = reinterpret_cast<float*>(gsm) + warp * (32 * 17);
  for (int c = 0; c < BN; c += 16) {
    float v[16];
    if (nk > 0) {
      tmem_ld16(tmem + (std::uint32_t(warp * 32) << 16) + std::uint32_t(c), v);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) tile[lane * 17 + i] = v[i];
    __syncwarp();
    const int col = lane & 15, n = n0 + c + col;
#pragma unroll 4
    for (int q = 0; q < 16; ++q) {
      const int r = 2 * q + (lane >> 4);
      const int m = m0 + warp * 32 + r;
      if (m >= g.M || n >= g.N) continue;
      float x = tile[r * 17 + col];
      switch (g.epi) {
        case kEpiBiasRelu:
          x = __fadd_rn(x, g.bias[n]);
          g.D[std::int64_t(m) * g.ldd + n] = x > 0.f ? x : 0.f;
          break;
        case kEpiMask:
          g.D[std::int64_t(m) * g.ldd + n] = g.mask[std::int64_t(m) * g.ldm + n] > 0.f ? x : 0.f;
          break;
        case kEpiF64:
          g.Dd[std::int64_t(m) * g.ldd + n] = double(x);
          break;
        default:
          g.D[std::int64_t(blockIdx.z) * g.M * g.ldd + std::int64_t(m) * g.ldd + n] = x;
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(kCols));
}

// ---- CUDA-core kernels of the wide path -------------------------------

// X[k][d] = f32(sum over the example's features of row[d]) (embed_sum,
// model.hpp:84-95), accumulated in f64. The wide path is not bit-exact (its
// GEMMs are 3xTF32), so the sum need not follow the feature order: one warp per
// example, lanes over features (independent 16-byte row loads), then a
// shuffle tree over the lanes per dimension — the feature-ordered chain of
// dependent loads cost ~0.2 ms per mini-batch at c4's 150 keys per example.
__global__ void __launch_bounds__(256)
    wide_embed_kernel(ShardMap sm, const std::int64_t* __restrict__ goff,
                      const std::uint32_t* __restrict__ occ_off,
                      const std::uint32_t* __restrict__ occ_row, const float* __restrict__ rows,
                      int rstride, int E, float* __restrict__ X) {
  pdl_wait();
  constexpr int kDims = 16;  // dims per pass (4 float4 per row)
  const int lane = threadIdx.x & 31;
  const std::uint64_t warps = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
  const bool vec = (E % 4 == 0) && (rstride % 4 == 0);
  for (std::uint64_t k = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5;
       k < sm.count; k += warps) {
    std::uint32_t o0, o1;
    if (goff) {
      const std::uint64_t ex = sm.first + k * sm.stride;
      o0 = std::uint32_t(goff[ex]);
      o1 = std::uint32_t(goff[ex + 1]);
    } else {
      o0 = occ_off[k];
      o1 = occ_off[k + 1];
    }
    for (int d0 = 0; d0 < E; d0 += kDims) {
      const int nd = E - d0 < kDims ? E - d0 : kDims;
      double acc[kDims];
#pragma unroll
      for (int i = 0; i < kDims; ++i) acc[i] = 0.0;
      for (std::uint32_t p = o0 + lane; p < o1; p += 32) {
        const float* row = rows + std::uint64_t(occ_row[p]) * rstride + d0;
        if (vec && nd == kDims) {
#pragma unroll
          for (int q = 0; q < kDims / 4; ++q) {
            const float4 v = ld_f4(row + 4 * q);
            acc[4 * q] += double(v.x);
            acc[4 * q + 1] += double(v.y);
            acc[4 * q + 2] += double(v.z);
            acc[4 * q + 3] += double(v.w);
          }
        } else {
#pragma unroll
          for (int i = 0; i < kDims; ++i)
            if (i < nd) acc[i] += double(row[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < kDims; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xFFFFFFFFu, acc[i], o);
      if (lane < nd) {
        double v = acc[0];
#pragma unroll
        for (int i = 1; i < kDims; ++i)
          if (lane == i) v = acc[i];
        X[k * E + d0 + lane] = __double2float_rn(v);
      }
    }
  }
}

// Output layer (width 1) + sigmoid + log loss + output delta, then the last
// hidden layer's masked delta (model.hpp:157-180): one warp per example.
//   z = b + w . h ;  p = sigmoid(z) ;  dz = p - y ;  dZ[i] = h[i] > 0 ? dz * w[i] : 0
__global__ void __launch_bounds__(256)
    wide_head_kernel(ShardMap sm, int K, const float* __restrict__ w, const float* __restrict__ b,
                     const float* __restrict__ H, const std::uint8_t* __restrict__ labels,
                     float* __restrict__ dz_out, float* __restrict__ dZ, double* __restrict__ loss,
                     DevError* err) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const std::uint64_t warps = (std::uint64_t(gridDim.x) * blockDim.x) >> 5;
  double lacc = 0.0;
  for (std::uint64_t k = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5;
       k < sm.count; k += warps) {
    const float* h = H + k * K;
    double part = 0.0;
    for (int i = lane; i < K; i += 32) part = __dadd_rn(part, __dmul_rn(double(w[i]), double(h[i])));
    for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xFFFFFFFFu, part, o));
    const double z = __dadd_rn(double(b[0]), part);
    if (!isfinite(z) && lane == 0) raise_error(err, 5, 0);
    const double p = 1.0 / (1.0 + exp(-z));
    const std::uint8_t y = labels[sm.first + k * sm.stride];
    if (lane == 0) {
      const double pc = fmin(fmax(p, 1e-12), 1.0 - 1e-12);
      lacc += y ? -log(pc) : -log(1.0 - pc);
      dz_out[k] = float(p - double(y));
    }
    const float dz = float(p - double(y));
    for (int i = lane; i < K; i += 32) dZ[k * K + i] = h[i] > 0.f ? __fmul_rn(dz, w[i]) : 0.f;
  }
  if (lane == 0 && lacc != 0.0) atomicAdd(loss, lacc);
}

// Output layer's gradients: g[i] = sum_k dz[k] H[k][i] / n (i < K), bias
// g[K] = sum_k dz[k] / n. One block per column: threads stride the examples,
// then a fixed-order block reduction (deterministic).
__global__ void __launch_bounds__(256)
    wide_head_grad_kernel(std::uint64_t n, int K, const float* __restrict__ dz,
                          const float* __restrict__ H, float* __restrict__ g) {
  pdl_wait();
  __shared__ float part[256];
  const int col = blockIdx.x;
  float acc = 0.f;
  for (std::uint64_t k = threadIdx.x; k < n; k += blockDim.x)
    acc = __fadd_rn(acc, col < K ? __fmul_rn(dz[k], H[k * K + col]) : dz[k]);
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) part[threadIdx.x] = __fadd_rn(part[threadIdx.x], part[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) g[col] = n ? __fdiv_rn(part[0], float(n)) : 0.f;
}

// Split-K reduce of [dW | db] partials P[z][o][i] (i <= in, column `in` is the
// bias) in slice order, / n, into the reference layout W[out][in] then
// bias[out] (types.hpp:41-60).
__global__ void wide_wgrad_reduce_kernel(const float* __restrict__ P, int splits, int out, int in,
                                         std::uint64_t n, float* __restrict__ gW,
                                         float* __restrict__ gb) {
  pdl_wait();
  const int cols = in + 1;
  const std::uint64_t total = std::uint64_t(out) * cols;
  const float inv = n ? 1.0f / float(n) : 0.f;
  (void)inv;
  for (std::uint64_t t = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; t < total;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s = __fadd_rn(s, P[std::uint64_t(z) * total + t]);
    const float v = n ? __fdiv_rn(s, float(n)) : 0.f;
    const int o = int(t / cols), i = int(t - std::uint64_t(o) * cols);
    if (i < in) gW[std::uint64_t(o) * in + i] = v;
    else gb[o] = v;
  }
}

}  // namespace hpsgpu

// Device-side helpers shared by the HBM-PS kernels (sm_100a).
#pragma once

#include <cstdint>

namespace hpsgpu {

constexpr std::uint64_t kEmptyKey = ~std::uint64_t{0};  // device_table.hpp:34
constexpr std::uint32_t kNoSlot = 0xFFFFFFFFu;

// Programmatic dependent launch (sm_90+): kernels are launched with
// programmatic stream serialization, so a kernel may start while its
// predecessor's last blocks finish; every kernel first waits here until the
// predecessor's memory operations are visible (a no-op without such a
// dependency).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

// Device error word: the first failure wins; the host maps it to the
// reference's hps::Error text after the phase completes.
struct DevError {
  int code;            // hps_status
  int pad;
  unsigned long long key;
};

__device__ __forceinline__ void raise_error(DevError* e, int code,
                                            unsigned long long key) {
  if (atomicCAS(&e->code, 0, code) == 0) e->key = key;
}

// splitmix64 finalizer, the table hash (common.hpp:57-62).
__host__ __device__ __forceinline__ std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Capacity rule of DeviceTable (device_table.hpp:38-45).
__host__ __device__ __forceinline__ std::uint64_t table_capacity(
    std::uint64_t n) {
  std::uint64_t want = (n * 4 + 2) / 3;
  if (want < 1) want = 1;
  std::uint64_t p = 1;
  while (p < want) p <<= 1;
  return p;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Streaming 128-bit accesses for row traffic that will not be re-read soon.
__device__ __forceinline__ float4 ld_f4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ void st_f4(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}

// The sparse optimizer applied in place by the owner (push/drain,
// device_table.hpp:88-95). A table row is RW floats: the embedding (E), then
// for Adagrad its accumulator state (E; the reference's SparseParam
// opt_state, types.hpp:30-39, which its SGD never touches). The pushed value
// per dimension is the SGD delta -(lr*g) (model.hpp:226-230: v += d), or for
// Adagrad the gradient g itself (self-pinned extension, BASELINE c3,
// oracle/hps_oracle.c or_adagrad_apply):
//   s' = s + g*g;   v' = v - (lr*g) / (sqrt(s') + eps)      (f32, every op _rn)
// 16-byte global -> shared copy (async proxy), zero-filled when !valid
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(valid ? 16 : 0));
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

struct Optim {
  int kind;  // 0 SGD, 1 Adagrad
  int E;     // embedding width (the pushed value's width)
  int RW;    // row width in the table and the value store
  float lr, eps;
  // the pushed value for gradient g (what the sparse reduce emits)
  __device__ __forceinline__ float push_value(float g) const {
    return kind == 0 ? -__fmul_rn(lr, g) : g;
  }
  // row[d] (and its state) updated with pushed value x
  __device__ __forceinline__ void apply(float* row, int d, float x) const {
    if (kind == 0) {
      row[d] = __fadd_rn(row[d], x);
    } else {
      float* st = row + E;
      const float s = __fadd_rn(st[d], __fmul_rn(x, x));
      st[d] = s;
      row[d] = __fsub_rn(row[d], __fdiv_rn(__fmul_rn(lr, x), __fadd_rn(__fsqrt_rn(s), eps)));
    }
  }
  // four consecutive dimensions d0..d0+3 (16-B aligned)
  __device__ __forceinline__ void apply4(float* row, int d0, float4 x) const {
    float4* v = reinterpret_cast<float4*>(row + d0);
    float4 a = *v;
    if (kind == 0) {
      a.x = __fadd_rn(a.x, x.x);
      a.y = __fadd_rn(a.y, x.y);
      a.z = __fadd_rn(a.z, x.z);
      a.w = __fadd_rn(a.w, x.w);
    } else {
      float4* sp = reinterpret_cast<float4*>(row + E + d0);
      float4 s = *sp;
      s.x = __fadd_rn(s.x, __fmul_rn(x.x, x.x));
      s.y = __fadd_rn(s.y, __fmul_rn(x.y, x.y));
      s.z = __fadd_rn(s.z, __fmul_rn(x.z, x.z));
      s.w = __fadd_rn(s.w, __fmul_rn(x.w, x.w));
      *sp = s;
      a.x = __fsub_rn(a.x, __fdiv_rn(__fmul_rn(lr, x.x), __fadd_rn(__fsqrt_rn(s.x), eps)));
      a.y = __fsub_rn(a.y, __fdiv_rn(__fmul_rn(lr, x.y), __fadd_rn(__fsqrt_rn(s.y), eps)));
      a.z = __fsub_rn(a.z, __fdiv_rn(__fmul_rn(lr, x.z), __fadd_rn(__fsqrt_rn(s.z), eps)));
      a.w = __fsub_rn(a.w, __fdiv_rn(__fmul_rn(lr, x.w), __fadd_rn(__fsqrt_rn(s.w), eps)));
    }
    *v = a;
  }
};

// Linear-probe lookup (device_table.hpp:119-128): slot or kNoSlot. The
// probe window starts at mix64(key) & (cap-1) and stops at the first empty.
__device__ __forceinline__ std::uint32_t probe_slot(
    const std::uint64_t* __restrict__ keys, std::uint64_t cap,
    std::uint64_t key) {
  std::uint64_t idx = mix64(key) & (cap - 1);
  for (std::uint64_t n = 0; n < cap; ++n) {
    const std::uint64_t k = __ldg(keys + idx);
    if (k == key) return std::uint32_t(idx);
    if (k == kEmptyKey) return kNoSlot;
    idx = (idx + 1) & (cap - 1);
  }
  return kNoSlot;
}

// Lookup in a table with the ascending-insert layout (every batch table:
// ordered linear probing, table_insert_ordered): when key k sits at slot p,
// every slot of [home(k), p) held a smaller key when k was placed and still
// does, so the first slot holding a key >= k decides — a miss stops at the
// first larger key instead of the first empty slot (kEmptyKey is the
// largest u64).
__device__ __forceinline__ std::uint32_t probe_slot_ordered(
    const std::uint64_t* __restrict__ keys, std::uint64_t cap, std::uint64_t key) {
  std::uint64_t idx = mix64(key) & (cap - 1);
  for (std::uint64_t n = 0; n < cap; ++n) {
    const std::uint64_t k = __ldg(keys + idx);
    if (k >= key) return k == key ? std::uint32_t(idx) : kNoSlot;
    idx = (idx + 1) & (cap - 1);
  }
  return kNoSlot;
}

// The same lookup in up to three ordered tables at once (a null table or
// cap 0 answers kNoSlot): the three home slots load together, and only the
// runs that continue past their home slot walk on.
__device__ __forceinline__ void probe3_ordered(std::uint64_t key, const std::uint64_t* t0,
                                               std::uint64_t c0, const std::uint64_t* t1,
                                               std::uint64_t c1, const std::uint64_t* t2,
                                               std::uint64_t c2, std::uint32_t* s0,
                                               std::uint32_t* s1, std::uint32_t* s2) {
  const std::uint64_t h = mix64(key);
  const std::uint64_t i0 = h & (c0 - 1), i1 = h & (c1 - 1), i2 = h & (c2 - 1);
  const std::uint64_t k0 = c0 ? __ldg(t0 + i0) : kEmptyKey;
  const std::uint64_t k1 = c1 ? __ldg(t1 + i1) : kEmptyKey;
  const std::uint64_t k2 = c2 ? __ldg(t2 + i2) : kEmptyKey;
  auto finish = [&](const std::uint64_t* t, std::uint64_t c, std::uint64_t i,
                    std::uint64_t k) -> std::uint32_t {
    if (!c) return kNoSlot;
    for (std::uint64_t n = 0; n < c; ++n) {
      if (k >= key) return k == key ? std::uint32_t(i) : kNoSlot;
      i = (i + 1) & (c - 1);
      k = __ldg(t + i);
    }
    return kNoSlot;
  };
  *s0 = finish(t0, c0, i0, k0);
  *s1 = finish(t1, c1, i1, k1);
  *s2 = finish(t2, c2, i2, k2);
}

}  // namespace hpsgpu

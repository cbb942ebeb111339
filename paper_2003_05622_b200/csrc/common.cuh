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

}  // namespace hpsgpu

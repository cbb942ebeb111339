// Microbenchmark of one in-kernel NVLink exchange phase between two GPUs of
// one process (the shape of p2p_serve_rows + signal_peers + p2p_wait in
// csrc/p2p.cuh), to locate the flat per-phase cost DESIGN.md §6 reports.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -o tools/p2p_phase_probe tools/p2p_phase_probe.cu
//   tools/p2p_phase_probe        (needs 2 GPUs with peer access)
//
// Per round, on both GPUs at once: a writer grid of `ctas` x 256 threads
// stores `rows` rows of 64 B into the peer's buffer (16 B per thread, rows at
// a stride of `stride` rows: 1 = contiguous, 2 = the G = 2 interleave), then
// each CTA fences (system scope, or GPU scope for the variant) and counts
// itself done; the last CTA raises the round's flag in the peer. A 1-CTA wait
// kernel spins until the peer's flag arrives. Reported: µs per round.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::printf("cuda %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void writer(float4* peer_rows, unsigned long long rows, int stride, int sys_fence,
                       unsigned* done, unsigned long long* peer_flag, unsigned long long round) {
  const unsigned long long items = rows * 4;  // 4 x 16 B per 64-B row
  for (unsigned long long t = blockIdx.x * 256ull + threadIdx.x; t < items;
       t += 256ull * gridDim.x) {
    const unsigned long long r = t >> 2;
    peer_rows[(r * stride) * 4 + (t & 3)] = make_float4(1.f, 2.f, 3.f, float(round));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // sys_fence bit 0: per-CTA fence at system scope (else GPU scope);
    // bit 1: the last CTA relies on st.release.sys alone (no extra fence)
    if (sys_fence & 1) __threadfence_system(); else __threadfence();
    const unsigned prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {
      *done = 0;
      if (!(sys_fence & 2)) __threadfence_system();
      st_release_sys(peer_flag, round);
    }
  }
}

__global__ void waiter(const unsigned long long* my_flag, unsigned long long round) {
  if (threadIdx.x == 0)
    while (ld_acquire_sys(my_flag) < round) __nanosleep(64);
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { std::printf("needs 2 GPUs\n"); return 0; }
  const unsigned long long max_rows = 1ull << 20;  // 64 MB, stride up to 2
  float4* rows[2];
  unsigned long long* flag[2];
  unsigned* done[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&rows[d], max_rows * 2 * 64));
    CK(cudaMalloc(&flag[d], 8));
    CK(cudaMalloc(&done[d], 4));
    CK(cudaMemset(flag[d], 0, 8));
    CK(cudaMemset(done[d], 0, 4));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  unsigned long long round = 0;
  struct Case { unsigned long long rows; int stride, ctas, sys; };
  const Case cases[] = {
      {0, 1, 1, 1},        {0, 1, 1, 0},        {0, 1, 1, 2},        {0, 1, 592, 1},
      {0, 1, 592, 0},      {0, 1, 592, 2},      {12500, 1, 592, 1},  {50000, 1, 592, 1},
      {50000, 2, 592, 1},  {50000, 2, 592, 0},  {50000, 2, 592, 2},  {50000, 2, 148, 1},
      {50000, 2, 148, 0},  {200000, 2, 592, 1}, {200000, 2, 592, 0}, {800000, 1, 592, 1},
  };
  std::printf("rows,stride,ctas,fence,us_per_round,GBps_per_direction\n");
  for (const Case& c : cases) {
    const int iters = 200;
    // each device's rounds captured into one graph (no host launch cost in
    // the timed region); warm-up pass first, then the timed pass
    for (int w = 0; w < 2; ++w) {
      const unsigned long long r0 = round;
      cudaGraphExec_t ge[2];
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(st[d], cudaStreamCaptureModeThreadLocal));
        for (int i = 1; i <= iters; ++i) {
          writer<<<c.ctas, 256, 0, st[d]>>>(rows[1 - d], c.rows, c.stride, c.sys, done[d],
                                           flag[1 - d], r0 + i);
          waiter<<<1, 32, 0, st[d]>>>(flag[d], r0 + i);
        }
        CK(cudaStreamEndCapture(st[d], &g));
        CK(cudaGraphInstantiate(&ge[d], g, 0));
        CK(cudaGraphDestroy(g));
      }
      round = r0 + iters;
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        CK(cudaGraphLaunch(ge[d], st[d]));
        CK(cudaEventRecord(e1[d], st[d]));
      }
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaStreamSynchronize(st[d]));
        CK(cudaGraphExecDestroy(ge[d]));
      }
    }
    float ms = 0;
    CK(cudaSetDevice(0));
    CK(cudaEventElapsedTime(&ms, e0[0], e1[0]));
    const double us = ms * 1e3 / iters;
    std::printf("%llu,%d,%d,%s,%.2f,%.1f\n", c.rows, c.stride, c.ctas, (c.sys & 1) ? ((c.sys & 2) ? "sys,rel" : "sys") : ((c.sys & 2) ? "gpu,rel" : "gpu"), us,
                c.rows * 64.0 / (us * 1e3));
  }
  return 0;
}

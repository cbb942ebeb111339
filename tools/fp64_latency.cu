// Microbenchmark: dependent-chain latency of DADD / DMUL+DADD / FADD and
// shared-memory-fed DADD chains on the GPU (sizes the floor of the
// sequential-order f64 reductions the reference's numerics require).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dadd(double* out, long long* cyc, int n, double x) {
  double a = x, b = x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void chain_dmuladd(double* out, long long* cyc, int n, double x) {
  double a = x, b = x * 1e-9, c = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, __dmul_rn(b, c));
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void chain_fadd(float* out, long long* cyc, int n, float x) {
  float a = x, b = x * 1e-9f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __fadd_rn(a, b);
  long long t1 = clock64();
  out[0] = a; cyc[0] = t1 - t0;
}
__global__ void chain_smem(double* out, long long* cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i * 1e-3;
  __syncthreads();
  double a = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, s[(i * 7 + threadIdx.x) & 1023]);
  long long t1 = clock64();
  out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int lat_main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 8192); cudaMalloc(&f, 64); cudaMalloc(&c, 8);
  const int n = 1 << 16;
  for (int rep = 0; rep < 2; ++rep) {
    chain_dadd<<<1, 1>>>(d, c, n, 1.0); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DADD chain: %.2f cycles/op\n", double(h) / n);
    chain_dmuladd<<<1, 1>>>(d, c, n, 1.0); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("DMUL->DADD chain (DADD-dependent): %.2f cycles/op\n", double(h) / n);
    chain_fadd<<<1, 1>>>(f, c, n, 1.0f); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("FADD chain: %.2f cycles/op\n", double(h) / n);
    chain_smem<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("LDS-fed DADD chain, 1 warp: %.2f cycles/op\n", double(h) / n);
    chain_smem<<<1, 256>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("LDS-fed DADD chain, 8 warps: %.2f cycles/op\n", double(h) / n);
  }
  return 0;
}
// (appended) DADD throughput: 8 independent chains per thread, full occupancy
__global__ void dadd_tput(double* out, int n) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  const double b = 1e-9;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __dadd_rn(a[j], b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fadd_tput(float* out, int n) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  const float b = 1e-9f;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __fadd_rn(a[j], b);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int tput_main() {
  double* d; float* f;
  cudaMalloc(&d, 148 * 8 * 1024 * 8);
  cudaMalloc(&f, 148 * 8 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    dadd_tput<<<148 * 8, 256>>>(d, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ops = 148.0 * 8 * 256 * n * 8;
    if (rep) printf("DADD throughput: %.2f Tops/s = %.1f lanes/clk/SM @1.965GHz\n", ops / ms / 1e9,
                    ops / (ms * 1e-3) / 148 / 1.965e9);
    cudaEventRecord(a);
    fadd_tput<<<148 * 8, 256>>>(f, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("FADD throughput: %.2f Tops/s = %.1f lanes/clk/SM @1.965GHz\n", ops / ms / 1e9,
                    ops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
int main() { lat_main(); return tput_main(); }

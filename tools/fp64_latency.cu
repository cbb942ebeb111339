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
int main() {
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

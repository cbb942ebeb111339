// Kernel microbenchmarks for the sequential-order f64 reductions at the c2
// mini-batch shape (D=1: n = 4096 examples, 100 keys each, Zipf-like
// segments). Uses the production kernels from the package headers.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -I../include -I../paper_2003_05622_b200/csrc kbench.cu -o kbench
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "model.cuh"

using namespace hpsgpu;

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                   \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

template <class F>
static float time_ms(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  // model {8,16,1} at E=16
  ModelDims md{};
  md.E = 16;
  md.L = 3;
  int dims[3] = {8, 16, 1};
  int off = 0, in = 16, hw = 0, dw = 0;
  for (int l = 0; l < 3; ++l) {
    md.dims[l] = dims[l];
    md.ins[l] = in;
    md.offs[l] = off;
    md.hoff[l] = hw;
    md.doff[l] = dw;
    hw += in;
    dw += dims[l];
    off += (in + 1) * dims[l];
    in = dims[l];
  }
  md.nw = off;
  md.hw = hw;
  md.dw = dw;
  md.maxw = 16;
  const std::uint64_t n = 4096;
  std::mt19937_64 rng(1);
  std::vector<double> hH(n * hw + 2), hD(n * dw + 2), hX(n * 16);
  for (auto& v : hH) v = double(rng() % 1000) / 997.0;
  for (auto& v : hD) v = double(rng() % 1000) / 991.0 - 0.5;
  for (auto& v : hX) v = double(rng() % 1000) / 983.0 - 0.5;
  double *H, *DL, *DX;
  float *grad, *out;
  CK(cudaMalloc(&H, hH.size() * 8));
  CK(cudaMalloc(&DL, hD.size() * 8));
  CK(cudaMalloc(&DX, hX.size() * 8));
  CK(cudaMalloc(&grad, md.nw * 4));
  CK(cudaMemcpy(H, hH.data(), hH.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(DL, hD.data(), hD.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(DX, hX.data(), hX.size() * 8, cudaMemcpyHostToDevice));
  double* part;
  unsigned* done;
  unsigned long long* fb;
  CK(cudaMalloc(&part, md.nw * kDGSlices * 32));
  CK(cudaMalloc(&done, 64 * 4));
  CK(cudaMalloc(&fb, 8));
  CK(cudaMemset(done, 0, 64 * 4));
  CK(cudaMemset(fb, 0, 8));
  float t = time_ms([&] {
    dense_grad_p1_kernel<<<dim3(dense_grad_groups(md), kDGSlices), 32>>>(md, n, H, DL, part);
    dense_grad_p2_kernel<<<dim3(dense_grad_groups(md), kDGSlices), 32>>>(md, n, H, DL, part,
                                                                         done, grad, fb);
  });
  CK(cudaGetLastError());
  printf("dense_grad_kernel n=%llu nw=%d: %.2f us (%.1f cycles/elem @1.965GHz)\n",
         (unsigned long long)n, md.nw, t * 1e3, t * 1e-3 * 1.965e9 / n);

  // long-segment reduce: 16 keys with segments of 4096, 2048, ... examples
  std::vector<std::uint32_t> seg, exs, list;
  seg.push_back(0);
  const int nkeys = 300;
  for (int k = 0; k < nkeys; ++k) {
    const std::uint32_t len = std::max<std::uint32_t>(65, std::uint32_t(4096.0 * 6 / (k + 6)));
    std::vector<std::uint32_t> ex(n);
    for (std::uint32_t i = 0; i < n; ++i) ex[i] = i;
    std::shuffle(ex.begin(), ex.end(), rng);
    std::sort(ex.begin(), ex.begin() + std::min<std::uint32_t>(len, n));
    for (std::uint32_t i = 0; i < std::min<std::uint32_t>(len, n); ++i) exs.push_back(ex[i]);
    seg.push_back(std::uint32_t(exs.size()));
    list.push_back(k);
  }
  std::uint32_t *dseg, *dexs, *dlist, *dbig, *dchunk, *dkd;
  unsigned long long *dnl, *dnb, *dni;
  BigPart* dpart;
  ChunkSum* dct;
  std::vector<std::uint32_t> med, bigl;
  for (int k = 0; k < nkeys; ++k) (seg[k + 1] - seg[k] > std::uint32_t(kBigChunk) ? bigl : med).push_back(k);
  CK(cudaMalloc(&dseg, seg.size() * 4));
  CK(cudaMalloc(&dexs, exs.size() * 4));
  CK(cudaMalloc(&dlist, nkeys * 4));
  CK(cudaMalloc(&dbig, nkeys * 4));
  CK(cudaMalloc(&dchunk, (nkeys + 1) * 4));
  CK(cudaMalloc(&dkd, nkeys * 4));
  CK(cudaMalloc(&dpart, 4096 * kBigThreads * sizeof(BigPart)));
  CK(cudaMalloc(&dct, 4096 * 16 * sizeof(ChunkSum)));
  CK(cudaMalloc(&dnl, 8));
  CK(cudaMalloc(&dnb, 8));
  CK(cudaMalloc(&dni, 8));
  CK(cudaMalloc(&out, nkeys * 16 * 4));
  CK(cudaMemset(dkd, 0, nkeys * 4));
  unsigned long long nm = med.size(), nbg = bigl.size();
  CK(cudaMemcpy(dseg, seg.data(), seg.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dexs, exs.data(), exs.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlist, med.data(), med.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dbig, bigl.data(), bigl.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dnl, &nm, 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dnb, &nbg, 8, cudaMemcpyHostToDevice));
  auto run_long = [&] {
    sparse_delta_long_kernel<<<kSMs * 2, kLongThreads>>>(16, 0.05f, n, dlist, dnl, dseg, dexs,
                                                        nullptr, DX, out, fb);
    big_plan_kernel<<<1, 256>>>(dbig, dnb, dseg, dchunk, dni);
    big_p1_kernel<<<kSMs * 4, kBigThreads>>>(16, dbig, dnb, dchunk, dni, dseg, dexs, DX, dpart, dct);
    big_p2_kernel<<<kSMs * 4, kBigThreads>>>(16, 0.05f, n, dbig, dnb, dchunk, dni, dseg, dexs,
                                            nullptr, DX, dpart, dct, dkd, out, fb);
  };
  {
    const float tm = time_ms([&] {
      sparse_delta_long_kernel<<<kSMs * 2, kLongThreads>>>(16, 0.05f, n, dlist, dnl, dseg, dexs,
                                                          nullptr, DX, out, fb);
    });
    const float tp = time_ms([&] { big_plan_kernel<<<1, 256>>>(dbig, dnb, dseg, dchunk, dni); });
    const float t1 = time_ms([&] {
      big_p1_kernel<<<kSMs * 4, kBigThreads>>>(16, dbig, dnb, dchunk, dni, dseg, dexs, DX, dpart, dct);
    });
    const float t2 = time_ms([&] {
      big_p2_kernel<<<kSMs * 4, kBigThreads>>>(16, 0.05f, n, dbig, dnb, dchunk, dni, dseg, dexs,
                                              nullptr, DX, dpart, dct, dkd, out, fb);
    });
    printf("  medium %.2f us, big plan %.2f us, big p1 %.2f us, big p2 %.2f us\n", tm * 1e3,
           tp * 1e3, t1 * 1e3, t2 * 1e3);
  }
  t = time_ms(run_long);
  CK(cudaGetLastError());
  printf("long-segment reduce (%zu medium + %zu big keys, %zu occurrences, max seg %u): %.2f us\n",
         med.size(), bigl.size(), exs.size(), seg[1] - seg[0], t * 1e3);
  // forward/backward of the shard (embed-sum of 100 rows per example + MLP)
  {
    const std::uint32_t nnz = 100, nrows = 150000;
    std::vector<std::uint32_t> occ_off(n + 1), occ_row(n * nnz);
    for (std::uint64_t i = 0; i <= n; ++i) occ_off[i] = std::uint32_t(i * nnz);
    for (auto& r : occ_row) r = std::uint32_t(rng() % nrows);
    std::vector<float> rows(std::size_t(nrows) * 16), w(md.nw);
    for (auto& v : rows) v = float(rng() % 1000) / 1e4f - 0.05f;
    for (auto& v : w) v = float(rng() % 1000) / 1e4f - 0.05f;
    std::vector<std::uint8_t> lab(n);
    for (auto& v : lab) v = rng() & 1;
    std::uint32_t *doff, *drow;
    float *drows, *dw;
    std::uint8_t* dlab;
    double* dloss;
    DevError* derr;
    CK(cudaMalloc(&doff, occ_off.size() * 4));
    CK(cudaMalloc(&drow, occ_row.size() * 4));
    CK(cudaMalloc(&drows, rows.size() * 4));
    CK(cudaMalloc(&dw, w.size() * 4));
    CK(cudaMalloc(&dlab, n));
    CK(cudaMalloc(&dloss, 8));
    CK(cudaMalloc(&derr, sizeof(DevError)));
    CK(cudaMemset(derr, 0, sizeof(DevError)));
    CK(cudaMemcpy(doff, occ_off.data(), occ_off.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(drow, occ_row.data(), occ_row.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dlab, lab.data(), n, cudaMemcpyHostToDevice));
    const int epb = 128 / 16;
    const size_t smem = size_t((md.nw + 1) & ~1) * 4 + size_t(epb) * (md.hw + md.dw + md.maxw) * 8;
    const ShardMap sm{0, 1, n};
    t = time_ms([&] {
      fwd_bwd_kernel<16><<<std::min<std::uint64_t>((n + epb - 1) / epb, kSMs * 8), 128, smem>>>(
          md, sm, dw, doff, (const std::int64_t*)nullptr, drow, drows, dlab, H, DL, DX, dloss, derr);
    });
    CK(cudaGetLastError());
    printf("fwd_bwd_kernel<16> n=%llu x %u features: %.2f us\n", (unsigned long long)n, nnz,
           t * 1e3);
  }
  unsigned long long hfb = 0;
  CK(cudaMemcpy(&hfb, fb, 8, cudaMemcpyDeviceToHost));
  printf("exact-order fallbacks over all timed launches: %llu\n", hfb);
  return 0;
}

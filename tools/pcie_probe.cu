// Host<->device transfer probe for the e2e design (diagnostic only):
// copy-engine DMA rates (H2D, D2H, both at once) for pinned buffers, and
// host-thread gather / scatter rates of 64-byte rows of a 640 MB store in
// ascending key order (the working-set pattern of the c2 workload).
//   nvcc -O2 -std=c++17 -o /tmp/pcie_probe tools/pcie_probe.cu -lpthread
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t MB = 1 << 20, bytes = 32 * MB;
  void *h1, *h2, *d1, *d2;
  cudaMallocHost(&h1, bytes);
  cudaMallocHost(&h2, bytes);
  cudaMalloc(&d1, bytes);
  cudaMalloc(&d2, bytes);
  std::memset(h1, 1, bytes);
  std::memset(h2, 2, bytes);
  cudaStream_t a, b;
  cudaStreamCreate(&a);
  cudaStreamCreate(&b);
  auto rate = [&](int mode) {
    for (int w = 0; w < 2; ++w) {
      if (mode & 1) cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, a);
      if (mode & 2) cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, b);
      cudaDeviceSynchronize();
    }
    const int it = 10;
    const double t0 = now();
    for (int i = 0; i < it; ++i) {
      if (mode & 1) cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, a);
      if (mode & 2) cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, b);
    }
    cudaDeviceSynchronize();
    return it * bytes / (now() - t0) / 1e9;
  };
  std::printf("DMA H2D %.1f GB/s, D2H %.1f GB/s, both at once %.1f GB/s per direction\n", rate(1),
              rate(2), rate(3));

  // host gather / scatter of 64-B rows (E = 16 floats), key-ordered sample
  const size_t dims = 10000000, E = 16, n = 400000;
  std::vector<float> store(dims * E, 1.0f);
  std::vector<std::uint64_t> keys;
  {
    std::mt19937_64 g(1);
    std::vector<std::uint64_t> all;
    // Zipf-like working set: dense low keys + a sparse tail
    for (std::uint64_t k = 0; k < 150000; ++k) all.push_back(k);
    std::uniform_int_distribution<std::uint64_t> u(150000, dims - 1);
    while (all.size() < n) all.push_back(u(g));
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    keys = all;
  }
  float* stage = static_cast<float*>(h1);
  const unsigned hw = std::thread::hardware_concurrency();
  std::printf("host threads available: %u; rows %zu\n", hw, keys.size());
  for (unsigned T : {1u, 4u, 8u, 16u, 32u}) {
    if (T > hw) break;
    for (int dir = 0; dir < 2; ++dir) {
      auto body = [&](unsigned t) {
        const size_t lo = keys.size() * t / T, hi = keys.size() * (t + 1) / T;
        for (size_t i = lo; i < hi; ++i) {
          float* s = store.data() + keys[i] * E;
          float* d = stage + i * E;
          if (dir == 0) std::memcpy(d, s, E * 4);
          else std::memcpy(s, d, E * 4);
        }
      };
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        const double t0 = now();
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t) th.emplace_back(body, t);
        for (auto& x : th) x.join();
        best = std::min(best, now() - t0);
      }
      std::printf("  %2u threads %s: %.3f ms (%.1f GB/s)\n", T, dir ? "scatter" : "gather ",
                  best * 1e3, keys.size() * E * 4 / best / 1e9);
    }
  }
  return 0;
}

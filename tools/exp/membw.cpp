// host memcpy bandwidth into a pinned 64 MB staging buffer, by thread count
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t total = size_t(4) << 30, chunk = size_t(64) << 20;
  std::vector<char> src(total);
  for (size_t i = 0; i < total; i += 4096) src[i] = char(i);
  char* stage;
  cudaMallocHost(&stage, chunk);
  for (unsigned nt : {1u, 4u, 8u, 16u, 32u}) {
    auto t0 = std::chrono::steady_clock::now();
    for (size_t off = 0; off < total; off += chunk) {
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nt; ++t) {
        const size_t a = chunk * t / nt, b = chunk * (t + 1) / nt;
        th.emplace_back([=, &src] { std::memcpy(stage + a, src.data() + off + a, b - a); });
      }
      for (auto& x : th) x.join();
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %2u: %.1f GB/s\n", nt, total / s / 1e9);
  }
  // DMA of the pinned stage alone
  char* d;
  cudaMalloc(&d, chunk);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 64; ++i) cudaMemcpy(d, stage, chunk, cudaMemcpyHostToDevice);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("pinned H2D: %.1f GB/s\n", 64.0 * chunk / s / 1e9);
  printf("nproc %u\n", std::thread::hardware_concurrency());
}

// Does a random-atomic storm (like K1) slow a concurrent 5.5 MB H2D copy, and vice versa?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void storm(unsigned long long* t, size_t n, int iters, unsigned long long seed) {
  unsigned long long x = seed ^ (blockIdx.x * 1315423911ull + threadIdx.x);
  for (int i = 0; i < iters; ++i) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    atomicCAS(t + (x >> 20) % n, 0ull, x);
  }
}

int main() {
  const size_t bytes = 5'500'000 / 16 * 16;
  const size_t n = (16ull << 30) / 8;  // 16 GB table
  void *h, *d;
  unsigned long long* t;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  cudaMalloc(&t, n * 8);
  cudaMemset(t, 0, n * 8);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a1, b1, a2, b2;
  cudaEventCreate(&a1); cudaEventCreate(&b1); cudaEventCreate(&a2); cudaEventCreate(&b2);
  for (int rep = 0; rep < 2; ++rep) {
    for (int mode = 0; mode < 3; ++mode) {  // 0 copy alone, 1 storm alone, 2 both
      cudaDeviceSynchronize();
      if (mode != 0) { cudaEventRecord(a1, s1); storm<<<592, 256, 0, s1>>>(t, n, 64, rep); cudaEventRecord(b1, s1); }
      if (mode != 1) { cudaEventRecord(a2, s2); cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s2); cudaEventRecord(b2, s2); }
      cudaDeviceSynchronize();
      float m1 = 0, m2 = 0;
      if (mode != 0) cudaEventElapsedTime(&m1, a1, b1);
      if (mode != 1) cudaEventElapsedTime(&m2, a2, b2);
      printf("%-12s storm %8.1f us   copy %8.1f us (%.1f GB/s)\n", mode == 0 ? "copy alone" : mode == 1 ? "storm alone" : "both",
             m1 * 1e3, m2 * 1e3, m2 > 0 ? bytes / (m2 * 1e-3) / 1e9 : 0.0);
    }
  }
  return 0;
}

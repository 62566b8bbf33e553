// H2D speed of a 5.5 MB staging block by allocation kind: cudaHostAlloc (several fresh
// buffers) vs a 2 MB-aligned transparent-huge-page mapping pinned with cudaHostRegister.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sys/mman.h>
#include <cuda_runtime.h>

static float copy_us(void* h, void* d, size_t bytes, cudaStream_t st) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float tot = 0;
  for (int r = 0; r < 13; ++r) {
    cudaEventRecord(a, st);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    cudaEventRecord(b, st);
    cudaStreamSynchronize(st);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 3) tot += ms;
  }
  return tot / 10 * 1e3;
}

int main() {
  const size_t bytes = 5'500'000 / 64 * 64;
  void* d;
  cudaMalloc(&d, bytes);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int k = 0; k < 4; ++k) {
    void* h;
    cudaHostAlloc(&h, bytes, k % 2 ? cudaHostAllocMapped : cudaHostAllocDefault);
    memset(h, 1, bytes);
    float us = copy_us(h, d, bytes, st);
    printf("cudaHostAlloc #%d          %8.1f us  %6.1f GB/s\n", k, us, bytes / (us * 1e-6) / 1e9);
  }
  for (int k = 0; k < 4; ++k) {
    const size_t len = (bytes + (2u << 20) - 1) / (2u << 20) * (2u << 20);
    void* m = mmap(nullptr, len + (2u << 20), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    char* h = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(m) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1));
    int adv = madvise(h, len, MADV_HUGEPAGE);
    memset(h, 1, len);
    cudaError_t e = cudaHostRegister(h, len, cudaHostRegisterDefault);
    float us = copy_us(h, d, bytes, st);
    printf("THP + cudaHostRegister #%d %8.1f us  %6.1f GB/s (madvise %d, register %s)\n", k, us,
           bytes / (us * 1e-6) / 1e9, adv, cudaGetErrorString(e));
  }
  return 0;
}

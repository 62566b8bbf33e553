// Does a host-written (cache-resident) staging block slow the H2D copy down?
// Writes 5.5 MB with normal stores or non-temporal stores right before each copy
// (DMA or pull kernel) and times the copy alone with events (tools/h2d_dirty.cu).
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include <immintrin.h>
#include <thread>
#include <vector>

__global__ void pull(const uint4* __restrict__ src, uint4* dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

static void write_nt(char* dst, const char* src, size_t n) {
  for (size_t i = 0; i < n; i += 32) {
    __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), v);
  }
  _mm_sfence();
}

int main() {
  const size_t bytes = 5'500'000 / 64 * 64;
  char *h, *src;
  void* d;
  cudaHostAlloc(reinterpret_cast<void**>(&h), bytes, cudaHostAllocMapped);
  src = static_cast<char*>(aligned_alloc(64, bytes));
  memset(src, 3, bytes);
  cudaMalloc(&d, bytes);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto par = [&](bool nt) {  // 8 threads write one chunk each (like the server's staging pool)
    std::vector<std::thread> th;
    const size_t c = bytes / 8 / 64 * 64;
    for (int k = 0; k < 8; ++k)
      th.emplace_back([&, k] {
        const size_t o = k * c, n = k == 7 ? bytes - o : c;
        if (nt) write_nt(h + o, src + o, n);
        else memcpy(h + o, src + o, n);
      });
    for (auto& t : th) t.join();
  };
  for (int mode = 0; mode < 5; ++mode) {
    for (int path = 0; path < 2; ++path) {
      float tot = 0;
      for (int r = 0; r < 23; ++r) {
        if (mode == 1) memcpy(h, src, bytes);
        if (mode == 2) write_nt(h, src, bytes);
        if (mode == 3) par(false);
        if (mode == 4) par(true);
        cudaEventRecord(a, st);
        if (path == 0) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
        else pull<<<148, 256, 0, st>>>(reinterpret_cast<const uint4*>(h), static_cast<uint4*>(d), bytes / 16);
        cudaEventRecord(b, st);
        cudaStreamSynchronize(st);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) tot += ms;
      }
      const char* names[] = {"untouched buffer", "written (normal stores)", "written (non-temporal)",
                             "8 threads (normal stores)", "8 threads (non-temporal)"};
      printf("%-28s %-6s %8.1f us  %6.1f GB/s\n", names[mode],
             path == 0 ? "DMA" : "pull", tot / 20 * 1e3, bytes / (tot / 20 * 1e-3) / 1e9);
    }
  }
  return 0;
}

// H2D paths for a ~5 MB staging block on this box: one DMA, chunked DMA, and a pull
// kernel reading mapped pinned memory (tools/h2d_chunks.cu; run under gpurun).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pull(const uint4* __restrict__ src, uint4* dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t bytes = 5'500'000 / 16 * 16;
  void *h, *hm, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&hm, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  memset(h, 1, bytes);
  memset(hm, 1, bytes);
  cudaStream_t st[4];
  for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a, st[0]);
    for (int r = 0; r < 20; ++r) fn();
    cudaEventRecord(b, st[0]);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-34s %8.1f us  %6.1f GB/s\n", name, ms / 20 * 1e3, bytes / (ms / 20 * 1e-3) / 1e9);
  };
  for (int chunks : {1, 2, 4, 8, 16}) {
    char name[64];
    snprintf(name, sizeof(name), "DMA pinned, %d chunk(s)", chunks);
    time(name, [&] {
      size_t c = (bytes / chunks + 15) / 16 * 16;
      for (size_t o = 0; o < bytes; o += c) cudaMemcpyAsync((char*)d + o, (char*)h + o, std::min(c, bytes - o),
                                                             cudaMemcpyHostToDevice, st[0]);
    });
  }
  time("DMA pinned, 4 chunks on 4 streams", [&] {
    size_t c = bytes / 4 / 16 * 16;
    for (int k = 0; k < 4; ++k) {
      size_t o = k * c, n = k == 3 ? bytes - o : c;
      cudaMemcpyAsync((char*)d + o, (char*)h + o, n, cudaMemcpyHostToDevice, st[k]);
    }
    for (int k = 1; k < 4; ++k) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      cudaEventRecord(e, st[k]);
      cudaStreamWaitEvent(st[0], e, 0);
      cudaEventDestroy(e);
    }
  });
  time("DMA mapped-pinned, 1 chunk", [&] { cudaMemcpyAsync(d, hm, bytes, cudaMemcpyHostToDevice, st[0]); });
  for (int blocks : {148, 296, 592}) {
    char name[64];
    snprintf(name, sizeof(name), "pull kernel, %d blocks", blocks);
    time(name, [&] { pull<<<blocks, 256, 0, st[0]>>>((const uint4*)hm, (uint4*)d, bytes / 16); });
  }
  return 0;
}

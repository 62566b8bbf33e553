// chase.cu — random 32-B sector access microbenchmark on B200 (tools/, not product).
// Measures dependent-load latency and random-access throughput over a large
// table, to bound what the draft-index kernels (one random sector per trie step)
// can reach. Usage: chase <table GiB> <span MiB per chain (0 = whole table)>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

struct __align__(32) Slot { unsigned long long next; unsigned long long pad[3]; };

__global__ void init_chain(Slot* s, uint64_t n, uint64_t seed) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    s[i].next = x;  // pseudo-random successor (mod n applied at use)
  }
}

template <int MODE>
__global__ void chase(const Slot* __restrict__ s, uint64_t n, uint64_t span, int steps, unsigned long long* out) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t base = span ? ((tid * 0x9E3779B97F4A7C15ull) % (n / span)) * span : 0;
  uint64_t m = span ? span : n;
  uint64_t cur = (tid * 0xD1B54A32D192ED03ull) % m;
  unsigned long long acc = 0;
  for (int k = 0; k < steps; ++k) {
    unsigned long long v;
    if (MODE == 0) {
      asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(s + base + cur));
    } else {
      unsigned long long a, b, c, d;
      asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(s + base + cur));
      v = a ^ (b & 1);
    }
    acc += v;
    cur = (v + k) % m;
  }
  if (acc == 42) out[0] = acc;
}

int main(int argc, char** argv) {
  double gib = argc > 1 ? atof(argv[1]) : 32.0;
  double span_mib = argc > 2 ? atof(argv[2]) : 0.0;
  int l2fetch = argc > 3 ? atoi(argv[3]) : -1;
  if (l2fetch >= 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, l2fetch);
  size_t limv = 0; cudaDeviceGetLimit(&limv, cudaLimitMaxL2FetchGranularity);
  uint64_t n = (uint64_t)(gib * (1ull << 30)) / sizeof(Slot);
  uint64_t span = (uint64_t)(span_mib * (1ull << 20)) / sizeof(Slot);
  Slot* s; cudaMalloc(&s, n * sizeof(Slot));
  unsigned long long* out; cudaMalloc(&out, 8);
  init_chain<<<148 * 16, 256>>>(s, n, 12345);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  printf("table %.1f GiB, span %.1f MiB, l2 fetch granularity %zu\n", gib, span_mib, limv);
  for (int mode = 0; mode < 2; ++mode) {
    for (int tpb : {32, 128, 512, 1024}) {
      for (int bps : {1, 2}) {
        int blocks = 148 * bps;
        int steps = 200;
        if (mode == 0) chase<0><<<blocks, tpb>>>(s, n, span, 20, out); else chase<1><<<blocks, tpb>>>(s, n, span, 20, out);
        cudaEventRecord(a);
        if (mode == 0) chase<0><<<blocks, tpb>>>(s, n, span, steps, out); else chase<1><<<blocks, tpb>>>(s, n, span, steps, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double threads = (double)blocks * tpb;
        double acc = threads * steps;
        printf("mode %s threads %8.0f  latency/step %7.1f ns  throughput %6.2f G acc/s  (%6.1f GB/s @32B)\n",
               mode ? "v4.u64" : "u64   ", threads, ms * 1e6 / steps, acc / ms / 1e6, acc * 32 / ms / 1e6);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}

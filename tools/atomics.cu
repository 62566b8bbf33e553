// atomics.cu — latency/throughput of the atomics the append kernel uses (tools/, not product).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct __align__(32) Slot { unsigned long long a, b, c, d; };

template <int MODE>
__global__ void chain(Slot* s, uint64_t n, int steps, unsigned long long* out) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t cur = (tid * 0x9E3779B97F4A7C15ull) % n;
  unsigned long long acc = 0;
  for (int k = 0; k < steps; ++k) {
    Slot* p = s + cur;
    unsigned long long v;
    if (MODE == 0) {  // load (cg)
      asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    } else if (MODE == 1) {  // 64-bit CAS (fails: compare value never matches)
      v = atomicCAS(&p->a, 0xFFFFFFFFFFFFFFFFull, 1ull);
    } else if (MODE == 2) {  // 128-bit CAS (fails)
      unsigned long long o0, o1;
      asm volatile("{\n\t.reg .b128 c, w, o;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 w, {%4, %5};\n\t"
                   "atom.global.cas.b128 o, [%6], c, w;\n\tmov.b128 {%0, %1}, o;\n\t}"
                   : "=l"(o0), "=l"(o1) : "l"(~0ull), "l"(~0ull), "l"(1ull), "l"(2ull), "l"(p) : "memory");
      v = o0 ^ o1;
    } else if (MODE == 3) {  // exch 32
      v = atomicExch(reinterpret_cast<unsigned*>(&p->c), (unsigned)k);
    } else {  // add 32 with return
      v = atomicAdd(reinterpret_cast<unsigned*>(&p->d), 1u);
    }
    acc += v;
    cur = (cur * 0x9E3779B97F4A7C15ull + v + k + 1) % n;
  }
  if (acc == 42) out[0] = acc;
}

int main() {
  const char* names[] = {"ld.cg   ", "cas64   ", "cas128  ", "exch32  ", "add32ret"};
  for (double gib : {0.05, 16.0}) {
    uint64_t n = (uint64_t)(gib * (1ull << 30)) / sizeof(Slot);
    Slot* s; cudaMalloc(&s, n * sizeof(Slot)); cudaMemset(s, 0x11, n * sizeof(Slot));
    unsigned long long* out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    printf("table %.2f GiB\n", gib);
    for (int mode = 0; mode < 5; ++mode) {
      for (int threads : {148 * 32, 148 * 256, 148 * 1024}) {
        int tpb = 256, blocks = threads / tpb;
        if (threads < tpb) { tpb = 32; blocks = threads / 32; }
        auto run = [&](int steps) {
          switch (mode) {
            case 0: chain<0><<<blocks, tpb>>>(s, n, steps, out); break;
            case 1: chain<1><<<blocks, tpb>>>(s, n, steps, out); break;
            case 2: chain<2><<<blocks, tpb>>>(s, n, steps, out); break;
            case 3: chain<3><<<blocks, tpb>>>(s, n, steps, out); break;
            default: chain<4><<<blocks, tpb>>>(s, n, steps, out); break;
          }
        };
        run(10);
        cudaEventRecord(e0);
        run(100);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("  %s threads %7d  latency/op %8.1f ns  throughput %7.2f G op/s\n", names[mode], blocks * tpb,
               ms * 1e6 / 100, (double)blocks * tpb * 100 / ms / 1e6);
      }
    }
    cudaFree(s);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

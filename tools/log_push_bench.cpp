// Microbenchmark: per-tick cost of growing 256 per-group history logs by 16 records each
// (the host bookkeeping of one C2 tick) with different containers. Build: g++ -O3.
#include <deque>
#include <vector>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <sys/mman.h>
#include <immintrin.h>
struct LogRec { uint64_t hoff, stored; uint32_t len; int32_t rid; };
template <size_t kChunk, bool kHuge>
struct ChunkLog {
  std::vector<LogRec*> chunks; size_t n = 0;
  void push_back(const LogRec& r) {
    if (n % kChunk == 0) {
      void* p = nullptr;
      size_t bytes = kChunk * sizeof(LogRec);
      if (kHuge) { p = aligned_alloc(2 << 20, (bytes + (2<<20) - 1) / (2<<20) * (2<<20)); madvise(p, bytes, MADV_HUGEPAGE); }
      else p = malloc(bytes);
      chunks.push_back(static_cast<LogRec*>(p));
    }
    chunks.back()[n % kChunk] = r; ++n;
  }
};
// blocks handed out from a free list that was touched beforehand (what a background
// pre-faulting pool provides)
struct PoolLog {
  static constexpr size_t kBlock = 256;
  static std::vector<LogRec*>& pool() { static std::vector<LogRec*> p; return p; }
  static void prefill(size_t blocks) {
    for (size_t i = 0; i < blocks; ++i) {
      auto* b = static_cast<LogRec*>(malloc(kBlock * sizeof(LogRec)));
      for (size_t k = 0; k < kBlock * sizeof(LogRec); k += 4096) reinterpret_cast<char*>(b)[k] = 0;
      reinterpret_cast<char*>(b)[kBlock * sizeof(LogRec) - 1] = 0;
      pool().push_back(b);
    }
  }
  std::vector<LogRec*> blocks; size_t n = 0;
  void push_back(const LogRec& r) {
    if (n % kBlock == 0) { blocks.push_back(pool().back()); pool().pop_back(); }
    blocks.back()[n % kBlock] = r; ++n;
  }
};
// fixed 256-entry blocks from malloc, records written with 8-B non-temporal stores (no
// read-for-ownership of the cold lines)
struct NtLog {
  static constexpr size_t kBlock = 256;
  std::vector<LogRec*> blocks; size_t n = 0;
  void push_back(const LogRec& r) {
    if (n % kBlock == 0) blocks.push_back(static_cast<LogRec*>(aligned_alloc(64, kBlock * sizeof(LogRec))));
    LogRec* d = blocks.back() + n % kBlock;
    const long long* src = reinterpret_cast<const long long*>(&r);
    long long* dst = reinterpret_cast<long long*>(d);
    _mm_stream_si64(dst, src[0]);
    _mm_stream_si64(dst + 1, src[1]);
    _mm_stream_si64(dst + 2, src[2]);
    ++n;
  }
};
template <class L> double bench(const char* name) {
  std::vector<L> logs(256);
  double tot = 0; int T = 2000;
  for (int t = 0; t < T; ++t) {
    auto a = std::chrono::steady_clock::now();
    for (int g = 0; g < 256; ++g)
      for (int r = 0; r < 16; ++r) logs[g].push_back(LogRec{uint64_t(t), uint64_t(t*16), 16u, r});
    auto b = std::chrono::steady_clock::now();
    if (t >= 100) tot += std::chrono::duration<double, std::micro>(b - a).count();
  }
  std::printf("%-28s %.1f us per tick\n", name, tot / (T - 100));
  return tot;
}
int main() {
  bench<std::deque<LogRec>>("deque");
  bench<ChunkLog<4096, false>>("chunk 4096 malloc");
  bench<ChunkLog<65536, false>>("chunk 64K malloc");
  bench<ChunkLog<87381, true>>("chunk 2MB hugepage");
  bench<std::vector<LogRec>>("vector");
  bench<NtLog>("nt stores, 256-entry blocks");
  PoolLog::prefill(2000 * 256 * 16 / PoolLog::kBlock + 512);
  bench<PoolLog>("pre-touched 256-entry blocks");
}

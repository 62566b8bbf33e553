// Peer exchange over NVLink / NVSwitch: the owner routing of draft-server
// traffic (fnv1a64(group) % N, dgds.cpp:10-14) without collectives.
//
// Every rank cudaMallocs one region and maps every peer's region through CUDA
// IPC, so one kernel can store straight into another GPU's HBM. A channel is a
// set of double-buffered slabs [parity][sender][rows][words] plus per-sender
// counts and a monotone sequence flag in each receiver's region:
//
//   send        — k_px_count + k_px_scatter: a two-pass stable partition that
//                 stores each record into its owner's slab (over NVLink) in record
//                 order per owner, every thread fencing its own stores at system
//                 scope; then k_px_publish stores the per-owner counts, fences
//                 once and stores flag = seq in every receiver.
//   k_px_wait   — one thread per sender spins (acquire, bounded) until the
//                 sender's flag reaches seq; the kernels after it read the slab.
//   k_px_signal — after the kernels that wrote replies into peers' slabs,
//                 publishes flag = seq to every peer.
//
// Slab reuse is made safe by the tick structure: a sender only
// rewrites a parity after a round trip that proves the owner finished reading it.
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dgds_b200.h"
#include "kernels.h"

#ifndef DGDS_PX_FENCE
#define DGDS_PX_FENCE 1  // 0: fence.sc.sys, 1: fence.acq_rel.sys, 2: (experiment) no per-thread fence
#endif

namespace {

constexpr int kMaxWorld = 8;
constexpr unsigned kFull = 0xffffffffu;

struct PxPeers {
  char* base[kMaxWorld];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Release-pattern fence (prior stores before later stores, system scope). Lighter than the
// sequentially consistent fence.sc.sys behind __threadfence_system().
__device__ __forceinline__ void fence_release_sys() {
#if DGDS_PX_FENCE == 0
  __threadfence_system();
#else
  asm volatile("fence.acq_rel.sys;" ::: "memory");
#endif
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct SendArgs {
  PxPeers peers;
  int32_t world, rank;
  int64_t n;
  const int32_t* owner;
  const int32_t* rec;
  int32_t words;
  int64_t cap;          // rows per sender in a slab
  uint64_t slab_off;    // byte offset of this parity's slab [world][cap][words] in every region
  uint64_t count_off;   // byte offset of this parity's int32 counts [world]
  uint64_t flag_off;    // byte offset of the channel's u64 flags [world]
  unsigned long long seq;
  int64_t* slot;        // per record: owner * cap + row, or -1 (not routed / overflow)
  int32_t* overflow;    // set to 1 when an owner receives more than cap rows (sticky)
  int32_t* cursor;      // [kMaxWorld] per-owner row cursors (zero between launches)
  int32_t origin_word;  // >= 0: that word of each copied row is set to the record's source index
  unsigned* done;       // finished-block counter (zero between launches)
};

__device__ __forceinline__ int32_t* dst_row(const SendArgs& A, int o, int64_t row) {
  return reinterpret_cast<int32_t*>(A.peers.base[o] + A.slab_off) + (A.rank * A.cap + row) * A.words;
}

// Copies the warp's nrec records (sources rec[w0 + r]) to their destination rows, lanes
// walking the (record, word) pairs linearly so each store instruction covers contiguous words.
// Optionally stamps word `origin_word` of the copy with the record's source index.
__device__ __forceinline__ void warp_copy_rows(const SendArgs& A, int64_t w0, int nrec, int my_owner,
                                               int64_t my_row, int lane) {
  constexpr int kBatch = 24;  // loads in flight per lane before the stores (a warp's 32 rows of <= 24 words: one batch)
  const int W = A.words;
  const int total = nrec * W;
  for (int base = 0; base < total; base += 32 * kBatch) {
    int32_t v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int idx = base + u * 32 + lane;
      v[u] = 0;
      if (idx < total) {
        const int r = idx / W;
        v[u] = A.rec[(w0 + r) * W + (idx - r * W)];
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int idx = base + u * 32 + lane;
      const int r = idx < total ? idx / W : 0;
      const int64_t row = __shfl_sync(kFull, my_row, r);
      const int o = __shfl_sync(kFull, my_owner, r);
      if (idx < total && row >= 0) {
        const int k = idx - r * W;
        dst_row(A, o, row)[k] = k == A.origin_word ? static_cast<int32_t>(w0 + r) : v[u];
      }
    }
  }
}

// Two-pass stable scatter. Block b owns records [b * chunk, (b + 1) * chunk).
// Pass 1: per-block per-owner counts. Pass 2: a block's rows for owner o start after the
// rows of all earlier blocks (record order kept per owner), copied warp-cooperatively.
constexpr int kSendBlock = 256;
constexpr int kMaxSendBlocks = 1024;

__global__ void __launch_bounds__(kSendBlock) k_px_count(SendArgs A, int64_t chunk, int32_t* blk_cnt) {
  __shared__ int cnt[kMaxWorld];
  if (threadIdx.x < kMaxWorld) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * chunk, b1 = min(A.n, b0 + chunk);
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = b0; i0 < b1; i0 += kSendBlock) {
    const int64_t i = i0 + threadIdx.x;
    int o = i < b1 ? A.owner[i] : -1;
    if (o >= A.world) o = -1;
    for (int p = 0; p < A.world; ++p) {
      const unsigned bal = __ballot_sync(kFull, o == p);
      if (lane == 0 && bal) atomicAdd(&cnt[p], __popc(bal));
    }
  }
  __syncthreads();
  if (threadIdx.x < A.world) blk_cnt[blockIdx.x * kMaxWorld + threadIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kSendBlock) k_px_scatter(SendArgs A, int64_t chunk, const int32_t* blk_cnt) {
  __shared__ int64_t base[kMaxWorld];
  __shared__ int wcnt[kSendBlock / 32][kMaxWorld];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {  // exclusive prefix over earlier blocks (and, for block 0, the totals): a block reduction
    __shared__ int64_t part[kSendBlock / 32][2 * kMaxWorld];
    int64_t pre[kMaxWorld], tot[kMaxWorld];
#pragma unroll
    for (int p = 0; p < kMaxWorld; ++p) pre[p] = tot[p] = 0;
    for (unsigned k = threadIdx.x; k < gridDim.x; k += kSendBlock) {
#pragma unroll
      for (int p = 0; p < kMaxWorld; ++p) {
        const int c = p < A.world ? blk_cnt[k * kMaxWorld + p] : 0;
        tot[p] += c;
        if (k < blockIdx.x) pre[p] += c;
      }
    }
#pragma unroll
    for (int p = 0; p < kMaxWorld; ++p) {
      for (int d = 16; d > 0; d >>= 1) {
        pre[p] += __shfl_xor_sync(kFull, pre[p], d);
        tot[p] += __shfl_xor_sync(kFull, tot[p], d);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int p = 0; p < kMaxWorld; ++p) {
        part[wid][p] = pre[p];
        part[wid][kMaxWorld + p] = tot[p];
      }
    }
    __syncthreads();
    if (threadIdx.x < A.world) {
      int64_t b = 0, t = 0;
      for (int w = 0; w < kSendBlock / 32; ++w) {
        b += part[w][threadIdx.x];
        t += part[w][kMaxWorld + threadIdx.x];
      }
      base[threadIdx.x] = b;
      (void)t;
    }
    __syncthreads();
  }
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * chunk, b1 = min(A.n, b0 + chunk);
  for (int64_t i0 = b0; i0 < b1; i0 += kSendBlock) {
    const int64_t i = i0 + threadIdx.x;
    int o = i < b1 ? A.owner[i] : -1;
    if (o >= A.world) o = -1;
    unsigned mine = 0;
    for (int p = 0; p < A.world; ++p) {
      const unsigned bal = __ballot_sync(kFull, o == p);
      if (lane == 0) wcnt[wid][p] = __popc(bal);
      if (o == p) mine = bal;
    }
    __syncthreads();
    int64_t row = -1;
    if (o >= 0) {
      int64_t r = base[o];
      for (int w = 0; w < wid; ++w) r += wcnt[w][o];
      row = r + __popc(mine & ((1u << lane) - 1u));
      if (row >= A.cap) {
        atomicExch(A.overflow, 1);
        row = -1;
      }
    }
    if (A.slot && i < b1) A.slot[i] = row >= 0 ? o * A.cap + row : -1;
    const int64_t w0 = i0 + wid * 32;
    if (w0 < b1) warp_copy_rows(A, w0, b1 - w0 < 32 ? static_cast<int>(b1 - w0) : 32, o, row, lane);
    __syncthreads();
    if (threadIdx.x < A.world) {
      int t = 0;
      for (int w = 0; w < kSendBlock / 32; ++w) t += wcnt[w][threadIdx.x];
      base[threadIdx.x] += t;
    }
    __syncthreads();
  }
  // every thread's own row stores are performed at system scope before the grid completes;
  // these fences overlap across all threads (no hand-off chain)
#if DGDS_PX_FENCE != 2
  fence_release_sys();
#endif
}

// After the scatter kernel (stream order: its stores are complete): one thread stores each
// receiver's count, one system-scope fence, then the flags. A single fence on the critical
// path — per-block fences plus a last-block hand-off cost three sequential ones.
__global__ void k_px_publish(SendArgs A, const int32_t* blk_cnt, int nb) {
  const int lane = threadIdx.x;  // one warp
  int64_t tot[kMaxWorld];
#pragma unroll
  for (int p = 0; p < kMaxWorld; ++p) tot[p] = 0;
  for (int b = lane; b < nb; b += 32) {
#pragma unroll
    for (int p = 0; p < kMaxWorld; ++p) tot[p] += p < A.world ? blk_cnt[b * kMaxWorld + p] : 0;
  }
#pragma unroll
  for (int p = 0; p < kMaxWorld; ++p)
    for (int d = 16; d > 0; d >>= 1) tot[p] += __shfl_xor_sync(kFull, tot[p], d);
  if (lane != 0) return;
  for (int o = 0; o < A.world; ++o)
    *reinterpret_cast<volatile int32_t*>(A.peers.base[o] + A.count_off + 4 * A.rank) =
        static_cast<int32_t>(tot[o] < A.cap ? tot[o] : A.cap);
  fence_release_sys();
  for (int o = 0; o < A.world; ++o)
    st_relaxed_sys(reinterpret_cast<unsigned long long*>(A.peers.base[o] + A.flag_off) + A.rank, A.seq);
}

__global__ void k_px_wait(const unsigned long long* flags, int world, unsigned long long seq, int32_t* status,
                          unsigned long long timeout_ns) {
  const int p = threadIdx.x;
  if (p >= world) return;
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(flags + p) < seq) {
    if (global_ns() - t0 > timeout_ns) {
      atomicExch(status, 1);  // a sender never arrived: the results of this launch are invalid
      return;
    }
    __nanosleep(64);
  }
}

__global__ void k_px_signal(PxPeers peers, int world, int rank, uint64_t flag_off, unsigned long long seq) {
  if (threadIdx.x != 0) return;
  __threadfence_system();  // writes of the preceding kernels (stream order) before the flags
  for (int o = 0; o < world; ++o)
    st_release_sys(reinterpret_cast<unsigned long long*>(peers.base[o] + flag_off) + rank, seq);
}

}  // namespace

struct dgds_px {
  int32_t device = 0, world = 1, rank = 0;
  uint64_t bytes = 0;
  char* local = nullptr;
  PxPeers peers{};
  bool opened[kMaxWorld] = {};
  int32_t* d_cursor = nullptr;  // [2][kMaxWorld]: one set per send kernel kind in flight
  unsigned* d_done = nullptr;   // [2]
  int32_t* d_status = nullptr;
  int32_t* d_blk_cnt = nullptr;  // [2][kMaxSendBlocks][kMaxWorld] per-block owner counts
  uint64_t launches = 0;
  int sms = 148;
  uint64_t timeout_ns = 30ull * 1000 * 1000 * 1000;
  std::mutex mu;
};

namespace {
int px_fail(int code, const std::string& m) { return dgds::set_error(code, m); }
#define PX_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) return px_fail(DGDS_ECUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)
}  // namespace

extern "C" {

int dgds_px_create(int32_t device, int32_t world, int32_t rank, uint64_t region_bytes, dgds_px** out,
                   void* handle_out) {
  if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world || region_bytes == 0)
    return px_fail(DGDS_EINVAL, "bad peer-exchange shape");
  int n = 0;
  PX_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return px_fail(DGDS_EINVAL, "no such CUDA device");
  PX_CUDA(cudaSetDevice(device));
  auto* px = new dgds_px();
  px->device = device;
  px->world = world;
  px->rank = rank;
  px->bytes = region_bytes;
  cudaDeviceGetAttribute(&px->sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaMalloc(&px->local, region_bytes);
  if (e == cudaSuccess) e = cudaMemset(px->local, 0, region_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&px->d_cursor, 2 * kMaxWorld * sizeof(int32_t) + 2 * sizeof(unsigned) + 16);
  if (e == cudaSuccess) {
    px->d_done = reinterpret_cast<unsigned*>(px->d_cursor + 2 * kMaxWorld);
    px->d_status = reinterpret_cast<int32_t*>(px->d_done + 2);
    e = cudaMemset(px->d_cursor, 0, 2 * kMaxWorld * sizeof(int32_t) + 2 * sizeof(unsigned) + 16);
  }
  if (e == cudaSuccess) e = cudaMalloc(&px->d_blk_cnt, 2ull * kMaxSendBlocks * kMaxWorld * sizeof(int32_t));
  if (e == cudaSuccess && handle_out) e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle_out), px->local);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (px->local) cudaFree(px->local);
    if (px->d_cursor) cudaFree(px->d_cursor);
    if (px->d_blk_cnt) cudaFree(px->d_blk_cnt);
    delete px;
    return px_fail(DGDS_ECUDA, std::string("peer region: ") + cudaGetErrorString(e));
  }
  px->peers.base[rank] = px->local;
  *out = px;
  return DGDS_OK;
}

int dgds_px_connect(dgds_px* px, const void* handles) {
  if (!px || !handles) return px_fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(px->mu);
  PX_CUDA(cudaSetDevice(px->device));
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int p = 0; p < px->world; ++p) {
    if (p == px->rank || px->peers.base[p]) continue;
    void* ptr = nullptr;
    PX_CUDA(cudaIpcOpenMemHandle(&ptr, h[p], cudaIpcMemLazyEnablePeerAccess));
    px->peers.base[p] = static_cast<char*>(ptr);
    px->opened[p] = true;
  }
  return DGDS_OK;
}

int dgds_px_connect_local(dgds_px* const* all, int32_t world) {
  if (!all || world < 1 || world > kMaxWorld) return px_fail(DGDS_EINVAL, "bad argument");
  for (int r = 0; r < world; ++r) {
    if (!all[r] || all[r]->world != world || all[r]->rank != r) return px_fail(DGDS_EINVAL, "rank mismatch");
  }
  for (int r = 0; r < world; ++r) {
    PX_CUDA(cudaSetDevice(all[r]->device));
    for (int p = 0; p < world; ++p) {
      if (all[p]->device != all[r]->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(all[p]->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return px_fail(DGDS_ECUDA, std::string("peer access: ") + cudaGetErrorString(e));
      }
      all[r]->peers.base[p] = all[p]->local;
    }
  }
  return DGDS_OK;
}

int dgds_px_region(dgds_px* px, int32_t peer, void** base) {
  if (!px || !base || peer < 0 || peer >= px->world) return px_fail(DGDS_EINVAL, "bad argument");
  if (!px->peers.base[peer]) return px_fail(DGDS_EINVAL, "peer not connected");
  *base = px->peers.base[peer];
  return DGDS_OK;
}

int dgds_px_send(dgds_px* px, int64_t n, const int32_t* d_owner, const int32_t* d_records, int32_t rec_words,
                 int64_t cap, uint64_t slab_off, uint64_t count_off, uint64_t flag_off, uint64_t seq,
                 int32_t stable, int32_t origin_word, int64_t* d_slot, int32_t* d_overflow, void* stream) {
  if (origin_word >= rec_words) return px_fail(DGDS_EINVAL, "origin word outside the record");
  if (!px || n < 0 || rec_words < 1 || cap < 0 || seq == 0 || !d_overflow || (n > 0 && (!d_owner || !d_records)))
    return px_fail(DGDS_EINVAL, "bad send arguments");
  for (int p = 0; p < px->world; ++p)
    if (!px->peers.base[p]) return px_fail(DGDS_EINVAL, "peer not connected");
  const uint64_t slab_bytes = static_cast<uint64_t>(px->world) * cap * rec_words * 4;
  if (slab_off + slab_bytes > px->bytes || count_off + 4ull * px->world > px->bytes ||
      flag_off + 8ull * px->world > px->bytes || (flag_off & 7) || (count_off & 3) || (slab_off & 3))
    return px_fail(DGDS_EINVAL, "channel outside the peer region");
  std::lock_guard<std::mutex> lk(px->mu);
  PX_CUDA(cudaSetDevice(px->device));
  SendArgs A{};
  A.peers = px->peers;
  A.world = px->world;
  A.rank = px->rank;
  A.n = n;
  A.owner = d_owner;
  A.rec = d_records;
  A.words = rec_words;
  A.cap = cap;
  A.slab_off = slab_off;
  A.count_off = count_off;
  A.flag_off = flag_off;
  A.seq = seq;
  A.slot = d_slot;
  A.overflow = d_overflow;
  A.origin_word = origin_word < 0 ? -1 : origin_word;
  const int kind = stable ? 1 : 0;  // separate scratch: a query and an append send may overlap
  A.cursor = px->d_cursor + kind * kMaxWorld;
  A.done = px->d_done + kind;
  auto st = static_cast<cudaStream_t>(stream);
  const int sms = px->sms;
  const int64_t rounds = (n + kSendBlock - 1) / kSendBlock;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(rounds, std::min(4 * sms, kMaxSendBlocks)));
  const int64_t chunk = (rounds + blocks - 1) / blocks * kSendBlock;
  const int64_t nb = std::max<int64_t>(1, (n + chunk - 1) / chunk);
  int32_t* blk = px->d_blk_cnt + kind * kMaxSendBlocks * kMaxWorld;
  k_px_count<<<static_cast<unsigned>(nb), kSendBlock, 0, st>>>(A, chunk, blk);
  k_px_scatter<<<static_cast<unsigned>(nb), kSendBlock, 0, st>>>(A, chunk, blk);
  k_px_publish<<<1, 32, 0, st>>>(A, blk, static_cast<int>(nb));
  ++px->launches;
  PX_CUDA(cudaGetLastError());
  ++px->launches;
  return DGDS_OK;
}

int dgds_px_wait(dgds_px* px, uint64_t flag_off, uint64_t seq, void* stream) {
  if (!px || seq == 0 || (flag_off & 7) || flag_off + 8ull * px->world > px->bytes)
    return px_fail(DGDS_EINVAL, "bad wait arguments");
  std::lock_guard<std::mutex> lk(px->mu);
  PX_CUDA(cudaSetDevice(px->device));
  k_px_wait<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const unsigned long long*>(px->local + flag_off), px->world, seq, px->d_status, px->timeout_ns);
  PX_CUDA(cudaGetLastError());
  ++px->launches;
  return DGDS_OK;
}

int dgds_px_signal(dgds_px* px, uint64_t flag_off, uint64_t seq, void* stream) {
  if (!px || seq == 0 || (flag_off & 7) || flag_off + 8ull * px->world > px->bytes)
    return px_fail(DGDS_EINVAL, "bad signal arguments");
  for (int p = 0; p < px->world; ++p)
    if (!px->peers.base[p]) return px_fail(DGDS_EINVAL, "peer not connected");
  std::lock_guard<std::mutex> lk(px->mu);
  PX_CUDA(cudaSetDevice(px->device));
  k_px_signal<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(px->peers, px->world, px->rank, flag_off, seq);
  PX_CUDA(cudaGetLastError());
  ++px->launches;
  return DGDS_OK;
}

int dgds_px_status(dgds_px* px, int32_t* timed_out, uint64_t* launches) {
  if (!px) return px_fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(px->mu);
  PX_CUDA(cudaSetDevice(px->device));
  if (timed_out) PX_CUDA(cudaMemcpy(timed_out, px->d_status, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (launches) *launches = px->launches;
  return DGDS_OK;
}

int dgds_px_set_timeout(dgds_px* px, uint64_t timeout_ns) {
  if (!px || timeout_ns == 0) return px_fail(DGDS_EINVAL, "bad argument");
  px->timeout_ns = timeout_ns;
  return DGDS_OK;
}

int dgds_px_destroy(dgds_px* px) {
  if (!px) return DGDS_OK;
  cudaSetDevice(px->device);
  cudaDeviceSynchronize();
  for (int p = 0; p < px->world; ++p)
    if (px->opened[p]) cudaIpcCloseMemHandle(px->peers.base[p]);
  cudaFree(px->local);
  cudaFree(px->d_cursor);
  cudaFree(px->d_blk_cnt);
  delete px;
  return DGDS_OK;
}

}  // extern "C"

// Peer exchange over NVLink / NVSwitch: the owner routing of draft-server
// traffic (fnv1a64(group) % N, dgds.cpp:10-14) without collectives.
//
// Every rank cudaMallocs one region and maps every peer's region through CUDA
// IPC, so one kernel can store straight into another GPU's HBM. A channel is a
// set of double-buffered slabs [parity][sender][rows][words] plus per-sender
// counts and a monotone sequence flag in each receiver's region:
//
//   k_px_send   — scatters records into slab rows of their owners (the owner's
//                 region, over NVLink) and, in its last block, publishes the
//                 per-owner counts followed by flag = seq with a system-scope
//                 release. Slot allocation is warp-aggregated atomics
//                 (unordered; queries) or a one-block stable partition (appends,
//                 whose per-stream order matters).
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
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/dgds_b200.h"
#include "kernels.h"

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
  unsigned* done;       // finished-block counter (zero between launches)
};

__device__ __forceinline__ int32_t* dst_row(const SendArgs& A, int o, int64_t row) {
  return reinterpret_cast<int32_t*>(A.peers.base[o] + A.slab_off) + (A.rank * A.cap + row) * A.words;
}

// Last block: publish counts, then the flag, to every receiver; reset the cursors.
__device__ void publish(const SendArgs& A) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this block's stores (observed through the barrier) before the count
    last = atomicAdd(A.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence_system();
  for (int o = 0; o < A.world; ++o) {
    const int32_t c = *reinterpret_cast<volatile int32_t*>(A.cursor + o);
    *reinterpret_cast<volatile int32_t*>(A.peers.base[o] + A.count_off + 4 * A.rank) =
        static_cast<int32_t>(c < A.cap ? c : A.cap);
  }
  __threadfence_system();
  for (int o = 0; o < A.world; ++o)
    st_release_sys(reinterpret_cast<unsigned long long*>(A.peers.base[o] + A.flag_off) + A.rank, A.seq);
  for (int o = 0; o < A.world; ++o) A.cursor[o] = 0;
  *A.done = 0;
}

// Unordered: each warp takes 32 records, allocates rows per owner with one atomic per
// (warp, owner), then copies the rows cooperatively (lanes = words, coalesced stores).
__global__ void __launch_bounds__(256) k_px_send_atomic(SendArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t w0 = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < A.n;
       w0 += warps * 32) {
    const int64_t i = w0 + lane;
    int o = i < A.n ? A.owner[i] : -1;
    if (o >= A.world) o = -1;
    const unsigned grp = __match_any_sync(kFull, o);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (o >= 0 && lane == leader) base = atomicAdd(A.cursor + o, __popc(grp));
    base = __shfl_sync(kFull, base, leader);
    int64_t row = o >= 0 ? base + __popc(grp & ((1u << lane) - 1u)) : -1;
    if (row >= A.cap) {
      atomicExch(A.overflow, 1);
      row = -1;
    }
    if (i < A.n) A.slot[i] = row >= 0 ? o * A.cap + row : -1;
    const int nrec = A.n - w0 < 32 ? static_cast<int>(A.n - w0) : 32;
    for (int r = 0; r < nrec; ++r) {
      const int64_t rr = __shfl_sync(kFull, row, r);
      const int oo = __shfl_sync(kFull, o, r);
      if (rr < 0) continue;
      const int32_t* src = A.rec + (w0 + r) * A.words;
      int32_t* dst = dst_row(A, oo, rr);
      for (int k = lane; k < A.words; k += 32) dst[k] = src[k];
    }
  }
  publish(A);
}

// Stable (one block): chunk by chunk, rows are assigned in record order per owner.
__global__ void __launch_bounds__(1024) k_px_send_stable(SendArgs A) {
  __shared__ int wcnt[32][kMaxWorld];
  __shared__ int base[kMaxWorld];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x < kMaxWorld) base[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < A.n; c0 += blockDim.x) {
    const int64_t i = c0 + threadIdx.x;
    int o = i < A.n ? A.owner[i] : -1;
    if (o >= A.world) o = -1;
    unsigned mine = 0;
    for (int p = 0; p < A.world; ++p) {
      const unsigned b = __ballot_sync(kFull, o == p);
      if (lane == 0) wcnt[wid][p] = __popc(b);
      if (o == p) mine = b;
    }
    __syncthreads();
    int64_t row = -1;
    if (o >= 0) {
      int r = base[o];
      for (int w = 0; w < wid; ++w) r += wcnt[w][o];
      row = r + __popc(mine & ((1u << lane) - 1u));
      if (row >= A.cap) {
        atomicExch(A.overflow, 1);
        row = -1;
      }
    }
    if (i < A.n) A.slot[i] = row >= 0 ? o * A.cap + row : -1;
    if (row >= 0) {
      const int32_t* src = A.rec + i * A.words;
      int32_t* dst = dst_row(A, o, row);
      for (int k = 0; k < A.words; ++k) dst[k] = src[k];
    }
    __syncthreads();
    if (threadIdx.x < A.world) {
      int t = 0;
      for (int w = 0; w < nw; ++w) t += wcnt[w][threadIdx.x];
      base[threadIdx.x] += t;
    }
    __syncthreads();
  }
  if (threadIdx.x < A.world) A.cursor[threadIdx.x] = base[threadIdx.x];
  __syncthreads();
  publish(A);
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
  uint64_t launches = 0;
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
  cudaError_t e = cudaMalloc(&px->local, region_bytes);
  if (e == cudaSuccess) e = cudaMemset(px->local, 0, region_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&px->d_cursor, 2 * kMaxWorld * sizeof(int32_t) + 2 * sizeof(unsigned) + 16);
  if (e == cudaSuccess) {
    px->d_done = reinterpret_cast<unsigned*>(px->d_cursor + 2 * kMaxWorld);
    px->d_status = reinterpret_cast<int32_t*>(px->d_done + 2);
    e = cudaMemset(px->d_cursor, 0, 2 * kMaxWorld * sizeof(int32_t) + 2 * sizeof(unsigned) + 16);
  }
  if (e == cudaSuccess && handle_out) e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle_out), px->local);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (px->local) cudaFree(px->local);
    if (px->d_cursor) cudaFree(px->d_cursor);
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
                 int32_t stable, int64_t* d_slot, int32_t* d_overflow, void* stream) {
  if (!px || n < 0 || rec_words < 1 || cap < 0 || seq == 0 || !d_overflow || (n > 0 && (!d_owner || !d_records || !d_slot)))
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
  const int kind = stable ? 1 : 0;  // separate cursors: a stable and an atomic send may run concurrently
  A.cursor = px->d_cursor + kind * kMaxWorld;
  A.done = px->d_done + kind;
  auto st = static_cast<cudaStream_t>(stream);
  if (stable) {
    k_px_send_stable<<<1, 1024, 0, st>>>(A);
  } else {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, px->device);
    const int64_t warps = (n + 31) / 32;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 4LL * sms)));
    k_px_send_atomic<<<blocks, 256, 0, st>>>(A);
  }
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
  delete px;
  return DGDS_OK;
}

}  // extern "C"

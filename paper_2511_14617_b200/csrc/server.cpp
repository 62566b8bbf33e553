// server.cpp — host side of the B200 DGDS: the extern "C" ABI declared in
// include/dgds_b200.h over the sm_100a kernels in kernels.cu.
//
// Host work here is O(records) bookkeeping that the reference performs per
// call under its shard mutex (proj/src/dgds.cpp:36-51,99-138): group lookup
// with lazy TTL expiry, auto-registration, per-stream gap check and version
// numbering in call order (cst.cpp:118-133). Record replies are therefore
// final before any device work completes. All trie work — insertion, suffix
// match, beam, verification — runs on the GPU; there is no CPU fallback: a
// missing device is an error.

#include <cuda_runtime.h>
#include <emmintrin.h>
#include <deque>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <unordered_map>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <vector>

#include "../../include/dgds_b200.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define DGDS_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(DGDS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

uint64_t fnv1a64(const void* data, size_t n) {  // detail::fnv1a64 (bytes.hpp:89-96)
  const auto* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// Probing is CAS-by-CAS at insert, so load sets the atomics per claim (C2: 0.42 -> 0.30
// took K1 from 227 to 206 us); memory is plentiful (C2 at load 0.30 is 53 GB of 180 GB).
constexpr double kMaxLoad = 0.60;     // rebuild threshold
constexpr double kTargetLoad = 0.35;  // load right after a rebuild
constexpr uint32_t kRootCap = 1u << 22;
constexpr uint64_t kMaxCap = (0xFFFFFFFFull - kRootCap - 2) / 4 * 4;

struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
  unsigned flags = cudaHostAllocDefault;  // cudaHostAllocMapped: kernels may store into it
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  int ensure(size_t bytes) {
    if (bytes <= cap) return DGDS_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    size_t c = std::max<size_t>(bytes, cap * 2);
    if (cudaHostAlloc(&p, c, flags) != cudaSuccess) {
      cap = 0;
      return fail(DGDS_ENOMEM, "cudaHostAlloc failed");
    }
    cap = c;
    return DGDS_OK;
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  int ensure(size_t bytes) {
    if (bytes <= cap) return DGDS_OK;
    if (p) cudaFree(p);
    p = nullptr;
    size_t c = std::max<size_t>(bytes, cap * 2);
    if (cudaMalloc(&p, c) != cudaSuccess) {
      cap = 0;
      return fail(DGDS_ENOMEM, "cudaMalloc failed");
    }
    cap = c;
    return DGDS_OK;
  }
};

// Persistent host workers for the O(n) staging / scatter loops of the host-buffer path
// (thread creation per call cost more than the work). The caller thread takes part.
class WorkerPool {
 public:
  explicit WorkerPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int threads() const { return static_cast<int>(th_.size()) + 1; }
  // fn(i) for i in [0, tasks), returns when all are done
  void run(int tasks, const std::function<void(int)>& fn) {
    join();
    if (tasks <= 1 || th_.empty()) {
      for (int i = 0; i < tasks; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      tasks_ = tasks;
      next_.store(0);
      pending_ = tasks;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }
  // fn(i) for i in [0, tasks) on the workers alone; returns at once, join() waits
  void post(int tasks, std::function<void(int)> fn) {
    join();
    if (th_.empty()) {
      for (int i = 0; i < tasks; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      owned_ = std::move(fn);
      fn_ = &owned_;
      tasks_ = tasks;
      next_.store(0);
      pending_ = tasks;
      posted_ = true;
      ++gen_;
    }
    cv_.notify_all();
  }
  void join() {
    std::unique_lock<std::mutex> lk(mu_);
    if (!posted_) return;
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
    posted_ = false;
  }

 private:
  void work() {
    int done = 0;
    for (int i = next_.fetch_add(1); i < tasks_; i = next_.fetch_add(1)) {
      (*fn_)(i);
      ++done;
    }
    if (done) {
      std::lock_guard<std::mutex> lk(mu_);
      pending_ -= done;
      if (pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (!fn_) continue;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  std::function<void(int)> owned_;  // a posted job
  bool posted_ = false;
  int tasks_ = 0;
  int pending_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

int host_threads() {
  if (const char* e = std::getenv("DGDS_HOST_THREADS")) return std::max(1, std::atoi(e));
  const int hc = static_cast<int>(std::thread::hardware_concurrency());
  return std::max(1, std::min(8, hc - 1));
}

struct LogRec {  // GroupDraftIndex::LogEntry (cst.hpp:120-124) + where its tokens live
  uint64_t off;
  uint64_t start;
  uint32_t len;
  int32_t rid;
};

struct StreamRec {
  uint64_t stored = 0;
  uint32_t slot = 0;
  int64_t batch_seg = -1;  // segment index in the batch being built
  uint64_t batch_stamp = 0;
};

// request-id -> stream: direct-indexed for small ids (the common case: a group's
// responses are numbered 0..G-1), hashed beyond
class StreamTable {
 public:
  static constexpr int32_t kDirect = 256;
  StreamRec* find(int32_t rid) {
    if (rid < kDirect) return rid < static_cast<int32_t>(present_.size()) && present_[rid] ? &direct_[rid] : nullptr;
    auto it = far_.find(rid);
    return it == far_.end() ? nullptr : &it->second;
  }
  StreamRec& insert(int32_t rid, const StreamRec& v) {
    if (rid < kDirect) {
      if (rid >= static_cast<int32_t>(present_.size())) {
        present_.resize(rid + 1, 0);
        direct_.resize(rid + 1);
      }
      present_[rid] = 1;
      direct_[rid] = v;
      ++n_;
      return direct_[rid];
    }
    ++n_;
    return far_.emplace(rid, v).first->second;
  }
  void clear() {
    present_.clear();
    direct_.clear();
    far_.clear();
    n_ = 0;
  }
  template <class F>
  void for_each(F&& f) {
    for (size_t i = 0; i < present_.size(); ++i)
      if (present_[i]) f(static_cast<int32_t>(i), direct_[i]);
    for (auto& kv : far_) f(kv.first, kv.second);
  }
  size_t size() const { return n_; }

 private:
  std::vector<uint8_t> present_;
  std::vector<StreamRec> direct_;
  std::unordered_map<int32_t, StreamRec> far_;
  size_t n_ = 0;
};

struct GroupRec {
  std::string gid;
  int32_t shard = 0;
  bool alive = false;
  uint32_t root = 0;
  double ttl = 0.0;
  double expires = 0.0;
  uint64_t version = 0;
  StreamTable streams;
  // Every accepted append of the group, in order (a deque: grows without copying).
  // Entries [delta_base, end) are versions log_floor+1 .. version (delta blobs);
  // all entries together hold every stream's tokens (full snapshots).
  std::deque<LogRec> log;
  size_t delta_base = 0;
  uint64_t log_floor = 0;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Debug: DGDS_HOST_TIMING=1 prints the host-path phases of each call to stderr.
struct PhaseClock {
  bool on;
  const char* name;
  std::chrono::steady_clock::time_point t0, last;
  std::string line;
  explicit PhaseClock(const char* n) : on(std::getenv("DGDS_HOST_TIMING") != nullptr), name(n) {
    if (on) t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* phase) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    line += std::string(" ") + phase + "=" +
            std::to_string(std::chrono::duration<double, std::micro>(t - last).count()).substr(0, 7);
    last = t;
  }
  ~PhaseClock() {
    if (on)
      std::fprintf(stderr, "[%s] total=%.1fus%s\n", name,
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(),
                   line.c_str());
  }
};

// Copy into pinned staging memory with non-temporal (streaming) stores. A staging block
// written by several threads with normal stores, then read by the device (DMA or a pull
// kernel), measured 8 GB/s on the GPU box instead of 52 GB/s: the device reads snoop
// lines still dirty in the writers' caches (tools/h2d_dirty.cu). The caller fences.
void nt_copy(void* dst, const void* src, size_t n) {
  char* d = static_cast<char*>(dst);
  const char* sp = static_cast<const char*>(src);
  const size_t head = std::min<size_t>(n, (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
  std::memcpy(d, sp, head);
  d += head;
  sp += head;
  n -= head;
  for (; n >= 16; n -= 16, d += 16, sp += 16)
    _mm_stream_si128(reinterpret_cast<__m128i*>(d), _mm_loadu_si128(reinterpret_cast<const __m128i*>(sp)));
  std::memcpy(d, sp, n);
}

}  // namespace

struct dgds_server;
static void free_plan_pool(dgds_server* s);  // after dgds_update_plan is complete
namespace {
int flush_pending(dgds_server* s);  // launches a submitted query batch; before any later device work
int launch_batch(dgds_server* s, bool timed);
// one chunk of a staged host query batch: handles | pat_len | patterns | args | truth | truth_left | limit
struct QInBlock {
  int64_t q0 = 0, m = 0;
  size_t base = 0, o_len = 0, o_pat = 0, o_args = 0, o_tr = 0, o_tl = 0, o_lm = 0, bytes = 0;
};
// device outputs of a host query batch (internal strides) + compaction scratch
struct QOutLayout {
  size_t sc = 0, sp = 0, nc = 0, ln = 0, tk = 0, v = 0, bs = 0, tot = 0, cmeta = 0, ctoff = 0, ccoff = 0, ctok = 0;
};
}  // namespace

struct dgds_server {
  dgds_params p{};
  int32_t D = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t staging_free = nullptr;
  // host-path query inputs: own staging pair and copy stream, so their H2D overlaps the
  // append kernel queued before them on `st`
  cudaStream_t copy_st = nullptr;
  // Host-path query batches in flight (dgds_speculate_submit / _wait): each owns a slot with
  // its staging, device outputs and mapped result block, so the next batch is staged while
  // this one runs. Copy-outs run on out_st, beside the next batch's append and query kernels.
  static constexpr int kQSlots = 2;
  struct QSlot {
    PinnedBuf hq, ho;  // mapped: the pull kernel reads hq, the copy-out kernel writes ho
    DevBuf dq, dout;
    cudaEvent_t done = nullptr;  // the batch's last copy-out finished
    uint64_t ticket = 0;         // 0: never used
    int64_t n = 0;
    bool verify = false;
    int err = DGDS_OK;  // the batch failed validation (nothing launched)
    std::string err_msg;
    size_t h_coff = 0, h_v = 0, h_meta = 0, h_toff = 0, h_tok = 0;
  } qslot[kQSlots];
  uint64_t last_ticket = 0;
  cudaStream_t out_st = nullptr;
  // optional chunking of one batch (DGDS_Q_CHUNKS, batches of >= 32K queries): chunk c's H2D
  // beside chunk c+1's staging, its copy-out beside chunk c+1's query kernel. Off by default:
  // the query kernel's fixed latency tail makes 4 x 16K queries slower than 1 x 64K.
  static constexpr int kMaxQChunks = 16;
  cudaEvent_t ev_h2d[kMaxQChunks] = {}, ev_cmp[kMaxQChunks] = {};
  int q_chunks = 1;
  int out_blocks = 148;  // copy-out grid when chunked; DGDS_OUT_BLOCKS
  // the submitted batch whose staging may still run on the workers (kernels not yet launched)
  struct PendingQuery {
    bool active = false;
    uint64_t ticket = 0;
    int64_t n = 0, args_stride = 0;
    int nch = 1;
    int32_t K = 1, Sx = 1, truth_stride = 0;
    bool verify = false;
    QInBlock blk[kMaxQChunks];
    QOutLayout out;
    std::atomic<int> left{0};           // staging tasks still running
    std::atomic<int64_t> bad{0};        // first invalid query (INT64_MAX: none)
    const int32_t* handles = nullptr;   // the caller's, for the error message
    int64_t ng = 0;                     // groups at submit
    std::atomic<cudaError_t> h2d_err{cudaSuccess};  // set by the last stager
    bool stager_launch = true;          // the last stager also launches the kernels
    bool launched = false;
    int launch_rc = DGDS_OK;
    std::string launch_msg;
  } pq;
  int stage_tasks = 8;  // workers of an asynchronous stage; DGDS_STAGE_TASKS
  bool async_stage = true;  // DGDS_ASYNC_STAGE=0: submit stages synchronously
  dgds::DevTrie T{};
  unsigned long long* d_used = nullptr;
  uint64_t used_ub = 0;  // upper bound on occupied slots since the last exact read

  int32_t* d_hist = nullptr;  // append-only token history (GDX1 blobs); K1 fills it
  uint64_t hist_cap = 0, hist_used = 0;
  uint64_t dead_hist_tokens = 0;  // history of retired groups (reclaimed by compact_memory)
  uint64_t compactions = 0;
  DevBuf d_blob, d_blob_pieces;
  PinnedBuf h_blob;

  uint32_t* d_root_of = nullptr;
  size_t root_of_cap = 0;
  uint32_t next_root_index = 0;

  uint64_t stream_cap = 0;
  uint32_t next_stream = 0;
  std::vector<uint32_t> free_streams;

  std::unordered_map<std::string, int32_t> intern;
  std::vector<GroupRec> groups;
  std::vector<uint64_t> shard_counts;
  uint64_t batch_stamp = 0;

  PinnedBuf h_stage, h_out;  // update staging; dgds_verify_batch results
  DevBuf d_stage, d_out;
  bool h2d_kernel = false;  // copy-engine H2D (no SMs taken from K1); DGDS_H2D=kernel: a pull kernel
  int h2d_blocks = 148;    // one CTA per SM (measured best); DGDS_H2D_BLOCKS
  std::unique_ptr<WorkerPool> pool;
  uint64_t plans_made = 0, plans_launched = 0;  // two-phase device updates (plan now, launch later)
  std::vector<struct dgds_update_plan*> plan_pool;  // recycled plans: their vectors keep capacity
  // planning scratch, reused across calls (per-call vectors of 16-130 KB were page-faulting)
  struct PlanScratch {
    std::vector<dgds::AppendSeg> segs;
    std::vector<dgds::AppendPiece> pieces;
    std::vector<uint32_t> cnt, fill;
  } scratch;
  WorkerPool& workers() {
    if (!pool) pool = std::make_unique<WorkerPool>(host_threads() - 1);
    return *pool;
  }
  int32_t* d_err = nullptr;
  unsigned long long* d_stat_part = nullptr;  // [kStatParts][8] query-counter partitions
  std::mutex mu;  // calls on one handle are serialized

  long long* d_dbg = nullptr;  // optional per-query phase timing buffer (debug)
  uint64_t last_d2h_bytes = 0;  // device->host bytes of the last host-path query call
  // kernel timing: event pairs around launches (kind 0 append, 1 query)
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending[2];
  uint64_t prof_launches[2] = {0, 0};
  double prof_ms[2] = {0.0, 0.0};
};

namespace {

int set_root(dgds_server* s, int32_t handle, uint32_t root) {
  if (int rc = flush_pending(s)) return rc;  // a submitted query reads root_of as it was
  if (static_cast<size_t>(handle) >= s->root_of_cap) {
    size_t nc = std::max<size_t>(1024, s->root_of_cap * 2);
    while (nc <= static_cast<size_t>(handle)) nc *= 2;
    uint32_t* nb = nullptr;
    DGDS_CUDA(cudaMalloc(&nb, nc * sizeof(uint32_t)));
    DGDS_CUDA(cudaMemsetAsync(nb, 0, nc * sizeof(uint32_t), s->st));
    if (s->d_root_of) {
      DGDS_CUDA(cudaMemcpyAsync(nb, s->d_root_of, s->root_of_cap * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s->st));
      DGDS_CUDA(cudaStreamSynchronize(s->st));
      cudaFree(s->d_root_of);
    }
    s->d_root_of = nb;
    s->root_of_cap = nc;
  }
  DGDS_CUDA(dgds::launch_set_u32(s->d_root_of + handle, root, s->st));
  return DGDS_OK;
}

int alloc_stream_slot(dgds_server* s, uint32_t* out) {
  if (!s->free_streams.empty()) {
    *out = s->free_streams.back();
    s->free_streams.pop_back();
    return DGDS_OK;
  }
  if (s->next_stream >= s->stream_cap) {
    if (int rc = flush_pending(s)) return rc;  // T.active / T.tail change under a staged batch's launch
    uint64_t nc = std::max<uint64_t>(1024, s->stream_cap * 2);
    uint32_t* na = nullptr;
    int32_t* nt = nullptr;
    DGDS_CUDA(cudaMalloc(&na, nc * dgds::kWarp * sizeof(uint32_t)));
    DGDS_CUDA(cudaMalloc(&nt, nc * dgds::kWarp * sizeof(int32_t)));
    if (s->T.active) {
      DGDS_CUDA(cudaMemcpyAsync(na, s->T.active, s->stream_cap * dgds::kWarp * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, s->st));
      DGDS_CUDA(cudaMemcpyAsync(nt, s->T.tail, s->stream_cap * dgds::kWarp * sizeof(int32_t),
                                cudaMemcpyDeviceToDevice, s->st));
      DGDS_CUDA(cudaStreamSynchronize(s->st));
      cudaFree(s->T.active);
      cudaFree(s->T.tail);
    }
    s->T.active = na;
    s->T.tail = nt;
    s->stream_cap = nc;
  }
  *out = s->next_stream++;
  return DGDS_OK;
}

void retire_group(dgds_server* s, GroupRec& g) {
  if (!g.alive) return;
  for (const LogRec& e : g.log) s->dead_hist_tokens += e.len;
  g.streams.for_each([&](int32_t, StreamRec& r) { s->free_streams.push_back(r.slot); });
  g.streams.clear();
  g.log.clear();
  g.log.shrink_to_fit();
  g.delta_base = 0;
  g.log_floor = 0;
  g.alive = false;
  g.version = 0;
  s->shard_counts[g.shard] -= 1;
  set_root(s, static_cast<int32_t>(&g - s->groups.data()), 0u);
}

int create_group(dgds_server* s, GroupRec& g, double ttl, double now) {
  if (s->next_root_index >= kRootCap) return fail(DGDS_EUNSUPPORTED, "group root ids exhausted");
  g.root = dgds::kRootTop - s->next_root_index++;
  g.alive = true;
  g.ttl = ttl;
  g.expires = now + ttl;
  g.version = 0;
  g.streams.clear();
  g.log.clear();
  g.delta_base = 0;
  g.log_floor = 0;
  s->shard_counts[g.shard] += 1;
  return set_root(s, static_cast<int32_t>(&g - s->groups.data()), g.root);
}

// find_entry with lazy expiry (dgds.cpp:25-34)
bool live_entry(dgds_server* s, GroupRec& g, double now) {
  if (!g.alive) return false;
  if (g.expires < now) {
    retire_group(s, g);
    return false;
  }
  return true;
}

int check_handle(dgds_server* s, int32_t h) {
  if (h < 0 || static_cast<size_t>(h) >= s->groups.size()) return fail(DGDS_EINVAL, "bad group handle");
  return DGDS_OK;
}

// validate_args (cst.cpp:18-25) + device limits
int check_args(const dgds_spec_args& a) {
  if (a.pattern_lookup_min < 1 || a.pattern_lookup_min > a.pattern_lookup_max)
    return fail(DGDS_EINVAL, "speculation args: need 1 <= pattern_lookup_min <= pattern_lookup_max");
  if (a.max_spec_tokens < 0) return fail(DGDS_EINVAL, "speculation args: max_spec_tokens must be >= 0");
  if (a.top_k < 1) return fail(DGDS_EINVAL, "speculation args: top_k must be >= 1");
  if (a.min_step_freq < 0.0) return fail(DGDS_EINVAL, "speculation args: min_step_freq must be >= 0");
  if (a.min_support < 0) return fail(DGDS_EINVAL, "speculation args: min_support must be >= 0");
  if (a.top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "top_k above DGDS_MAX_TOP_K");
  return DGDS_OK;
}

uint64_t cap_for(uint64_t nodes, double load) {  // slots, a multiple of the probe window
  uint64_t c = static_cast<uint64_t>(std::ceil(static_cast<double>(nodes) / load));
  c = std::max<uint64_t>(c, 1024);
  return (c + dgds::kWindow - 1) / dgds::kWindow * dgds::kWindow;
}

int read_used(dgds_server* s, uint64_t* out) {
  unsigned long long u = 0;
  unsigned long long parts[dgds::kUsedParts * 8];
  DGDS_CUDA(cudaMemcpyAsync(parts, s->d_used, sizeof(parts), cudaMemcpyDeviceToHost, s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  for (int p = 0; p < dgds::kUsedParts; ++p) u += parts[p * 8];
  *out = u;
  return DGDS_OK;
}

// Grow (and garbage-collect dropped groups) by rebuilding into a larger table.
int rebuild(dgds_server* s, uint64_t new_cap) {
  if (new_cap > kMaxCap) new_cap = kMaxCap / dgds::kWindow * dgds::kWindow;
  dgds::DevTrie to = s->T;
  to.cap = new_cap;
  DGDS_CUDA(cudaMalloc(&to.slots, new_cap * sizeof(dgds::Slot)));
  DGDS_CUDA(cudaMemsetAsync(to.slots, 0, new_cap * sizeof(dgds::Slot), s->st));
  unsigned long long* d_used_new = nullptr;
  DGDS_CUDA(cudaMalloc(&d_used_new, dgds::kUsedParts * 8 * sizeof(unsigned long long)));
  DGDS_CUDA(cudaMemsetAsync(d_used_new, 0, dgds::kUsedParts * 8 * sizeof(unsigned long long), s->st));
  to.used = d_used_new;
  std::vector<uint32_t> alive((kRootCap + 31) / 32, 0);
  std::vector<uint32_t> live_slots, live_sizes;
  for (auto& g : s->groups) {
    if (!g.alive) continue;
    const uint32_t r = dgds::kRootTop - g.root;
    alive[r >> 5] |= 1u << (r & 31);
    g.streams.for_each([&](int32_t, StreamRec& r) {
      live_slots.push_back(r.slot);
      live_sizes.push_back(static_cast<uint32_t>(std::min<uint64_t>(r.stored, s->D)));
    });
  }
  uint32_t *d_alive = nullptr, *d_remap = nullptr, *d_ls = nullptr;
  DGDS_CUDA(cudaMalloc(&d_alive, alive.size() * 4));
  DGDS_CUDA(cudaMalloc(&d_remap, s->T.cap * 4));
  DGDS_CUDA(cudaMalloc(&d_ls, std::max<size_t>(1, live_slots.size()) * 8));
  DGDS_CUDA(cudaMemcpyAsync(d_alive, alive.data(), alive.size() * 4, cudaMemcpyHostToDevice, s->st));
  DGDS_CUDA(cudaMemsetAsync(d_remap, 0, s->T.cap * 4, s->st));
  if (!live_slots.empty()) {
    DGDS_CUDA(cudaMemcpyAsync(d_ls, live_slots.data(), live_slots.size() * 4, cudaMemcpyHostToDevice, s->st));
    DGDS_CUDA(cudaMemcpyAsync(d_ls + live_slots.size(), live_sizes.data(), live_sizes.size() * 4,
                              cudaMemcpyHostToDevice, s->st));
  }
  DGDS_CUDA(dgds::launch_rebuild(s->T, to, d_alive, d_remap, s->st));
  DGDS_CUDA(dgds::launch_remap_active(s->T.active, d_ls, d_ls + live_slots.size(),
                                      static_cast<int64_t>(live_slots.size()), d_remap, s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));  // host vectors above must outlive the copies
  cudaFree(d_alive);
  cudaFree(d_remap);
  cudaFree(d_ls);
  cudaFree(s->T.slots);
  cudaFree(s->d_used);
  s->T.slots = to.slots;
  s->T.cap = new_cap;
  s->T.used = d_used_new;
  s->d_used = d_used_new;
  return read_used(s, &s->used_ub);
}

int ensure_capacity(dgds_server* s, uint64_t worst_new) {
  if (int rc = flush_pending(s)) return rc;  // a submitted query reads the table as it was
  const double limit = kMaxLoad * static_cast<double>(s->T.cap);
  if (static_cast<double>(s->used_ub + worst_new) <= limit) return DGDS_OK;
  int rc = read_used(s, &s->used_ub);
  if (rc) return rc;
  if (static_cast<double>(s->used_ub + worst_new) <= limit) return DGDS_OK;
  const uint64_t want = std::max<uint64_t>(cap_for(s->used_ub + worst_new, kTargetLoad), s->T.cap * 2);
  if (s->used_ub + worst_new > static_cast<uint64_t>(kMaxLoad * static_cast<double>(std::min(want, kMaxCap))))
    return fail(DGDS_ENOMEM, "draft-index arena exceeds the 32-bit node-id space");
  return rebuild(s, want);
}

// Window insertions at positions start+1 .. start+n: sum min(D, pos).
uint64_t worst_windows(uint64_t start, uint64_t n, uint64_t D) {
  uint64_t total = 0;
  const uint64_t lo = start + 1, hi = start + n;  // inclusive positions
  if (lo <= D) {
    const uint64_t top = std::min(hi, D);
    total += (lo + top) * (top - lo + 1) / 2;
  }
  if (hi > D) total += (hi - std::max(lo, D + 1) + 1) * D;
  return total;
}

struct PendingPiece {
  int64_t seg;
  uint64_t tok_off;
  uint64_t hist_off;
  uint32_t n;
};

// Grow the history arena to hold hist_used tokens (stream-ordered copy; rare).
int ensure_hist(dgds_server* s) {
  if (s->hist_used <= s->hist_cap) return DGDS_OK;
  if (int rc = flush_pending(s)) return rc;  // T.hist changes under a staged batch's launch
  uint64_t nc = std::max<uint64_t>(s->hist_used, s->hist_cap * 2);
  int32_t* nb = nullptr;
  if (cudaMalloc(&nb, nc * sizeof(int32_t)) != cudaSuccess) return fail(DGDS_ENOMEM, "history arena allocation failed");
  if (s->d_hist) {
    DGDS_CUDA(cudaStreamSynchronize(s->st));  // appends in flight finish writing the old arena
    DGDS_CUDA(cudaMemcpy(nb, s->d_hist, s->hist_cap * sizeof(int32_t), cudaMemcpyDeviceToDevice));
    cudaFree(s->d_hist);
  }
  s->d_hist = nb;
  s->hist_cap = nc;
  s->T.hist = nb;
  return DGDS_OK;
}

// Shared host logic of update_batch / update_batch_device: replies in call
// order (DraftServer::update_cst, dgds.cpp:36-51 -> GroupDraftIndex::append,
// cst.cpp:118-133), plus the device segment table.
// Record i's tokens are tokens[tok_start(i) .. tok_start(i) + tok_count(i)).
int plan_updates(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids, const uint64_t* prev,
                 const uint64_t* offs, const uint64_t* counts, double now, dgds_update_reply* rep,
                 std::vector<dgds::AppendSeg>& segs, std::vector<dgds::AppendPiece>& pieces, uint64_t* worst) {
  // offs[n+1] cumulative (counts == nullptr), or offs[n] starts + counts[n]
  auto tstart = [&](int64_t i) { return offs[i]; };
  auto tcount = [&](int64_t i) { return counts ? counts[i] : offs[i + 1] - offs[i]; };
  for (int64_t i = 0; i < n; ++i) {
    int rc = check_handle(s, handles[i]);
    if (rc) return rc;
    if (rids[i] < 0) return fail(DGDS_EINVAL, "request_id must be nonnegative");
    if (!counts && offs[i + 1] < offs[i]) return fail(DGDS_EINVAL, "token offsets must be nondecreasing");
  }
  PhaseClock pcl("plan_updates");
  const uint64_t stamp = ++s->batch_stamp;
  segs.clear();
  *worst = 0;
  // Records of different groups are independent (version, streams and log are per group), so
  // large batches are planned in parallel with the groups partitioned over the host workers;
  // each worker walks the batch in call order for its groups. Global state (group roots,
  // stream slots) is touched under one mutex — only when a group or stream is created.
  // Measured: the pool wake-up and cross-core traffic on group/stream records cost more than
  // the planning saves at bench sizes (4096 records: 0.34 -> 0.61 ms per step), so the parallel
  // path is opt-in (DGDS_PARALLEL_PLAN=<min records>).
  static const int64_t par_min = [] {
    const char* e = std::getenv("DGDS_PARALLEL_PLAN");
    return e ? std::max<int64_t>(1, std::atoll(e)) : INT64_MAX;
  }();
  WorkerPool& pool = s->workers();
  const int W = (n >= par_min && pool.threads() > 1) ? pool.threads() : 1;
  struct Part {
    std::vector<dgds::AppendSeg> segs;
    std::vector<PendingPiece> pend;
    uint64_t worst = 0;
    int rc = DGDS_OK;
    std::string msg;
  };
  thread_local std::vector<Part> parts;  // kept across calls: capacity persists
  parts.resize(W);
  for (Part& P : parts) {
    P.segs.clear();
    P.pend.clear();
    P.worst = 0;
    P.rc = DGDS_OK;
  }
  std::mutex gmu;
  std::atomic<uint64_t> hist_at{s->hist_used};
  uint64_t hist_one = s->hist_used;
  auto work = [&](int w) {
    Part& P = parts[w];
    if (W > 1) cudaSetDevice(s->p.device);
    for (int64_t i = 0; i < n; ++i) {
      if (W > 1 && handles[i] % W != w) continue;
      GroupRec& g = s->groups[handles[i]];
      if (!g.alive || g.expires < now) {
        std::lock_guard<std::mutex> lk(gmu);
        if (!live_entry(s, g, now)) {
          const int rc = create_group(s, g, s->p.default_ttl_seconds, now);  // auto-register (dgds.cpp:42-47)
          if (rc) {
            P.rc = rc;
            P.msg = dgds_last_error();
            return;
          }
        }
      }
      g.expires = now + g.ttl;
      StreamRec* found = g.streams.find(rids[i]);
      if (!found) {  // a mismatched append still creates the stream (cst.cpp:121)
        StreamRec fresh;
        {
          std::lock_guard<std::mutex> lk(gmu);
          const int rc = alloc_stream_slot(s, &fresh.slot);
          if (rc) {
            P.rc = rc;
            P.msg = dgds_last_error();
            return;
          }
        }
        found = &g.streams.insert(rids[i], fresh);
      }
      StreamRec& sr = *found;
      const uint64_t cnt = tcount(i);
      if (prev[i] != sr.stored) {
        rep[i] = dgds_update_reply{0, 0, g.version, sr.stored};
        continue;
      }
      if (cnt == 0) {
        rep[i] = dgds_update_reply{1, 0, g.version, sr.stored};
        continue;
      }
      if (sr.batch_stamp != stamp) {
        sr.batch_stamp = stamp;
        sr.batch_seg = static_cast<int64_t>(P.segs.size());  // local to this worker until the merge
        dgds::AppendSeg sg{};
        sg.stream = sr.slot;
        sg.root = g.root;
        sg.start = sr.stored;
        P.segs.push_back(sg);
      }
      uint64_t hoff;
      if (W == 1) {  // single planner: no locked read-modify-write per record
        hoff = hist_one;
        hist_one += cnt;
      } else {
        hoff = hist_at.fetch_add(cnt, std::memory_order_relaxed);
      }
      P.pend.push_back(PendingPiece{sr.batch_seg, tstart(i), hoff, static_cast<uint32_t>(cnt)});
      g.log.push_back(LogRec{hoff, sr.stored, static_cast<uint32_t>(cnt), rids[i]});
      P.worst += worst_windows(sr.stored, cnt, static_cast<uint64_t>(s->D));
      sr.stored += cnt;
      g.version += 1;
      rep[i] = dgds_update_reply{1, 0, g.version, sr.stored};
    }
  };
  pcl.mark("validate_setup");
  if (W > 1) pool.run(W, work);
  else work(0);
  pcl.mark("records");
  s->hist_used = W == 1 ? hist_one : hist_at.load();
  for (const Part& P : parts)
    if (P.rc) return fail(P.rc, P.msg);
  // merge the workers' segments; group pieces by segment, keeping call order inside a segment
  if (W == 1 && parts[0].pend.size() == parts[0].segs.size()) {  // one piece per segment: no grouping
    Part& P = parts[0];
    segs.assign(P.segs.begin(), P.segs.end());  // copy: both vectors keep their capacity
    *worst = P.worst;
    pieces.resize(P.pend.size());
    for (size_t k = 0; k < P.pend.size(); ++k) {
      const PendingPiece& pp = P.pend[k];
      segs[pp.seg].piece0 = static_cast<uint32_t>(k);
      segs[pp.seg].npieces = 1;
      pieces[k] = dgds::AppendPiece{pp.tok_off, pp.hist_off, pp.n, 0};
    }
    pcl.mark("pieces_fast");
    return DGDS_OK;
  }
  std::vector<int64_t> base(W + 1, 0);
  for (int w = 0; w < W; ++w) base[w + 1] = base[w] + static_cast<int64_t>(parts[w].segs.size());
  segs.reserve(base[W]);
  for (int w = 0; w < W; ++w) segs.insert(segs.end(), parts[w].segs.begin(), parts[w].segs.end());
  std::vector<uint32_t>& cnt = s->scratch.cnt;
  cnt.assign(segs.size() + 1, 0);
  size_t npend = 0;
  for (int w = 0; w < W; ++w) {
    *worst += parts[w].worst;
    for (const auto& pp : parts[w].pend) cnt[base[w] + pp.seg + 1]++;
    npend += parts[w].pend.size();
  }
  for (size_t k = 0; k < segs.size(); ++k) {
    segs[k].piece0 = cnt[k];
    segs[k].npieces = cnt[k + 1];
    cnt[k + 1] += cnt[k];
  }
  pieces.assign(npend, dgds::AppendPiece{});
  std::vector<uint32_t>& fill = s->scratch.fill;
  fill.assign(segs.size(), 0);
  for (int w = 0; w < W; ++w) {
    for (const auto& pp : parts[w].pend) {
      const int64_t sg = base[w] + pp.seg;
      const uint32_t at = segs[sg].piece0 + fill[sg]++;
      pieces[at] = dgds::AppendPiece{pp.tok_off, pp.hist_off, pp.n, 0};
    }
  }
  return DGDS_OK;
}

cudaEvent_t pooled_event(dgds_server* s) {
  if (!s->ev_pool.empty()) {
    cudaEvent_t e = s->ev_pool.back();
    s->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets one kernel launch with events on its stream when profiling is on.
struct LaunchTimer {
  dgds_server* s;
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchTimer(dgds_server* srv, int k, cudaStream_t stream) : s(srv), kind(k), st(stream) {
    if (s->profiling) {
      a = pooled_event(s);
      b = pooled_event(s);
      cudaEventRecord(a, st);
    }
  }
  ~LaunchTimer() {
    if (a) {
      cudaEventRecord(b, st);
      s->ev_pending[kind].emplace_back(a, b);
    }
  }
};

// Make `st` (user stream) and the server stream observe one total order.
struct StreamJoin {  // work of a device-API call runs on the caller's stream, ordered after the server's
  dgds_server* s;
  cudaStream_t user;
  cudaEvent_t ev = nullptr;
  // NULL is the legacy default stream (CUDA convention; torch's default stream), not the server's
  StreamJoin(dgds_server* srv, void* u) : s(srv), user(u ? static_cast<cudaStream_t>(u) : cudaStreamLegacy) {
    if (user != s->st) {
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, s->st);
      cudaStreamWaitEvent(user, ev, 0);
    }
  }
  cudaStream_t stream() const { return user; }
  ~StreamJoin() {
    if (ev) {
      cudaEventRecord(ev, user);
      cudaStreamWaitEvent(s->st, ev, 0);
      cudaEventDestroy(ev);
    }
  }
};

}  // namespace

namespace dgds {
int set_error(int code, const std::string& msg) { return fail(code, msg); }  // shared with peer.cu
}  // namespace dgds

namespace {

}  // namespace

extern "C" {

const char* dgds_last_error(void) { return g_err.c_str(); }
const char* dgds_version_string(void) { return "dgds-b200 0.1 (sm_100a)"; }

uint64_t dgds_fnv1a64(const void* data, size_t n) { return fnv1a64(data, n); }

int32_t dgds_shard_of_group(const char* gid, size_t len, int32_t shard_count) {  // dgds.cpp:10-14
  if (shard_count < 1) return fail(DGDS_EINVAL, "shard_count must be >= 1");
  return static_cast<int32_t>(fnv1a64(gid, len) % static_cast<uint64_t>(shard_count));
}

int dgds_create(const dgds_params* params, dgds_server** out) {
  if (!params || !out) return fail(DGDS_EINVAL, "null argument");
  const dgds_params& p = *params;
  if (p.shard_count < 1) return fail(DGDS_EINVAL, "shard_count must be >= 1");
  if (p.max_pattern_len < 1 || p.max_spec_len < 0) return fail(DGDS_EINVAL, "draft index limits out of range");
  if (p.max_pattern_len + p.max_spec_len > DGDS_MAX_DEPTH)
    return fail(DGDS_EUNSUPPORTED, "max_pattern_len + max_spec_len exceeds DGDS_MAX_DEPTH (32)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(DGDS_ECUDA, "no CUDA device");
  if (p.device < 0 || p.device >= ndev) return fail(DGDS_EINVAL, "bad device ordinal");
  DGDS_CUDA(cudaSetDevice(p.device));
  auto s = std::make_unique<dgds_server>();
  s->p = p;
  for (auto& q : s->qslot) q.hq.flags = q.ho.flags = cudaHostAllocMapped;
  if (const char* e = std::getenv("DGDS_H2D")) s->h2d_kernel = std::strcmp(e, "kernel") == 0;
  cudaDeviceGetAttribute(&s->h2d_blocks, cudaDevAttrMultiProcessorCount, p.device);
  if (const char* e = std::getenv("DGDS_H2D_BLOCKS")) s->h2d_blocks = std::max(1, std::atoi(e));
  s->D = p.max_pattern_len + p.max_spec_len;
  s->shard_counts.assign(p.shard_count, 0);
  DGDS_CUDA(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
  DGDS_CUDA(cudaEventCreateWithFlags(&s->staging_free, cudaEventDisableTiming));
  DGDS_CUDA(cudaStreamCreateWithFlags(&s->copy_st, cudaStreamNonBlocking));
  DGDS_CUDA(cudaStreamCreateWithFlags(&s->out_st, cudaStreamNonBlocking));
  for (auto& q : s->qslot) DGDS_CUDA(cudaEventCreateWithFlags(&q.done, cudaEventDisableTiming));
  for (int c = 0; c < dgds_server::kMaxQChunks; ++c) {
    DGDS_CUDA(cudaEventCreateWithFlags(&s->ev_h2d[c], cudaEventDisableTiming));
    DGDS_CUDA(cudaEventCreateWithFlags(&s->ev_cmp[c], cudaEventDisableTiming));
  }
  if (const char* e = std::getenv("DGDS_Q_CHUNKS"))
    s->q_chunks = std::min(dgds_server::kMaxQChunks, std::max(1, std::atoi(e)));
  s->out_blocks = s->h2d_blocks;
  if (const char* e = std::getenv("DGDS_OUT_BLOCKS")) s->out_blocks = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("DGDS_ASYNC_STAGE")) s->async_stage = std::atoi(e) != 0;
  if (const char* e = std::getenv("DGDS_STAGE_TASKS")) s->stage_tasks = std::max(1, std::atoi(e));
  const uint64_t nodes = p.expected_nodes ? p.expected_nodes : (1ull << 20);
  double init_load = 0.35;  // expected_nodes is an upper bound, so the real load starts lower
  if (const char* e = std::getenv("DGDS_INIT_LOAD")) init_load = std::min(0.9, std::max(0.05, std::atof(e)));
  uint64_t cap = std::min(cap_for(nodes, init_load), kMaxCap);  // both multiples of the probe window
  s->T.cap = cap;
  s->T.depth_cap = s->D;
  s->T.lim_pattern = p.max_pattern_len;
  s->T.lim_spec = p.max_spec_len;
  s->T.ahead = 0;  // the bulk L2 prefetch measured slower than the register preload alone
  if (const char* e = std::getenv("DGDS_PREFETCH_AHEAD")) s->T.ahead = std::max(0, std::atoi(e));
  s->T.dbg = nullptr;
  if (std::getenv("DGDS_APPEND_DBG")) {  // debug: per-warp K1 timing, read with dgds_debug_append_timing
    DGDS_CUDA(cudaMalloc(&s->T.dbg, 65536 * 2 * sizeof(unsigned long long)));
    DGDS_CUDA(cudaMemset(s->T.dbg, 0, 65536 * 2 * sizeof(unsigned long long)));
  }
  s->T.claim_cas = 1;  // CAS-first claim (measured faster: fewer random accesses per insert)
  if (const char* e = std::getenv("DGDS_CLAIM")) s->T.claim_cas = std::strcmp(e, "load") == 0 ? 0 : 1;
  DGDS_CUDA(cudaMalloc(&s->T.slots, cap * sizeof(dgds::Slot)));
  DGDS_CUDA(cudaMemsetAsync(s->T.slots, 0, cap * sizeof(dgds::Slot), s->st));
  DGDS_CUDA(cudaMalloc(&s->d_used, dgds::kUsedParts * 8 * sizeof(unsigned long long)));
  DGDS_CUDA(cudaMemsetAsync(s->d_used, 0, dgds::kUsedParts * 8 * sizeof(unsigned long long), s->st));
  s->T.used = s->d_used;
  s->stream_cap = std::max<uint64_t>(p.expected_streams ? p.expected_streams : 4096, 64);
  DGDS_CUDA(cudaMalloc(&s->T.active, s->stream_cap * dgds::kWarp * sizeof(uint32_t)));
  DGDS_CUDA(cudaMalloc(&s->T.tail, s->stream_cap * dgds::kWarp * sizeof(int32_t)));
  DGDS_CUDA(cudaMalloc(&s->d_err, sizeof(int32_t)));
  DGDS_CUDA(cudaMemsetAsync(s->d_err, 0, sizeof(int32_t), s->st));
  s->hist_cap = std::max<uint64_t>(1ull << 20, nodes / 20);  // ~ tokens (nodes per token ~ 17-24)
  DGDS_CUDA(cudaMalloc(&s->d_hist, s->hist_cap * sizeof(int32_t)));
  s->T.hist = s->d_hist;
  DGDS_CUDA(cudaMalloc(&s->d_stat_part, dgds::kStatParts * 8 * sizeof(unsigned long long)));
  DGDS_CUDA(cudaMemsetAsync(s->d_stat_part, 0, dgds::kStatParts * 8 * sizeof(unsigned long long), s->st));
  s->root_of_cap = 1024;
  DGDS_CUDA(cudaMalloc(&s->d_root_of, s->root_of_cap * sizeof(uint32_t)));
  DGDS_CUDA(cudaMemsetAsync(s->d_root_of, 0, s->root_of_cap * sizeof(uint32_t), s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  *out = s.release();
  return DGDS_OK;
}

int dgds_destroy(dgds_server* s) {
  if (!s) return DGDS_OK;
  cudaSetDevice(s->p.device);
  flush_pending(s);  // a staged batch: its workers finish, its kernels run
  if (s->st) cudaStreamSynchronize(s->st);
  if (s->out_st) cudaStreamSynchronize(s->out_st);
  if (s->copy_st) cudaStreamSynchronize(s->copy_st);
  cudaFree(s->T.slots);
  cudaFree(s->T.active);
  cudaFree(s->T.tail);
  cudaFree(s->d_used);
  cudaFree(s->d_root_of);
  cudaFree(s->d_err);
  cudaFree(s->d_stat_part);
  cudaFree(s->d_hist);
  free_plan_pool(s);
  if (s->staging_free) cudaEventDestroy(s->staging_free);
  for (auto& q : s->qslot)
    if (q.done) cudaEventDestroy(q.done);
  if (s->copy_st) cudaStreamDestroy(s->copy_st);
  for (int c = 0; c < dgds_server::kMaxQChunks; ++c) {
    if (s->ev_h2d[c]) cudaEventDestroy(s->ev_h2d[c]);
    if (s->ev_cmp[c]) cudaEventDestroy(s->ev_cmp[c]);
  }
  if (s->out_st) cudaStreamDestroy(s->out_st);
  for (auto e : s->ev_pool) cudaEventDestroy(e);
  for (auto& v : s->ev_pending)
    for (auto& pr : v) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  if (s->st) cudaStreamDestroy(s->st);
  delete s;
  return DGDS_OK;
}

void* dgds_cuda_stream(dgds_server* s) { return s ? static_cast<void*>(s->st) : nullptr; }

int dgds_intern(dgds_server* s, const char* gid, size_t len, int32_t* handle) {
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  std::string key(gid, len);
  auto it = s->intern.find(key);
  if (it != s->intern.end()) {
    *handle = it->second;
    return DGDS_OK;
  }
  const int32_t h = static_cast<int32_t>(s->groups.size());
  GroupRec g;
  g.gid = key;
  g.shard = static_cast<int32_t>(fnv1a64(gid, len) % static_cast<uint64_t>(s->p.shard_count));
  s->groups.push_back(std::move(g));
  s->intern.emplace(std::move(key), h);
  *handle = h;
  return DGDS_OK;
}

int dgds_register_group(dgds_server* s, int32_t h, double ttl, double now) {  // dgds.cpp:99-110
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  if (int rc = check_handle(s, h)) return rc;
  if (!(ttl > 0.0)) return fail(DGDS_EINVAL, "register_group: ttl_seconds must be > 0");
  cudaSetDevice(s->p.device);
  GroupRec& g = s->groups[h];
  if (!live_entry(s, g, now)) return create_group(s, g, ttl, now);
  g.ttl = ttl;
  g.expires = now + ttl;
  return DGDS_OK;
}

}  // extern "C"
namespace {
int maybe_compact(dgds_server* s);  // memory reclamation, below
}  // namespace
extern "C" {

int dgds_drop_group(dgds_server* s, int32_t h) {  // dgds.cpp:112-116
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  if (int rc = check_handle(s, h)) return rc;
  cudaSetDevice(s->p.device);
  retire_group(s, s->groups[h]);
  return maybe_compact(s);
}

int dgds_sweep_expired(dgds_server* s, double now) {  // dgds.cpp:118-128
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  cudaSetDevice(s->p.device);
  for (auto& g : s->groups)
    if (g.alive && g.expires < now) retire_group(s, g);
  return maybe_compact(s);
}

int dgds_has_group(dgds_server* s, int32_t h, int32_t* out) {
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  if (int rc = check_handle(s, h)) return rc;
  *out = s->groups[h].alive ? 1 : 0;
  return DGDS_OK;
}

int dgds_group_version(dgds_server* s, int32_t h, uint64_t* out) {
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  if (int rc = check_handle(s, h)) return rc;
  *out = s->groups[h].alive ? s->groups[h].version : 0;
  return DGDS_OK;
}

int dgds_stored_tokens(dgds_server* s, int32_t h, int32_t rid, uint64_t* out) {
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  if (int rc = check_handle(s, h)) return rc;
  GroupRec& g = s->groups[h];
  StreamRec* r = g.streams.find(rid);
  *out = (g.alive && r) ? r->stored : 0;
  return DGDS_OK;
}

int dgds_shard_group_count(dgds_server* s, int32_t shard, uint64_t* out) {
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  if (shard < 0 || shard >= s->p.shard_count) return fail(DGDS_EINVAL, "bad shard");
  *out = s->shard_counts[shard];
  return DGDS_OK;
}

int dgds_index_slots(dgds_server* s, uint64_t* slots) {
  if (!s || !slots) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  *slots = s->T.cap;
  return DGDS_OK;
}

int dgds_node_count(dgds_server* s, uint64_t* out) {
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  cudaSetDevice(s->p.device);
  uint64_t u = 0;
  if (int rc = read_used(s, &u)) return rc;
  s->used_ub = u;
  // + group roots, matching nodes_.size() (root counted) per live group
  uint64_t roots = 0;
  for (const auto& g : s->groups) roots += g.alive ? 1 : 0;
  *out = u + roots;
  return DGDS_OK;
}

}  // extern "C"

// dgds_update_batch without the lock (also the replica path of dgds_apply_blob)
static int update_batch_locked(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids,
                               const uint64_t* prev, const uint64_t* offs, const int32_t* tokens, double now,
                               dgds_update_reply* rep) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  PhaseClock pc("update_batch");
  DGDS_CUDA(cudaSetDevice(s->p.device));
  const uint64_t ntok = offs[n] - offs[0];
  {
    int32_t any = 0;  // branch-free sign scan (vectorised)
    for (uint64_t i = offs[0]; i < offs[n]; ++i) any |= tokens[i];
    if (any < 0) return fail(DGDS_EINVAL, "negative token");
  }
  std::vector<dgds::AppendSeg>& segs = s->scratch.segs;
  std::vector<dgds::AppendPiece>& pieces = s->scratch.pieces;
  uint64_t worst = 0;
  if (int rc = plan_updates(s, n, handles, rids, prev, offs, nullptr, now, rep, segs, pieces, &worst)) return rc;
  pc.mark("plan");
  if (segs.empty()) return DGDS_OK;
  if (int rc = ensure_capacity(s, worst)) return rc;
  if (int rc = ensure_hist(s)) return rc;
  // one pinned staging block -> one H2D copy: segs | pieces | tokens
  const size_t b_seg = segs.size() * sizeof(dgds::AppendSeg);
  const size_t o_piece = align_up(b_seg, 256);
  const size_t b_piece = pieces.size() * sizeof(dgds::AppendPiece);
  const size_t o_tok = align_up(o_piece + b_piece, 256);
  const size_t total = o_tok + ntok * sizeof(int32_t);
  DGDS_CUDA(cudaEventSynchronize(s->staging_free));
  if (int rc = s->h_stage.ensure(total)) return rc;
  if (int rc = s->d_stage.ensure(total)) return rc;
  char* h = static_cast<char*>(s->h_stage.p);
  for (auto& pc : pieces) pc.tok_off -= offs[0];
  nt_copy(h, segs.data(), b_seg);
  nt_copy(h + o_piece, pieces.data(), b_piece);
  nt_copy(h + o_tok, tokens + offs[0], ntok * sizeof(int32_t));
  _mm_sfence();
  char* d = static_cast<char*>(s->d_stage.p);
  pc.mark("stage");
  if (int rc = flush_pending(s)) return rc;  // K1 after the query batch submitted before it
  DGDS_CUDA(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s->st));
  DGDS_CUDA(cudaEventRecord(s->staging_free, s->st));
  {
    LaunchTimer lt(s, 0, s->st);
    DGDS_CUDA(dgds::launch_append(s->T, reinterpret_cast<const dgds::AppendSeg*>(d),
                                  static_cast<int64_t>(segs.size()), reinterpret_cast<const dgds::AppendPiece*>(d + o_piece),
                                  reinterpret_cast<const int32_t*>(d + o_tok), s->st));
  }
  s->used_ub += worst;
  return DGDS_OK;
}

extern "C" int dgds_update_batch(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids,
                                 const uint64_t* prev, const uint64_t* offs, const int32_t* tokens, double now,
                                 dgds_update_reply* rep) {
  if (!s) return fail(DGDS_EINVAL, "null server");
  std::lock_guard<std::mutex> lk(s->mu);  // a pending query batch is flushed at the first device work
  return update_batch_locked(s, n, handles, rids, prev, offs, tokens, now, rep);
}

extern "C" {

}  // extern "C"

// A planned device update: host bookkeeping done (replies final), device work pending.
struct dgds_update_plan {
  std::vector<dgds::AppendSeg> segs;
  std::vector<dgds::AppendPiece> pieces;
  const int32_t* d_tokens = nullptr;
  uint64_t seq = 0;
};

static void free_plan_pool(dgds_server* s) {
  for (auto* pl : s->plan_pool) delete pl;
  s->plan_pool.clear();
}

// Host half: validation, bookkeeping (replies, versions, history log), capacity. Plans must be
// launched in the order they were made (K1 of a later plan reads the stream rows K1 of an
// earlier one writes), which dgds_update_launch checks.
static int plan_device(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids, const uint64_t* prev,
                       const uint64_t* offs, const uint64_t* counts, const int32_t* d_tokens, double now,
                       dgds_update_reply* rep, dgds_update_plan* plan) {
  uint64_t worst = 0;
  if (int rc = plan_updates(s, n, handles, rids, prev, offs, counts, now, rep, plan->segs, plan->pieces, &worst))
    return rc;
  if (plan->segs.empty()) return DGDS_OK;
  if (int rc = ensure_capacity(s, worst)) return rc;
  if (int rc = ensure_hist(s)) return rc;
  s->used_ub += worst;  // at plan time: a later plan's capacity check must see pending inserts
  plan->d_tokens = d_tokens;
  plan->seq = ++s->plans_made;
  return DGDS_OK;
}

// Device half: stage the segment/piece tables, H2D, K1 — stream-ordered on `stream`.
static int launch_plan(dgds_server* s, dgds_update_plan* plan, void* stream, PhaseClock& pc) {
  if (plan->segs.empty()) return DGDS_OK;
  if (plan->seq != s->plans_launched + 1) return fail(DGDS_ESTATE, "update plans must be launched in the order made");
  s->plans_launched = plan->seq;
  StreamJoin join(s, stream);
  const size_t b_seg = plan->segs.size() * sizeof(dgds::AppendSeg);
  const size_t o_piece = align_up(b_seg, 256);
  const size_t total = o_piece + plan->pieces.size() * sizeof(dgds::AppendPiece);
  DGDS_CUDA(cudaEventSynchronize(s->staging_free));
  pc.mark("staging_wait");
  if (int rc = s->h_stage.ensure(total)) return rc;
  if (int rc = s->d_stage.ensure(total)) return rc;
  char* h = static_cast<char*>(s->h_stage.p);
  nt_copy(h, plan->segs.data(), b_seg);
  nt_copy(h + o_piece, plan->pieces.data(), plan->pieces.size() * sizeof(dgds::AppendPiece));
  _mm_sfence();
  pc.mark("stage");
  char* d = static_cast<char*>(s->d_stage.p);
  DGDS_CUDA(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, join.stream()));
  DGDS_CUDA(cudaEventRecord(s->staging_free, join.stream()));
  {
    LaunchTimer lt(s, 0, join.stream());
    DGDS_CUDA(dgds::launch_append(s->T, reinterpret_cast<const dgds::AppendSeg*>(d),
                                  static_cast<int64_t>(plan->segs.size()),
                                  reinterpret_cast<const dgds::AppendPiece*>(d + o_piece), plan->d_tokens,
                                  join.stream()));
  }
  pc.mark("copy_launch");
  return DGDS_OK;
}

static int update_device_impl(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids, const uint64_t* prev,
                       const uint64_t* offs, const uint64_t* counts, const int32_t* d_tokens, double now,
                       dgds_update_reply* rep, void* stream) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  PhaseClock pc("update_device");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  thread_local dgds_update_plan plan;
  plan.segs.clear();
  plan.pieces.clear();
  if (int rc = plan_device(s, n, handles, rids, prev, offs, counts, d_tokens, now, rep, &plan)) return rc;
  pc.mark("plan");
  return launch_plan(s, &plan, stream, pc);
}

extern "C" {

int dgds_update_batch_device(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids,
                             const uint64_t* prev, const uint64_t* offs, const int32_t* d_tokens, double now,
                             dgds_update_reply* rep, void* stream) {
  return update_device_impl(s, n, handles, rids, prev, offs, nullptr, d_tokens, now, rep, stream);
}

int dgds_update_batch_device_strided(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids,
                                     const uint64_t* prev, const uint64_t* tok_starts, const uint64_t* tok_counts,
                                     const int32_t* d_tokens, double now, dgds_update_reply* rep, void* stream) {
  return update_device_impl(s, n, handles, rids, prev, tok_starts, tok_counts, d_tokens, now, rep, stream);
}

}  // extern "C"

// Unpack routed append rows (host metadata) into update arrays; returns the record count.
static int routed_arrays(int32_t n_seg, int64_t seg_rows, const int32_t* h_counts, const int32_t* h_meta,
                         int32_t meta_stride, int32_t row_words, int64_t* out_n) {
  if (!h_counts || !h_meta || n_seg < 1 || seg_rows < 0 || meta_stride < 5 || row_words < 6)
    return fail(DGDS_EINVAL, "bad routed append arguments");
  int64_t n = 0;
  for (int g = 0; g < n_seg; ++g) {
    if (h_counts[g] < 0 || h_counts[g] > seg_rows) return fail(DGDS_EINVAL, "segment count out of range");
    n += h_counts[g];
  }
  *out_n = n;
  return DGDS_OK;
}

namespace {
struct RoutedScratch {  // built before the server lock is taken: per thread, capacity kept
  std::vector<int32_t> handles, rids;
  std::vector<uint64_t> prev, starts, counts;
  std::vector<dgds_update_reply> rep;
};
int fill_routed(RoutedScratch& r, int64_t n, int32_t n_seg, int64_t seg_rows, const int32_t* h_counts,
                const int32_t* h_meta, int32_t meta_stride, int32_t row_words) {
  r.handles.resize(n);
  r.rids.resize(n);
  r.prev.resize(n);
  r.starts.resize(n);
  r.counts.resize(n);
  r.rep.resize(n);
  int64_t i = 0;
  for (int g = 0; g < n_seg; ++g) {
    for (int64_t j = 0; j < h_counts[g]; ++j, ++i) {
      const int64_t row = g * seg_rows + j;
      const int32_t* m = h_meta + row * meta_stride;
      r.handles[i] = m[0];
      r.rids[i] = m[1];
      r.prev[i] = static_cast<uint64_t>(static_cast<uint32_t>(m[2])) |
                  (static_cast<uint64_t>(static_cast<uint32_t>(m[3])) << 32);
      const int32_t cnt = m[4];
      if (cnt < 0 || cnt > row_words - 5) return fail(DGDS_EINVAL, "routed append token count out of range");
      r.counts[i] = static_cast<uint64_t>(cnt);
      r.starts[i] = static_cast<uint64_t>(row) * row_words + 5;
    }
  }
  return DGDS_OK;
}
}  // namespace

extern "C" {

int dgds_update_batch_routed(dgds_server* s, int32_t n_seg, int64_t seg_rows, const int32_t* h_counts,
                             const int32_t* h_meta, int32_t meta_stride, const int32_t* d_rows, int32_t row_words,
                             double now, int64_t* n_rejected, void* stream) {
  if (!s || !d_rows) return fail(DGDS_EINVAL, "bad routed append arguments");
  int64_t n = 0;
  if (int rc = routed_arrays(n_seg, seg_rows, h_counts, h_meta, meta_stride, row_words, &n)) return rc;
  if (n_rejected) *n_rejected = 0;
  if (n == 0) return DGDS_OK;
  thread_local RoutedScratch r;
  if (int rc = fill_routed(r, n, n_seg, seg_rows, h_counts, h_meta, meta_stride, row_words)) return rc;
  if (int rc = update_device_impl(s, n, r.handles.data(), r.rids.data(), r.prev.data(), r.starts.data(),
                                  r.counts.data(), d_rows, now, r.rep.data(), stream))
    return rc;
  if (n_rejected) {
    int64_t bad = 0;
    for (int64_t k = 0; k < n; ++k) bad += r.rep[k].ok ? 0 : 1;
    *n_rejected = bad;
  }
  return DGDS_OK;
}

int dgds_update_plan_routed(dgds_server* s, int32_t n_seg, int64_t seg_rows, const int32_t* h_counts,
                            const int32_t* h_meta, int32_t meta_stride, const int32_t* d_rows, int32_t row_words,
                            double now, int64_t* n_rejected, dgds_update_plan** out) {
  if (!s || !d_rows || !out) return fail(DGDS_EINVAL, "bad routed append arguments");
  *out = nullptr;
  int64_t n = 0;
  if (int rc = routed_arrays(n_seg, seg_rows, h_counts, h_meta, meta_stride, row_words, &n)) return rc;
  if (n_rejected) *n_rejected = 0;
  std::unique_ptr<dgds_update_plan> plan;
  {
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc_ = flush_pending(s)) return rc_;
    if (!s->plan_pool.empty()) {
      plan.reset(s->plan_pool.back());
      s->plan_pool.pop_back();
    }
  }
  if (!plan) plan = std::make_unique<dgds_update_plan>();
  plan->segs.clear();
  plan->pieces.clear();
  plan->d_tokens = nullptr;
  plan->seq = 0;
  if (n > 0) {
    thread_local RoutedScratch r;
    if (int rc = fill_routed(r, n, n_seg, seg_rows, h_counts, h_meta, meta_stride, row_words)) return rc;
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc_ = flush_pending(s)) return rc_;
    DGDS_CUDA(cudaSetDevice(s->p.device));
    if (int rc = plan_device(s, n, r.handles.data(), r.rids.data(), r.prev.data(), r.starts.data(), r.counts.data(),
                             d_rows, now, r.rep.data(), plan.get()))
      return rc;
    if (n_rejected) {
      int64_t bad = 0;
      for (int64_t k = 0; k < n; ++k) bad += r.rep[k].ok ? 0 : 1;
      *n_rejected = bad;
    }
  }
  *out = plan.release();
  return DGDS_OK;
}

int dgds_update_launch(dgds_server* s, dgds_update_plan* plan, void* stream) {
  if (!s || !plan) return fail(DGDS_EINVAL, "null argument");
  PhaseClock pc("update_launch");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  const cudaError_t e = cudaSetDevice(s->p.device);
  const int rc = e == cudaSuccess ? launch_plan(s, plan, stream, pc)
                                  : fail(DGDS_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  s->plan_pool.push_back(plan);  // recycled (the staging copy above does not keep references)
  return rc;
}

int dgds_copy_rows_d2h(void* h_dst, int64_t dst_pitch, const void* d_src, int64_t src_pitch, int64_t width,
                       int64_t rows, void* stream) {
  if (rows < 0 || width < 0 || (rows > 0 && (!h_dst || !d_src)) || dst_pitch < width || src_pitch < width)
    return fail(DGDS_EINVAL, "bad strided copy");
  if (rows == 0 || width == 0) return DGDS_OK;
  DGDS_CUDA(cudaMemcpy2DAsync(h_dst, dst_pitch, d_src, src_pitch, width, rows, cudaMemcpyDeviceToHost,
                              stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy));
  return DGDS_OK;
}

}  // extern "C"

namespace {

// One host-buffer query batch: its results live in the mapped pinned block of its slot
// (valid until the batch submitted kQSlots later reuses the slot).
struct HostResult {
  int64_t n = 0, ncand = 0, ntok = 0;
  const int64_t* cand_off = nullptr;  // [n + 1]
  const dgds::CandMeta* meta = nullptr;  // [ncand], candidate_before order within a query
  const int64_t* tok_off = nullptr;   // [ncand + 1]
  const int32_t* tokens = nullptr;    // [ntok]
  const int32_t* verify = nullptr;    // [3][n] drafted | accepted | emitted, or null
};

// Stage queries [j0, j1) of chunk b (chunk-relative) into its pinned block: pattern rows are
// built in cache, then streamed out with non-temporal stores.
// Returns the first query of the range with a bad handle (>= ng) or decreasing offsets, or -1.
int64_t stage_rows(const QInBlock& b, char* hb, int64_t j0, int64_t j1, int32_t P, int64_t ng, const int32_t* handles,
                   const uint64_t* pat_offs, const int32_t* patterns, const int32_t* truth, int32_t truth_stride,
                   const int32_t* truth_left, const int32_t* limit, bool verify) {
  if (j0 >= j1) return -1;
  int64_t bad = -1;
  const int64_t q0 = b.q0 + j0;
  int32_t* hl = reinterpret_cast<int32_t*>(hb + b.o_len);
  int32_t* hp = reinterpret_cast<int32_t*>(hb + b.o_pat);
  thread_local std::vector<int32_t> lens, rows;
  lens.resize(j1 - j0);
  rows.assign(static_cast<size_t>(j1 - j0) * P, 0);
  for (int64_t j = j0; j < j1; ++j) {
    const int64_t i = b.q0 + j;
    const int32_t hd = handles[i];
    if ((hd < 0 || hd >= ng || pat_offs[i + 1] < pat_offs[i]) && bad < 0) bad = i;
    const uint64_t L = pat_offs[i + 1] - pat_offs[i];
    lens[j - j0] = static_cast<int32_t>(std::min<uint64_t>(L, 0x7FFFFFFF));
    const uint64_t keep = std::min<uint64_t>(L, static_cast<uint64_t>(P));
    const int32_t* src = patterns + pat_offs[i + 1] - keep;
    int32_t* dst = rows.data() + (j - j0) * P;
    for (uint64_t k = 0; k < keep; ++k) dst[k] = src[k];
  }
  nt_copy(hl + j0, lens.data(), (j1 - j0) * 4);
  nt_copy(hp + j0 * P, rows.data(), rows.size() * 4);
  nt_copy(hb + j0 * 4, handles + q0, (j1 - j0) * 4);
  if (verify) {
    nt_copy(hb + b.o_tr + static_cast<size_t>(j0) * truth_stride * 4, truth + q0 * truth_stride,
            static_cast<size_t>(j1 - j0) * truth_stride * 4);
    nt_copy(hb + b.o_tl + j0 * 4, truth_left + q0, (j1 - j0) * 4);
    nt_copy(hb + b.o_lm + j0 * 4, limit + q0, (j1 - j0) * 4);
  }
  _mm_sfence();  // streaming stores globally visible before the copy is issued
  return bad;
}

// Issue the H2D of every chunk of the pending batch (from the worker that staged last).
// The batch's H2D, one copy per chunk block (per-row copies queued by each stager measured
// slower: many small copies from several threads), from the worker that staged last; then the
// per-chunk events the query launches wait on.
cudaError_t issue_h2d(dgds_server* s) {
  dgds_server::PendingQuery& pq = s->pq;
  dgds_server::QSlot& slot = s->qslot[pq.ticket % dgds_server::kQSlots];
  char* h = static_cast<char*>(slot.hq.p);
  char* d = static_cast<char*>(slot.dq.p);
  cudaError_t e = cudaSetDevice(s->p.device);
  for (int c = 0; c < pq.nch && e == cudaSuccess; ++c) {
    const QInBlock& b = pq.blk[c];
    if (s->h2d_kernel) {  // the GPU pulls the mapped staging block
      dgds::CopyOutRegions Rin{};
      Rin.n = 1;
      Rin.total_idx[0] = -1;
      Rin.begin_idx[0] = -1;
      Rin.fixed_bytes[0] = static_cast<int64_t>(b.bytes);
      Rin.src[0] = h + b.base;
      Rin.dst[0] = d + b.base;
      // a narrow grid: enough reads in flight for PCIe, SMs left to the append kernel running beside it
      e = dgds::launch_copy_out(nullptr, Rin, Rin.fixed_bytes[0], s->copy_st, s->h2d_blocks);
    } else {
      e = cudaMemcpyAsync(d + b.base, h + b.base, b.bytes, cudaMemcpyHostToDevice, s->copy_st);
    }
    if (e == cudaSuccess) e = cudaEventRecord(s->ev_h2d[c], s->copy_st);
  }
  return e;
}

// Check the arguments, then stage (and validate handles / offsets) on the worker pool without
// waiting: the caller's next host work (typically the next tick's dgds_update_batch planning)
// overlaps the staging. The worker that stages last issues the H2D and launches the kernels;
// any later call that touches the device first joins it (flush_pending), so every batch sees
// exactly the updates launched before it. Caller holds s->mu.
int speculate_submit(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                     const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride, const int32_t* truth,
                     int32_t truth_stride, const int32_t* truth_left, const int32_t* limit, bool verify,
                     uint64_t* ticket) {
  PhaseClock pc("speculate_submit");
  if (int rc = flush_pending(s)) return rc;
  const int64_t nargs = args_stride ? n : 1;
  int32_t max_k = 1, max_s = 1;
  for (int64_t i = 0; i < nargs; ++i) {
    const dgds_spec_args& a = args[i * args_stride];
    if (int rc = check_args(a)) return rc;
    max_k = std::max(max_k, a.top_k);
    max_s = std::max(max_s, std::min(a.max_spec_tokens, s->p.max_spec_len));
  }
  if (verify && (!truth || !truth_left || !limit || truth_stride < 0))
    return fail(DGDS_EINVAL, "verify needs truth inputs");
  pc.mark("args");
  const int32_t P = s->p.max_pattern_len;  // only the last max_pattern_len tokens can matter
  dgds_server::PendingQuery& pq = s->pq;
  // optional chunks of the batch (DGDS_Q_CHUNKS): chunk c's copy-out beside chunk c+1's query
  int nch = n >= 32768 ? s->q_chunks : 1;
  const int64_t per = static_cast<int64_t>(align_up((n + nch - 1) / nch, 256));
  nch = static_cast<int>((n + per - 1) / per);
  size_t in_all = 0;
  for (int c = 0; c < nch; ++c) {  // per-chunk block: handles | pat_len | patterns | args | truth | truth_left | limit
    QInBlock& b = pq.blk[c];
    b.q0 = c * per;
    b.m = std::min<int64_t>(per, n - b.q0);
    b.base = in_all;
    b.o_len = align_up(b.m * 4, 256);
    b.o_pat = align_up(b.o_len + b.m * 4, 256);
    b.o_args = align_up(b.o_pat + static_cast<size_t>(b.m) * P * 4, 256);
    b.o_tr = align_up(b.o_args + (args_stride ? b.m : 1) * sizeof(dgds_spec_args), 256);
    b.o_tl = align_up(b.o_tr + (verify ? static_cast<size_t>(b.m) * truth_stride * 4 : 0), 256);
    b.o_lm = align_up(b.o_tl + (verify ? b.m * 4 : 0), 256);
    b.bytes = align_up(b.o_lm + (verify ? b.m * 4 : 0), 16);  // the copy-in kernel moves 16-B units
    in_all = align_up(b.base + b.bytes, 256);
  }
  const uint64_t tk = s->last_ticket + 1;
  dgds_server::QSlot& slot = s->qslot[tk % dgds_server::kQSlots];
  DGDS_CUDA(cudaEventSynchronize(slot.done));  // the slot's previous batch is complete
  slot.ticket = 0;  // its results are gone from here on
  pc.mark("slot_wait");
  // device outputs (internal strides) + compaction scratch; mapped result block
  const int32_t K = max_k, Sx = max_s;
  const int64_t nk = static_cast<int64_t>(n) * K;
  QOutLayout& o = pq.out;
  o.sc = 0;
  o.sp = align_up(o.sc + nk * 8, 256);
  o.nc = align_up(o.sp + nk * 8, 256);
  o.ln = align_up(o.nc + n * 4, 256);
  o.tk = align_up(o.ln + nk * 4, 256);
  o.v = align_up(o.tk + static_cast<size_t>(nk) * Sx * 4, 256);
  o.bs = align_up(o.v + (verify ? static_cast<size_t>(n) * 12 : 0), 256);
  o.tot = align_up(o.bs + static_cast<size_t>((per + 255) / 256) * 16, 256);
  o.cmeta = align_up(o.tot + static_cast<size_t>(nch) * 16, 256);
  o.ctoff = align_up(o.cmeta + nk * sizeof(dgds::CandMeta), 256);
  o.ccoff = align_up(o.ctoff + nk * 8, 256);
  o.ctok = align_up(o.ccoff + (n + 1) * 8, 256);
  const size_t dev_total = o.ctok + static_cast<size_t>(nk) * Sx * 4;
  slot.h_coff = 256;  // totals | cand_off | verify | meta | tok_off | tokens
  slot.h_v = align_up(slot.h_coff + (n + 1) * 8, 256);
  slot.h_meta = align_up(slot.h_v + (verify ? n * 12 : 0), 256);
  slot.h_toff = align_up(slot.h_meta + nk * sizeof(dgds::CandMeta), 256);
  slot.h_tok = align_up(slot.h_toff + (nk + 1) * 8, 256);
  if (int rc = slot.hq.ensure(in_all)) return rc;
  if (int rc = slot.dq.ensure(in_all)) return rc;
  if (int rc = slot.dout.ensure(dev_total)) return rc;
  if (int rc = slot.ho.ensure(slot.h_tok + static_cast<size_t>(nk) * Sx * 4)) return rc;
  char* h = static_cast<char*>(slot.hq.p);
  for (int c = 0; c < nch; ++c) {  // args: tiny, copied here
    const QInBlock& b = pq.blk[c];
    auto* ha = reinterpret_cast<dgds_spec_args*>(h + b.base + b.o_args);
    if (!args_stride) ha[0] = args[0];
    else
      for (int64_t j = 0; j < b.m; ++j) ha[j] = args[(b.q0 + j) * args_stride];
  }
  pq.n = n;
  pq.nch = nch;
  pq.K = K;
  pq.Sx = Sx;
  pq.args_stride = args_stride;
  pq.truth_stride = truth_stride;
  pq.verify = verify;
  pq.ticket = tk;
  pq.h2d_err = cudaSuccess;
  pq.handles = handles;
  pq.ng = static_cast<int64_t>(s->groups.size());
  pq.stager_launch = !s->profiling;  // LaunchTimer state belongs to the caller's thread
  pq.launched = false;
  pq.launch_rc = DGDS_OK;
  slot.ticket = tk;
  slot.err = DGDS_OK;
  slot.n = n;
  slot.verify = verify;
  s->last_ticket = tk;
  *ticket = tk;
  // stage (and validate) on the workers; tasks cover [0, n) and split at chunk boundaries. An
  // asynchronous stage uses a few workers: it overlaps the caller's next host work, which
  // would otherwise be starved of memory bandwidth.
  WorkerPool& pool = s->workers();
  const bool async = s->async_stage && n >= 8192 && pool.threads() > 1;
  const int tasks = n < 8192 ? 1 : async ? std::min(s->stage_tasks, pool.threads() - 1) : 4 * pool.threads();
  const int64_t span = (n + tasks - 1) / tasks;
  const int64_t ng = static_cast<int64_t>(s->groups.size());
  pq.left.store(tasks);
  pq.bad.store(INT64_MAX);
  auto job = [s, h, span, n, per, P, ng, handles, pat_offs, patterns, truth, truth_stride, truth_left, limit,
              verify](int t) {
    const int64_t i0 = t * span, i1 = std::min<int64_t>(n, i0 + span);
    int64_t first_bad = INT64_MAX;
    for (int64_t i = i0; i < i1;) {
      const int c = static_cast<int>(i / per);
      const QInBlock& b = s->pq.blk[c];
      const int64_t e = std::min<int64_t>(i1, b.q0 + b.m);
      const int64_t bad = stage_rows(b, h + b.base, i - b.q0, e - b.q0, P, ng, handles, pat_offs, patterns, truth,
                                     truth_stride, truth_left, limit, verify);
      if (bad >= 0 && bad < first_bad) first_bad = bad;
      i = e;
    }
    if (first_bad != INT64_MAX) {
      int64_t cur = s->pq.bad.load();
      while (first_bad < cur && !s->pq.bad.compare_exchange_weak(cur, first_bad)) {
      }
    }
    if (s->pq.left.fetch_sub(1) == 1 && s->pq.bad.load() == INT64_MAX) {  // the last stager
      dgds_server::PendingQuery& q = s->pq;  // (nothing is launched for an invalid batch)
      if (q.h2d_err == cudaSuccess) q.h2d_err = issue_h2d(s);
      if (q.h2d_err == cudaSuccess && q.stager_launch) {
        q.launch_rc = launch_batch(s, false);
        if (q.launch_rc) q.launch_msg = dgds_last_error();
        q.launched = true;
      }
    }
  };
  pq.active = true;
  if (async) {
    pool.post(tasks, job);  // a bad handle / offset is reported by the batch's wait
  } else {
    pool.run(tasks, job);
    if (pq.bad.load() != INT64_MAX) {  // staged here: report at submit, nothing was queued
      const int64_t i = pq.bad.load();
      pq.active = false;
      slot.ticket = 0;
      s->last_ticket = tk - 1;
      if (int rc = check_handle(s, handles[i])) return rc;
      return fail(DGDS_EINVAL, "pattern offsets must be nondecreasing");
    }
  }
  pc.mark("post");
  return DGDS_OK;
}

// Launch a staged batch's kernels (its H2D issued): query (+ verify), compaction, copy-out.
// Run by the worker that staged last, or by flush_pending when that worker could not (profiling
// timers are main-thread state). Reads server state that every main-thread mutation of it
// (root table, index table, stream and history arrays) first flushes, i.e. joins the worker.
int launch_batch(dgds_server* s, bool timed) {
  dgds_server::PendingQuery& pq = s->pq;
  dgds_server::QSlot& slot = s->qslot[pq.ticket % dgds_server::kQSlots];
  const QOutLayout& o = pq.out;
  const int64_t n = pq.n;
  const int32_t K = pq.K, Sx = pq.Sx, P = s->p.max_pattern_len;
  const bool verify = pq.verify;
  const int nch = pq.nch;
  char* d = static_cast<char*>(slot.dq.p);
  char* dout = static_cast<char*>(slot.dout.p);
  char* ho = static_cast<char*>(slot.ho.p);
  long long* d_bs = reinterpret_cast<long long*>(dout + o.bs);
  long long* d_tot = reinterpret_cast<long long*>(dout + o.tot);  // [chunk][candidates, tokens], cumulative
  auto* d_meta = reinterpret_cast<dgds::CandMeta*>(dout + o.cmeta);
  auto* d_toff = reinterpret_cast<int64_t*>(dout + o.ctoff);
  auto* d_coff = reinterpret_cast<int64_t*>(dout + o.ccoff);
  int32_t* d_ctok = reinterpret_cast<int32_t*>(dout + o.ctok);
  int32_t* d_v = reinterpret_cast<int32_t*>(dout + o.v);
  for (int c = 0; c < nch; ++c) {
    const QInBlock& b = pq.blk[c];
    const char* db = d + b.base;
    const int64_t q0 = b.q0, m = b.m;
    DGDS_CUDA(cudaStreamWaitEvent(s->st, s->ev_h2d[c], 0));
    dgds::QueryLaunch L{};
    L.T = s->T;
    L.root_of = s->d_root_of;
    L.n_handles = static_cast<int32_t>(s->root_of_cap);
    L.n = m;
    L.handles = reinterpret_cast<const int32_t*>(db);
    L.pat_len = reinterpret_cast<const int32_t*>(db + b.o_len);
    L.patterns = reinterpret_cast<const int32_t*>(db + b.o_pat);
    L.pat_stride = P;
    L.args = reinterpret_cast<const dgds_spec_args*>(db + b.o_args);
    L.args_stride = pq.args_stride ? 1 : 0;
    L.k_stride = K;
    L.s_stride = Sx;
    dgds::soa_strides(L);
    L.scores = reinterpret_cast<double*>(dout + o.sc) + q0 * K;
    L.supports = reinterpret_cast<int64_t*>(dout + o.sp) + q0 * K;
    L.n_cands = reinterpret_cast<int32_t*>(dout + o.nc) + q0;
    L.lens = reinterpret_cast<int32_t*>(dout + o.ln) + q0 * K;
    L.tokens = reinterpret_cast<int32_t*>(dout + o.tk) + q0 * K * Sx;
    L.err_flag = s->d_err;
    L.stat_part = s->d_stat_part;
    if (verify) {
      L.truth = reinterpret_cast<const int32_t*>(db + b.o_tr);
      L.truth_stride = pq.truth_stride;
      L.truth_left = reinterpret_cast<const int32_t*>(db + b.o_tl);
      L.limit = reinterpret_cast<const int32_t*>(db + b.o_lm);
      L.v_drafted = d_v + q0;
      L.v_accepted = d_v + n + q0;
      L.v_emitted = d_v + 2 * n + q0;
    }
    if (timed) {
      LaunchTimer lt(s, 1, s->st);
      DGDS_CUDA(dgds::launch_query(L, K, Sx, s->st));
    } else {
      DGDS_CUDA(dgds::launch_query(L, K, Sx, s->st));
    }
    DGDS_CUDA(dgds::launch_compact(m, K, Sx, L.n_cands, L.lens, L.scores, L.supports, L.tokens, d_bs, d_tot + 2 * c,
                                   d_meta, d_ctok, d_coff + q0, d_toff, c ? d_tot + 2 * (c - 1) : nullptr, s->st));
    DGDS_CUDA(cudaEventRecord(s->ev_cmp[c], s->st));
    DGDS_CUDA(cudaStreamWaitEvent(s->out_st, s->ev_cmp[c], 0));
    dgds::CopyOutRegions R{};
    auto region = [&](const void* src, char* dst, int tot, int begin, int elem, int64_t fixed) {
      const int i = R.n++;
      R.src[i] = static_cast<const char*>(src);
      R.dst[i] = dst;
      R.total_idx[i] = tot;
      R.begin_idx[i] = begin;
      R.elem_bytes[i] = elem;
      R.fixed_bytes[i] = fixed;
    };
    const int tc = 2 * c, tb = c ? 2 * (c - 1) : -1;
    region(d_coff + q0, ho + slot.h_coff + q0 * 8, -1, -1, 0, m * 8);
    if (verify)
      for (int k = 0; k < 3; ++k)
        region(d_v + k * n + q0, ho + slot.h_v + (k * n + q0) * 4, -1, -1, 0, m * 4);
    region(d_meta, ho + slot.h_meta, tc, tb, sizeof(dgds::CandMeta), 0);
    region(d_toff, ho + slot.h_toff, tc, tb, 8, 0);
    region(d_ctok, ho + slot.h_tok, tc + 1, c ? tb + 1 : -1, 4, 0);
    if (c == nch - 1) region(d_tot + tc, ho, -1, -1, 0, 16);
    DGDS_CUDA(dgds::launch_copy_out(d_tot, R, m * K * static_cast<int64_t>(sizeof(dgds::CandMeta) + 8 + Sx * 4),
                                    s->out_st, nch > 1 ? s->out_blocks : 592));
  }
  DGDS_CUDA(cudaEventRecord(slot.done, s->out_st));  // after st's work (out_st waited on it)
  return DGDS_OK;
}

// Completes the pending batch: joins its staging workers and, unless the last of them did,
// launches its kernels. Runs before any later call on the server touches the device.
// Caller holds s->mu.
int flush_pending(dgds_server* s) {
  dgds_server::PendingQuery& pq = s->pq;
  if (!pq.active) return DGDS_OK;
  PhaseClock pc("flush_pending");
  s->workers().join();
  pq.active = false;
  pc.mark("join");
  dgds_server::QSlot& slot = s->qslot[pq.ticket % dgds_server::kQSlots];
  if (pq.bad.load() != INT64_MAX) {  // reported by the batch's wait, not by the call that flushed
    const int64_t i = pq.bad.load();
    const int32_t hd = pq.handles[i];
    slot.err = DGDS_EINVAL;
    slot.err_msg = (hd < 0 || hd >= pq.ng) ? "bad group handle" : "pattern offsets must be nondecreasing";
    return DGDS_OK;
  }
  if (pq.h2d_err.load() != cudaSuccess) return fail(DGDS_ECUDA, cudaGetErrorString(pq.h2d_err.load()));
  if (pq.launched) {
    if (pq.launch_rc) return fail(pq.launch_rc, pq.launch_msg);
    return DGDS_OK;
  }
  const int rc = launch_batch(s, true);
  pc.mark("launch");
  return rc;
}

// Waits for a submitted batch and describes its results. Caller holds s->mu.
int speculate_finish(dgds_server* s, uint64_t ticket, HostResult* r) {
  if (ticket == 0 || ticket > s->last_ticket) return fail(DGDS_EINVAL, "unknown query ticket");
  if (s->pq.active && s->pq.ticket == ticket)  // waiting on the batch still being staged
    if (int rc = flush_pending(s)) return rc;
  {
    const dgds_server::QSlot& sl = s->qslot[ticket % dgds_server::kQSlots];
    if (sl.ticket == ticket && sl.err) return fail(sl.err, sl.err_msg);
  }
  dgds_server::QSlot& slot = s->qslot[ticket % dgds_server::kQSlots];
  if (slot.ticket != ticket) return fail(DGDS_EINVAL, "query ticket expired (its result slot was reused)");
  DGDS_CUDA(cudaEventSynchronize(slot.done));
  char* ho = static_cast<char*>(slot.ho.p);
  const int64_t n = slot.n;
  r->n = n;
  r->ncand = reinterpret_cast<const long long*>(ho)[0];
  r->ntok = reinterpret_cast<const long long*>(ho)[1];
  auto* coff = reinterpret_cast<int64_t*>(ho + slot.h_coff);
  auto* toff = reinterpret_cast<int64_t*>(ho + slot.h_toff);
  coff[n] = r->ncand;
  toff[r->ncand] = r->ntok;
  r->cand_off = coff;
  r->meta = reinterpret_cast<const dgds::CandMeta*>(ho + slot.h_meta);
  r->tok_off = toff;
  r->tokens = reinterpret_cast<const int32_t*>(ho + slot.h_tok);
  r->verify = slot.verify ? reinterpret_cast<const int32_t*>(ho + slot.h_v) : nullptr;
  s->last_d2h_bytes =
      16 + (n + 1) * 8 + (slot.verify ? n * 12 : 0) + r->ncand * (sizeof(dgds::CandMeta) + 8) + r->ntok * 4;
  return DGDS_OK;
}

int speculate_host(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                   const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride, const int32_t* truth,
                   int32_t truth_stride, const int32_t* truth_left, const int32_t* limit, bool verify,
                   HostResult* r) {
  uint64_t t = 0;
  if (int rc = speculate_submit(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride,
                                truth_left, limit, verify, &t))
    return rc;
  PhaseClock pc("speculate_wait");
  return speculate_finish(s, t, r);
}

}  // namespace

extern "C" {

int dgds_speculate_verify_batch(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                                const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                                const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                                const int32_t* limit, dgds_candidates* out, dgds_verify_out* vout) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  if (!out) return fail(DGDS_EINVAL, "null output");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  {
    const int64_t nargs = args_stride ? n : 1;
    int32_t max_k = 1, max_s = 1;
    for (int64_t i = 0; i < nargs; ++i) {
      if (int rc = check_args(args[i * args_stride])) return rc;
      max_k = std::max(max_k, args[i * args_stride].top_k);
      max_s = std::max(max_s, std::min(args[i * args_stride].max_spec_tokens, s->p.max_spec_len));
    }
    if (out->k_stride < max_k || out->s_stride < max_s)
      return fail(DGDS_EBUFFER, "candidate buffer strides too small");
  }
  HostResult r;
  if (int rc = speculate_host(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride, truth_left,
                              limit, vout != nullptr, &r))
    return rc;
  PhaseClock pc("scatter");
  // scatter into the caller's strided buffers, in parallel chunks (per-query offsets are known)
  WorkerPool& pool = s->workers();
  const int tasks = n >= 8192 ? 4 * pool.threads() : 1;
  const int64_t chunk = (n + tasks - 1) / tasks;
  pool.run(tasks, [&](int t) {
    const int64_t q0 = t * chunk, q1 = std::min<int64_t>(n, q0 + chunk);
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t c0 = r.cand_off[q], c1 = r.cand_off[q + 1];
      out->n_cands[q] = static_cast<int32_t>(c1 - c0);
      for (int64_t c = c0; c < c1; ++c) {
        const int64_t di = q * out->k_stride + (c - c0);
        const dgds::CandMeta& m = r.meta[c];
        out->lens[di] = m.len;
        out->scores[di] = m.score;
        out->supports[di] = m.support;
        std::memcpy(out->tokens + di * out->s_stride, r.tokens + r.tok_off[c], m.len * 4);
      }
    }
    if (vout && q0 < q1) {
      std::memcpy(vout->drafted + q0, r.verify + q0, (q1 - q0) * 4);
      std::memcpy(vout->accepted + q0, r.verify + n + q0, (q1 - q0) * 4);
      std::memcpy(vout->emitted + q0, r.verify + 2 * n + q0, (q1 - q0) * 4);
    }
  });
  return DGDS_OK;
}

}  // extern "C"

static void fill_view(const HostResult& r, dgds_result_view* out) {
  out->n_queries = r.n;
  out->n_cands = r.ncand;
  out->n_tokens = r.ntok;
  out->cand_off = r.cand_off;
  out->cands = reinterpret_cast<const dgds_cand_meta*>(r.meta);
  out->tok_off = r.tok_off;
  out->tokens = r.tokens;
  if (r.verify) {
    out->drafted = r.verify;
    out->accepted = r.verify + r.n;
    out->emitted = r.verify + 2 * r.n;
  }
}

extern "C" {

int dgds_speculate_verify_view(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                               const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                               const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                               const int32_t* limit, dgds_result_view* out) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (!out) return fail(DGDS_EINVAL, "null output");
  *out = dgds_result_view{};
  if (n == 0) return DGDS_OK;
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  HostResult r;
  if (int rc = speculate_host(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride, truth_left,
                              limit, truth != nullptr, &r))
    return rc;
  fill_view(r, out);
  return DGDS_OK;
}

int dgds_speculate_submit(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                          const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                          const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                          const int32_t* limit, uint64_t* ticket) {
  if (!s || !ticket) return fail(DGDS_EINVAL, "null argument");
  if (n <= 0) return fail(DGDS_EINVAL, "submit needs a non-empty batch");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  return speculate_submit(s, n, handles, pat_offs, patterns, args, args_stride, truth, truth_stride, truth_left,
                          limit, truth != nullptr, ticket);
}

int dgds_speculate_wait(dgds_server* s, uint64_t ticket, dgds_result_view* out) {
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  *out = dgds_result_view{};
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  DGDS_CUDA(cudaSetDevice(s->p.device));
  HostResult r;
  if (int rc = speculate_finish(s, ticket, &r)) return rc;
  fill_view(r, out);
  return DGDS_OK;
}

int dgds_replies_submit(dgds_server* s, int64_t n, const int32_t* d_replies, const dgds_query_record_layout* lay,
                        int32_t max_top_k, int32_t max_spec, void* stream, uint64_t* ticket) {
  if (!s || !lay || !d_replies || !ticket) return fail(DGDS_EINVAL, "null argument");
  if (n <= 0) return fail(DGDS_EINVAL, "submit needs a non-empty batch");
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (max_spec < 1) return fail(DGDS_EINVAL, "max_spec must be >= 1");
  const dgds_query_record_layout& y = *lay;
  if (y.reply_words < 1 || (y.reply_words & 1) || (y.off_scores & 1) || (y.off_supports & 1))
    return fail(DGDS_EINVAL, "bad record layout (reply words and 8-byte fields must be even)");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc = flush_pending(s)) return rc;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  const cudaStream_t js = join.stream();
  const uint64_t tk = s->last_ticket + 1;
  dgds_server::QSlot& slot = s->qslot[tk % dgds_server::kQSlots];
  DGDS_CUDA(cudaEventSynchronize(slot.done));  // the slot's previous batch is complete
  slot.ticket = 0;
  const bool verify = y.off_verify >= 0;
  const int32_t K = max_top_k, Sx = max_spec;
  const int64_t nk = n * K;
  // device: block sums | totals | meta | tok_off | cand_off | tokens | verify [3][n]
  const int64_t nblk = (n + 255) / 256;
  const size_t o_bs = 0;
  const size_t o_tot = align_up(o_bs + static_cast<size_t>(nblk) * 16, 256);
  const size_t o_cmeta = align_up(o_tot + 16, 256);
  const size_t o_ctoff = align_up(o_cmeta + nk * sizeof(dgds::CandMeta), 256);
  const size_t o_ccoff = align_up(o_ctoff + nk * 8, 256);
  const size_t o_ctok = align_up(o_ccoff + (n + 1) * 8, 256);
  const size_t o_v = align_up(o_ctok + static_cast<size_t>(nk) * Sx * 4, 256);
  const size_t dev_total = o_v + (verify ? n * 12 : 0);
  slot.h_coff = 256;  // totals | cand_off | verify | meta | tok_off | tokens
  slot.h_v = align_up(slot.h_coff + (n + 1) * 8, 256);
  slot.h_meta = align_up(slot.h_v + (verify ? n * 12 : 0), 256);
  slot.h_toff = align_up(slot.h_meta + nk * sizeof(dgds::CandMeta), 256);
  slot.h_tok = align_up(slot.h_toff + (nk + 1) * 8, 256);
  if (int rc = slot.dout.ensure(dev_total)) return rc;
  if (int rc = slot.ho.ensure(slot.h_tok + static_cast<size_t>(nk) * Sx * 4)) return rc;
  char* dout = static_cast<char*>(slot.dout.p);
  char* ho = static_cast<char*>(slot.ho.p);
  long long* d_bs = reinterpret_cast<long long*>(dout + o_bs);
  long long* d_tot = reinterpret_cast<long long*>(dout + o_tot);
  auto* d_meta = reinterpret_cast<dgds::CandMeta*>(dout + o_cmeta);
  auto* d_toff = reinterpret_cast<int64_t*>(dout + o_ctoff);
  auto* d_coff = reinterpret_cast<int64_t*>(dout + o_ccoff);
  int32_t* d_ctok = reinterpret_cast<int32_t*>(dout + o_ctok);
  int32_t* d_v = reinterpret_cast<int32_t*>(dout + o_v);
  dgds::CmpIn in{};  // reply records: int32 fields at stride reply_words, 8-byte fields at reply_words / 2
  in.n_cands = d_replies + y.off_n_cands;
  in.qs_nc = y.reply_words;
  in.lens = d_replies + y.off_lens;
  in.qs_len = y.reply_words;
  in.scores = reinterpret_cast<const double*>(d_replies + y.off_scores);
  in.qs_sc = y.reply_words / 2;
  in.supports = reinterpret_cast<const int64_t*>(d_replies + y.off_supports);
  in.qs_sp = y.reply_words / 2;
  in.tokens = d_replies + y.off_tokens;
  in.qs_tok = y.reply_words;
  in.cs_tok = max_spec;
  in.verify = verify ? d_replies + y.off_verify : nullptr;
  in.qs_v = y.reply_words;
  DGDS_CUDA(dgds::launch_compact_in(n, in, d_bs, d_tot, d_meta, d_ctok, d_coff, d_toff, verify ? d_v : nullptr,
                                    nullptr, js));
  // the copy-out (PCIe-bound) runs on out_st, so the caller's stream moves on
  DGDS_CUDA(cudaEventRecord(s->ev_cmp[0], js));
  DGDS_CUDA(cudaStreamWaitEvent(s->out_st, s->ev_cmp[0], 0));
  dgds::CopyOutRegions R{};
  auto region = [&](const void* src, char* dst, int tot, int elem, int64_t fixed) {
    const int i = R.n++;
    R.src[i] = static_cast<const char*>(src);
    R.dst[i] = dst;
    R.total_idx[i] = tot;
    R.begin_idx[i] = -1;
    R.elem_bytes[i] = elem;
    R.fixed_bytes[i] = fixed;
  };
  region(d_coff, ho + slot.h_coff, -1, 0, n * 8);
  if (verify) region(d_v, ho + slot.h_v, -1, 0, n * 12);
  region(d_meta, ho + slot.h_meta, 0, sizeof(dgds::CandMeta), 0);
  region(d_toff, ho + slot.h_toff, 0, 8, 0);
  region(d_ctok, ho + slot.h_tok, 1, 4, 0);
  region(d_tot, ho, -1, 0, 16);
  DGDS_CUDA(dgds::launch_copy_out(d_tot, R, nk * static_cast<int64_t>(sizeof(dgds::CandMeta) + 8 + Sx * 4),
                                  s->out_st));
  DGDS_CUDA(cudaEventRecord(slot.done, s->out_st));
  slot.ticket = tk;
  slot.n = n;
  slot.verify = verify;
  slot.err = DGDS_OK;
  s->last_ticket = tk;
  *ticket = tk;
  return DGDS_OK;
}

int dgds_speculate_batch(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                         const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                         dgds_candidates* out) {
  return dgds_speculate_verify_batch(s, n, handles, pat_offs, patterns, args, args_stride, nullptr, 0, nullptr,
                                     nullptr, out, nullptr);
}

int dgds_speculate_device(dgds_server* s, int64_t n, const int32_t* d_handles, const int32_t* d_pat_len,
                          const int32_t* d_patterns, int32_t pat_stride, const dgds_spec_args* d_args,
                          int64_t args_stride, int32_t max_top_k, int32_t max_spec, const dgds_candidates* d_out,
                          const int32_t* d_truth, int32_t truth_stride, const int32_t* d_truth_left,
                          const int32_t* d_limit, const dgds_verify_out* d_vout, dgds_query_stats* d_stats,
                          void* stream) {
  if (max_spec <= 0 || max_spec > s->p.max_spec_len) max_spec = std::max(1, s->p.max_spec_len);
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (pat_stride < s->p.max_pattern_len) return fail(DGDS_EINVAL, "pat_stride must be >= max_pattern_len");
  if (d_out && (d_out->k_stride < max_top_k || d_out->s_stride < 1)) return fail(DGDS_EBUFFER, "bad output strides");
  if (d_vout && (!d_truth || !d_truth_left || !d_limit)) return fail(DGDS_EINVAL, "verify needs truth inputs");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  dgds::QueryLaunch L{};
  L.T = s->T;
  L.root_of = s->d_root_of;
  L.n_handles = static_cast<int32_t>(s->root_of_cap);
  L.n = n;
  L.handles = d_handles;
  L.pat_len = d_pat_len;
  L.patterns = d_patterns;
  L.pat_stride = pat_stride;
  L.args = d_args;
  L.args_stride = args_stride;
  if (d_out) {
    L.k_stride = d_out->k_stride;
    L.s_stride = d_out->s_stride;
    dgds::soa_strides(L);
    L.n_cands = d_out->n_cands;
    L.lens = d_out->lens;
    L.scores = d_out->scores;
    L.supports = d_out->supports;
    L.tokens = d_out->tokens;
  }
  L.in_qstride = 1;
  L.v_qstride = 1;
  if (d_vout) {
    L.truth = d_truth;
    L.truth_stride = truth_stride;
    L.truth_left = d_truth_left;
    L.limit = d_limit;
    L.v_drafted = d_vout->drafted;
    L.v_accepted = d_vout->accepted;
    L.v_emitted = d_vout->emitted;
  }
  L.stats = d_stats;
  L.err_flag = s->d_err;
  L.stat_part = s->d_stat_part;
  L.dbg = s->d_dbg;
  {
    LaunchTimer lt(s, 1, join.stream());
    DGDS_CUDA(dgds::launch_query(L, max_top_k, max_spec, join.stream()));
  }
  return DGDS_OK;
}

static int speculate_records_impl(dgds_server* s, int64_t n, const int32_t* d_records,
                                  const dgds_query_record_layout* lay, const dgds_spec_args* d_args,
                                  int64_t args_stride, int32_t max_top_k, int32_t max_spec, int32_t* d_replies,
                                  int32_t n_seg, int64_t seg_rows, const int32_t* d_seg_count,
                                  int32_t* const* seg_out, int32_t origin_field, dgds_query_stats* d_stats,
                                  void* stream) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  if (!lay || !d_records || !d_args || (!d_replies && !seg_out)) return fail(DGDS_EINVAL, "null argument");
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (max_spec <= 0 || max_spec > s->p.max_spec_len) max_spec = std::max(1, s->p.max_spec_len);
  const dgds_query_record_layout& y = *lay;
  if (y.rec_words < 1 || y.reply_words < 1 || (y.reply_words & 1) || (y.off_scores & 1) || (y.off_supports & 1))
    return fail(DGDS_EINVAL, "bad record layout (reply words and 8-byte fields must be even)");
  if (y.rec_words - y.off_pattern < s->p.max_pattern_len)
    return fail(DGDS_EINVAL, "query record pattern field shorter than max_pattern_len");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  dgds::QueryLaunch L{};
  L.T = s->T;
  L.root_of = s->d_root_of;
  L.n_handles = static_cast<int32_t>(s->root_of_cap);
  L.n = n;
  L.handles = d_records + y.off_handle;
  L.pat_len = d_records + y.off_pat_len;
  L.patterns = d_records + y.off_pattern;
  L.pat_stride = y.rec_words;
  L.args = d_args;
  L.args_stride = args_stride;
  L.k_stride = max_top_k;
  L.s_stride = max_spec;
  L.in_qstride = y.rec_words;
  L.rec_words_out = y.reply_words;
  L.rec_out = d_replies;
  if (seg_out) {
    L.seg_rows = seg_rows;
    L.seg_count = d_seg_count;
    if (origin_field >= 0) L.seg_origin = d_records + origin_field;
    for (int i = 0; i < n_seg; ++i) L.seg_out[i] = seg_out[i];
  }
  L.off_nc = y.off_n_cands;
  L.off_len = y.off_lens;
  L.off_sc = y.off_scores;
  L.off_sp = y.off_supports;
  L.off_tk = y.off_tokens;
  L.off_v = y.off_verify;
  if (y.off_verify >= 0) {
    L.truth = d_records + y.off_truth;
    L.truth_stride = y.rec_words;
    L.truth_left = d_records + y.off_truth_left;
    L.limit = d_records + y.off_limit;
  }
  L.stats = d_stats;
  L.err_flag = s->d_err;
  L.stat_part = s->d_stat_part;
  L.dbg = s->d_dbg;
  {
    LaunchTimer lt(s, 1, join.stream());
    DGDS_CUDA(dgds::launch_query(L, max_top_k, max_spec, join.stream()));
  }
  return DGDS_OK;
}

int dgds_speculate_records(dgds_server* s, int64_t n, const int32_t* d_records, const dgds_query_record_layout* lay,
                           const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k, int32_t max_spec,
                           int32_t* d_replies, dgds_query_stats* d_stats, void* stream) {
  return speculate_records_impl(s, n, d_records, lay, d_args, args_stride, max_top_k, max_spec, d_replies, 0, 0,
                                nullptr, nullptr, -1, d_stats, stream);
}

int dgds_speculate_records_seg(dgds_server* s, int32_t n_seg, int64_t seg_rows, const int32_t* d_records,
                               const int32_t* d_seg_count, const dgds_query_record_layout* lay,
                               const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k,
                               int32_t max_spec, int32_t* const* seg_out, int32_t origin_field,
                               dgds_query_stats* d_stats, void* stream) {
  if (n_seg < 1 || n_seg > dgds::kMaxSegments || seg_rows < 0) return fail(DGDS_EINVAL, "bad segment shape");
  if (lay && origin_field >= lay->rec_words) return fail(DGDS_EINVAL, "origin field outside the record");
  if (!d_seg_count || !seg_out) return fail(DGDS_EINVAL, "null argument");
  for (int i = 0; i < n_seg; ++i)
    if (!seg_out[i]) return fail(DGDS_EINVAL, "null segment output");
  return speculate_records_impl(s, static_cast<int64_t>(n_seg) * seg_rows, d_records, lay, d_args, args_stride,
                                max_top_k, max_spec, nullptr, n_seg, seg_rows, d_seg_count, seg_out, origin_field,
                                d_stats, stream);
}

int dgds_verify_batch(dgds_server* s, int64_t n, const dgds_candidates* c, const int32_t* truth, int32_t truth_stride,
                      const int32_t* truth_left, const int32_t* limit, dgds_verify_out* out) {
  if (n < 0) return fail(DGDS_EINVAL, "negative batch size");
  if (n == 0) return DGDS_OK;
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  const int K = c->k_stride, Sx = c->s_stride;
  const size_t o_ln = align_up(n * 4, 256);
  const size_t o_tk = align_up(o_ln + n * K * 4, 256);
  const size_t o_tr = align_up(o_tk + static_cast<size_t>(n) * K * Sx * 4, 256);
  const size_t o_tl = align_up(o_tr + static_cast<size_t>(n) * truth_stride * 4, 256);
  const size_t o_lm = align_up(o_tl + n * 4, 256);
  const size_t in_total = o_lm + n * 4;
  DGDS_CUDA(cudaEventSynchronize(s->staging_free));
  if (int rc = s->h_stage.ensure(in_total)) return rc;
  if (int rc = s->d_stage.ensure(in_total)) return rc;
  if (int rc = s->h_out.ensure(n * 12)) return rc;
  if (int rc = s->d_out.ensure(n * 12)) return rc;
  char* h = static_cast<char*>(s->h_stage.p);
  std::memcpy(h, c->n_cands, n * 4);
  std::memcpy(h + o_ln, c->lens, n * K * 4);
  std::memcpy(h + o_tk, c->tokens, static_cast<size_t>(n) * K * Sx * 4);
  std::memcpy(h + o_tr, truth, static_cast<size_t>(n) * truth_stride * 4);
  std::memcpy(h + o_tl, truth_left, n * 4);
  std::memcpy(h + o_lm, limit, n * 4);
  char* d = static_cast<char*>(s->d_stage.p);
  int32_t* dv = static_cast<int32_t*>(s->d_out.p);
  DGDS_CUDA(cudaMemcpyAsync(d, h, in_total, cudaMemcpyHostToDevice, s->st));
  DGDS_CUDA(cudaEventRecord(s->staging_free, s->st));
  DGDS_CUDA(dgds::launch_verify(n, K, Sx, reinterpret_cast<const int32_t*>(d), reinterpret_cast<const int32_t*>(d + o_ln),
                                reinterpret_cast<const int32_t*>(d + o_tk), reinterpret_cast<const int32_t*>(d + o_tr),
                                truth_stride, reinterpret_cast<const int32_t*>(d + o_tl),
                                reinterpret_cast<const int32_t*>(d + o_lm), dv, dv + n, dv + 2 * n, s->st));
  DGDS_CUDA(cudaMemcpyAsync(s->h_out.p, dv, n * 12, cudaMemcpyDeviceToHost, s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  const int32_t* hv = static_cast<const int32_t*>(s->h_out.p);
  std::memcpy(out->drafted, hv, n * 4);
  std::memcpy(out->accepted, hv + n, n * 4);
  std::memcpy(out->emitted, hv + 2 * n, n * 4);
  return DGDS_OK;
}

int32_t dgds_draft_len(int32_t sd_enabled, int32_t adaptive, int32_t cap, int32_t budget, int32_t n_running) {
  if (!sd_enabled) return 0;  // engine.cpp:78-85
  if (n_running < 1) n_running = 1;
  const int32_t d = adaptive ? std::min(cap, budget / n_running) : cap;
  return std::max(d, 0);
}

// Debug: record per-query phase cycles of device-API query launches into d_buf[n][8].
int dgds_debug_query_timing(dgds_server* s, void* d_buf) {
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  s->d_dbg = static_cast<long long*>(d_buf);
  return DGDS_OK;
}

int dgds_last_transfer(dgds_server* s, uint64_t* d2h_bytes) {
  *d2h_bytes = s->last_d2h_bytes;
  return DGDS_OK;
}

int dgds_profile_enable(dgds_server* s, int32_t on) {
  std::lock_guard<std::mutex> lk(s->mu);
  // host state only: no flush
  s->profiling = on != 0;
  return DGDS_OK;
}

int dgds_profile_read(dgds_server* s, dgds_profile* out, int32_t reset) {
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  for (int k = 0; k < 2; ++k) {
    for (auto& pr : s->ev_pending[k]) {
      DGDS_CUDA(cudaEventSynchronize(pr.second));
      float ms = 0.f;
      DGDS_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
      s->prof_ms[k] += ms;
      s->prof_launches[k] += 1;
      s->ev_pool.push_back(pr.first);
      s->ev_pool.push_back(pr.second);
    }
    s->ev_pending[k].clear();
  }
  out->append_launches = s->prof_launches[0];
  out->query_launches = s->prof_launches[1];
  out->append_ms = s->prof_ms[0];
  out->query_ms = s->prof_ms[1];
  if (reset) {
    s->prof_launches[0] = s->prof_launches[1] = 0;
    s->prof_ms[0] = s->prof_ms[1] = 0.0;
  }
  return DGDS_OK;
}

static DevBuf* route_scratch(cudaStream_t st, size_t bytes, int* rc);

int dgds_route_pack(int64_t n, int32_t world, const int32_t* d_owner, const uint32_t* d_records, int32_t rec_words,
                    uint32_t* d_out, int64_t* d_counts, int64_t* d_perm, void* stream) {
  if (world < 1 || world > 8) return fail(DGDS_EUNSUPPORTED, "route_pack supports 1..8 ranks");
  if (n < 0 || rec_words < 1) return fail(DGDS_EINVAL, "bad route_pack sizes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ntiles = std::max<int64_t>(1, (n + 1023) / 1024);
  int rc = 0;
  DevBuf* buf = route_scratch(st, ntiles * world * sizeof(int64_t), &rc);
  if (rc) return rc;
  cudaError_t e = dgds::launch_route_pack(n, world, d_owner, d_records, rec_words, d_out, d_counts, d_perm, buf->p, st);
  if (e != cudaSuccess) return fail(DGDS_ECUDA, cudaGetErrorString(e));
  return DGDS_OK;
}

int dgds_route_pack_padded(int64_t n, int32_t world, const int32_t* d_owner, const uint32_t* d_records,
                           int32_t rec_words, int64_t cap, uint32_t* d_out, int64_t* d_slot, int32_t* d_overflow,
                           void* stream) {
  if (world < 1 || world > 8) return fail(DGDS_EUNSUPPORTED, "route_pack supports 1..8 ranks");
  if (n < 0 || rec_words < 1 || cap < 1) return fail(DGDS_EINVAL, "bad route_pack sizes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ntiles = std::max<int64_t>(1, (n + 1023) / 1024);
  int rc = 0;
  DevBuf* buf = route_scratch(st, ntiles * world * sizeof(int64_t), &rc);
  if (rc) return rc;
  cudaError_t e = dgds::launch_route_pack_padded(n, world, d_owner, d_records, rec_words, cap, d_out, d_slot,
                                                 d_overflow, buf->p, st);
  if (e != cudaSuccess) return fail(DGDS_ECUDA, cudaGetErrorString(e));
  return DGDS_OK;
}

int dgds_route_unpack(int64_t n, const uint32_t* d_in, int32_t rec_words, const int64_t* d_perm, uint32_t* d_out,
                      void* stream) {
  DGDS_CUDA(dgds::launch_route_unpack(n, d_in, rec_words, d_perm, d_out, static_cast<cudaStream_t>(stream)));
  return DGDS_OK;
}

}  // extern "C"

// Grow-only routing scratch per (device, stream): calls on one stream are ordered,
// calls on different streams may overlap, so they never share a buffer.
static DevBuf* route_scratch(cudaStream_t st, size_t bytes, int* rc) {
  static std::mutex scratch_mu;
  static std::map<std::pair<int, cudaStream_t>, DevBuf> scratch;
  int dev = 0;
  cudaGetDevice(&dev);
  DevBuf* buf;
  {
    std::lock_guard<std::mutex> lk(scratch_mu);
    buf = &scratch[{dev, st}];
  }
  *rc = buf->ensure(bytes);
  return buf;
}

// ---------------------------------------------------------------------------
// Replica sync: GDX1 delta / full-snapshot blobs (GroupDraftIndex::delta_since /
// full_snapshot / apply_blob / compact_log, cst.cpp:233-329) and
// DraftServer::fetch_cst (dgds.cpp:53-97). Blobs are big-endian (bytes.hpp).
// The tokens come from the device history arena that K1 fills; the record
// framing and byte swap are done by k_blob_fill, the preamble on the host.

namespace {

constexpr uint8_t kBlobDelta = 1, kBlobFull = 2;

size_t blob_preamble_bytes(const std::string& gid) { return 4 + 1 + 2 + gid.size() + 8 + 8 + 4; }

void put_be(uint8_t*& p, uint64_t v, int bytes) {
  for (int b = bytes - 1; b >= 0; --b) *p++ = static_cast<uint8_t>(v >> (8 * b));
}

void write_preamble(uint8_t* p, uint8_t kind, const std::string& gid, uint64_t from, uint64_t to, uint32_t n) {
  *p++ = 'G';
  *p++ = 'D';
  *p++ = 'X';
  *p++ = '1';
  *p++ = kind;
  put_be(p, gid.size(), 2);
  std::memcpy(p, gid.data(), gid.size());
  p += gid.size();
  put_be(p, from, 8);
  put_be(p, to, 8);
  put_be(p, n, 4);
}

struct BlobReader {  // detail::ByteReader (bytes.hpp) over a caller buffer
  const uint8_t* p;
  const uint8_t* end;
  bool ok = true;
  uint64_t get(int bytes) {
    if (end - p < bytes) {
      ok = false;
      p = end;
      return 0;
    }
    uint64_t v = 0;
    for (int b = 0; b < bytes; ++b) v = (v << 8) | *p++;
    return v;
  }
  std::string str() {
    const uint64_t n = get(2);
    if (!ok || static_cast<uint64_t>(end - p) < n) {
      ok = false;
      return {};
    }
    std::string s(reinterpret_cast<const char*>(p), n);
    p += n;
    return s;
  }
};

}  // namespace

extern "C" {

int dgds_fetch_cst(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* cached, double now,
                   dgds_fetch_reply* rep, const uint8_t** blobs) {
  if (!s || n < 0 || (n > 0 && (!handles || !cached || !rep || !blobs))) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  for (int64_t i = 0; i < n; ++i)
    if (int rc = check_handle(s, handles[i])) return rc;
  std::vector<dgds::BlobPiece> pieces;
  struct Pre {
    int64_t i;
    uint8_t kind;
    uint64_t from, to;
    uint32_t count;
  };
  std::vector<Pre> pre;
  uint64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    GroupRec& g = s->groups[handles[i]];
    dgds_fetch_reply& r = rep[i];
    r = dgds_fetch_reply{};
    if (!live_entry(s, g, now)) {  // lazy expiry erases it (dgds.cpp:25-34)
      r.kind = DGDS_FETCH_UNKNOWN_GROUP;
      continue;
    }
    g.expires = now + g.ttl;
    const uint64_t cur = g.version, c = cached[i];
    r.version = cur;
    if (c == cur && c != 0) {
      r.kind = DGDS_FETCH_UP_TO_DATE;
      continue;
    }
    if (c == cur) {  // both 0: nothing appended yet, the reference answers UpToDate too
      r.kind = DGDS_FETCH_UP_TO_DATE;
      continue;
    }
    const bool delta = c != 0 && c < cur && c >= g.log_floor;  // else Full (stale, fresh or compacted)
    const uint64_t base = (total + 7) & ~7ull;
    uint64_t pos = base + blob_preamble_bytes(g.gid);
    if (delta) {
      const size_t first = g.delta_base + static_cast<size_t>(c - g.log_floor);
      for (size_t k = first; k < g.log.size(); ++k) {
        const LogRec& e = g.log[k];
        pos += 16;
        pieces.push_back(dgds::BlobPiece{e.off, pos, e.start, e.len, static_cast<uint32_t>(e.rid), 1, 0});
        pos += 4ull * e.len;
      }
      pre.push_back(Pre{i, kBlobDelta, c, cur, static_cast<uint32_t>(g.log.size() - first)});
    } else {
      // std::map order: request id ascending; a stream's tokens are its log entries in order
      std::vector<std::pair<int32_t, uint64_t>> st;  // (rid, stored)
      g.streams.for_each([&](int32_t rid, StreamRec& sr) { st.emplace_back(rid, sr.stored); });
      std::sort(st.begin(), st.end());
      std::vector<uint32_t> order(g.log.size());
      for (size_t k = 0; k < order.size(); ++k) order[k] = static_cast<uint32_t>(k);
      std::stable_sort(order.begin(), order.end(),
                       [&](uint32_t a, uint32_t b) { return g.log[a].rid < g.log[b].rid; });
      size_t o = 0;
      for (const auto& [rid, stored] : st) {
        pos += 12;
        while (o < order.size() && g.log[order[o]].rid < rid) ++o;  // (no stream without a record)
        bool first = true;
        for (; o < order.size() && g.log[order[o]].rid == rid; ++o) {
          const LogRec& e = g.log[order[o]];
          pieces.push_back(dgds::BlobPiece{e.off, pos, stored, e.len, static_cast<uint32_t>(rid), first ? 2u : 0u, 0});
          first = false;
          pos += 4ull * e.len;
        }
        if (first) pieces.push_back(dgds::BlobPiece{0, pos, 0, 0, static_cast<uint32_t>(rid), 2, 0});  // empty stream
      }
      pre.push_back(Pre{i, kBlobFull, 0, cur, static_cast<uint32_t>(st.size())});
    }
    r.kind = delta ? DGDS_FETCH_DELTA : DGDS_FETCH_FULL;
    r.blob_off = base;
    r.blob_len = pos - base;
    total = pos;
  }
  if (total == 0) {
    *blobs = static_cast<const uint8_t*>(s->h_blob.p);
    return DGDS_OK;
  }
  if (int rc = s->d_blob.ensure(total)) return rc;
  if (int rc = s->h_blob.ensure(total)) return rc;
  if (!pieces.empty()) {
    if (int rc = s->d_blob_pieces.ensure(pieces.size() * sizeof(dgds::BlobPiece))) return rc;
    DGDS_CUDA(cudaMemcpyAsync(s->d_blob_pieces.p, pieces.data(), pieces.size() * sizeof(dgds::BlobPiece),
                              cudaMemcpyHostToDevice, s->st));
    DGDS_CUDA(dgds::launch_blob_fill(static_cast<const dgds::BlobPiece*>(s->d_blob_pieces.p),
                                     static_cast<int64_t>(pieces.size()), s->d_hist,
                                     static_cast<uint8_t*>(s->d_blob.p), s->st));
  }
  DGDS_CUDA(cudaMemcpyAsync(s->h_blob.p, s->d_blob.p, total, cudaMemcpyDeviceToHost, s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  uint8_t* hb = static_cast<uint8_t*>(s->h_blob.p);
  for (const Pre& p : pre) {
    const GroupRec& g = s->groups[handles[p.i]];
    write_preamble(hb + rep[p.i].blob_off, p.kind, g.gid, p.from, p.to, p.count);
  }
  *blobs = hb;
  return DGDS_OK;
}

int dgds_compact_group(dgds_server* s, int32_t h, uint64_t before_version) {  // dgds.cpp:153-158, cst.cpp:324-329
  if (!s) return fail(DGDS_EINVAL, "null server");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  if (int rc = check_handle(s, h)) return rc;
  GroupRec& g = s->groups[h];
  if (!g.alive) return DGDS_OK;
  const uint64_t floor = std::min(before_version, g.version);
  if (floor <= g.log_floor) return DGDS_OK;
  g.delta_base += static_cast<size_t>(floor - g.log_floor);  // the entries stay: full snapshots need them
  g.log_floor = floor;
  return DGDS_OK;
}

int dgds_apply_blob(dgds_server* s, int32_t h, const uint8_t* blob, uint64_t len, double now, uint64_t* version) {
  if (!s || (!blob && len)) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  if (int rc = check_handle(s, h)) return rc;
  GroupRec& g = s->groups[h];
  BlobReader r{blob, blob + len};
  char magic[4];
  for (char& c : magic) c = static_cast<char>(r.get(1));
  if (!r.ok || std::memcmp(magic, "GDX1", 4) != 0) return fail(DGDS_EBLOB, "bad draft blob magic");
  const uint8_t kind = static_cast<uint8_t>(r.get(1));
  const std::string gid = r.str();
  if (!r.ok) return fail(DGDS_EBLOB, "truncated record");
  if (gid != g.gid) return fail(DGDS_EBLOB, "draft blob for group " + gid + " applied to " + g.gid);
  const uint64_t from = r.get(8), to = r.get(8);
  if (!r.ok) return fail(DGDS_EBLOB, "truncated record");
  if (!live_entry(s, g, now)) {  // a replica starts empty (version 0)
    if (int rc = create_group(s, g, s->p.default_ttl_seconds, now)) return rc;
  }
  g.expires = now + g.ttl;
  std::vector<int32_t> rids, toks;
  std::vector<uint64_t> prevs, offs{0};
  auto read_tokens = [&](uint64_t cnt) -> bool {
    if (static_cast<uint64_t>(r.end - r.p) / 4 < cnt) {
      r.ok = false;
      return false;
    }
    for (uint64_t k = 0; k < cnt; ++k) toks.push_back(static_cast<int32_t>(static_cast<uint32_t>(r.get(4))));
    return true;
  };
  if (kind == kBlobDelta) {
    if (from != g.version)
      return fail(DGDS_EBLOB, "delta expects replica at version " + std::to_string(from) + ", replica is at " +
                                  std::to_string(g.version));
    const uint64_t cnt = r.get(4);
    // entries apply in order; like the reference, stop at the first one out of order
    std::unordered_map<int32_t, uint64_t> stored;
    bool bad = false;
    for (uint64_t k = 0; k < cnt && r.ok; ++k) {
      const int32_t rid = static_cast<int32_t>(static_cast<uint32_t>(r.get(4)));
      const uint64_t start = r.get(8);
      const uint64_t n = r.get(4);
      if (!r.ok || !read_tokens(n)) break;
      auto it = stored.find(rid);
      if (it == stored.end()) {
        const StreamRec* sr = g.streams.find(rid);
        it = stored.emplace(rid, sr ? sr->stored : 0).first;
      }
      if (n > 0 && start != it->second) {  // append() would reply ok=false
        toks.resize(offs.back());
        bad = true;
        break;
      }
      it->second += n;
      rids.push_back(rid);
      prevs.push_back(start);
      offs.push_back(toks.size());
    }
    if (!r.ok && !bad) return fail(DGDS_EBLOB, "truncated record");
    std::vector<int32_t> hs(rids.size(), h);
    std::vector<dgds_update_reply> rep(rids.size());
    if (!rids.empty()) {
      if (int rc = update_batch_locked(s, static_cast<int64_t>(rids.size()), hs.data(), rids.data(), prevs.data(),
                                       offs.data(), toks.data(), now, rep.data()))
        return rc;
    }
    if (bad) return fail(DGDS_EBLOB, "delta entry out of order during apply");
    if (g.version != to) return fail(DGDS_EBLOB, "delta apply ended at unexpected version");
  } else if (kind == kBlobFull) {
    const uint64_t cnt = r.get(4);
    for (uint64_t k = 0; k < cnt && r.ok; ++k) {
      rids.push_back(static_cast<int32_t>(static_cast<uint32_t>(r.get(4))));
      const uint64_t n = r.get(8);
      if (!r.ok || !read_tokens(n)) break;
      prevs.push_back(0);
      offs.push_back(toks.size());
    }
    if (!r.ok) return fail(DGDS_EBLOB, "truncated record");
    // replace the replica: a fresh root, no streams, no history (cst.cpp:300-318)
    const double ttl = g.ttl;
    retire_group(s, g);
    if (int rc = create_group(s, g, ttl, now)) return rc;
    std::vector<int32_t> hs(rids.size(), h);
    std::vector<dgds_update_reply> rep(rids.size());
    if (!rids.empty()) {
      if (int rc = update_batch_locked(s, static_cast<int64_t>(rids.size()), hs.data(), rids.data(), prevs.data(),
                                       offs.data(), toks.data(), now, rep.data()))
        return rc;
    }
    g.version = to;  // a restored replica owns no history older than the snapshot
    g.delta_base = g.log.size();
    g.log_floor = to;
  } else {
    return fail(DGDS_EBLOB, "unknown draft blob kind");
  }
  if (version) *version = g.version;
  return DGDS_OK;
}

}  // extern "C"

extern "C" {

int dgds_batch_speculate_zc(dgds_server* s, int64_t n, const int32_t* d_handles, const int64_t* d_pat_end,
                            const int32_t* d_pat_len, const int32_t* d_pattern_buffer, const int64_t* d_out_offsets,
                            int32_t* d_output_buffer, const dgds_query_record_layout* lay,
                            const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k, int32_t max_spec,
                            dgds_query_stats* d_stats, void* stream) {
  if (!s || n < 0) return fail(DGDS_EINVAL, "bad batch");
  if (n == 0) return DGDS_OK;
  if (!d_handles || !d_pat_end || !d_pat_len || !d_pattern_buffer || !d_out_offsets || !d_output_buffer || !lay ||
      !d_args)
    return fail(DGDS_EINVAL, "null argument");
  if (max_top_k < 1 || max_top_k > DGDS_MAX_TOP_K) return fail(DGDS_EUNSUPPORTED, "max_top_k out of range");
  if (max_spec <= 0 || max_spec > s->p.max_spec_len) max_spec = std::max(1, s->p.max_spec_len);
  const dgds_query_record_layout& y = *lay;
  if (y.reply_words < 1 || (y.off_scores & 1) || (y.off_supports & 1))
    return fail(DGDS_EINVAL, "bad reply layout (8-byte fields must be even)");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  StreamJoin join(s, stream);
  dgds::QueryLaunch L{};
  L.T = s->T;
  L.root_of = s->d_root_of;
  L.n_handles = static_cast<int32_t>(s->root_of_cap);
  L.n = n;
  L.handles = d_handles;
  L.pat_len = d_pat_len;
  L.patterns = d_pattern_buffer;
  L.pat_end = d_pat_end;
  L.pat_stride = 0x7FFFFFFF;  // the pattern is read in place: no row clamp
  L.in_qstride = 1;
  L.args = d_args;
  L.args_stride = args_stride;
  L.k_stride = max_top_k;
  L.s_stride = max_spec;
  L.rec_words_out = y.reply_words;
  L.rec_out = d_output_buffer;
  L.out_off = d_out_offsets;
  L.off_nc = y.off_n_cands;
  L.off_len = y.off_lens;
  L.off_sc = y.off_scores;
  L.off_sp = y.off_supports;
  L.off_tk = y.off_tokens;
  L.off_v = -1;  // the engine verifies with the target model
  L.stats = d_stats;
  L.err_flag = s->d_err;
  L.stat_part = s->d_stat_part;
  L.dbg = s->d_dbg;
  {
    LaunchTimer lt(s, 1, join.stream());
    DGDS_CUDA(dgds::launch_query(L, max_top_k, max_spec, join.stream()));
  }
  return DGDS_OK;
}

}  // extern "C"

extern "C" int dgds_touch_group(dgds_server* s, int32_t h, double now) {  // update_cst before append (dgds.cpp:39-48)
  if (!s) return fail(DGDS_EINVAL, "null server");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  if (int rc = check_handle(s, h)) return rc;
  GroupRec& g = s->groups[h];
  if (!live_entry(s, g, now))
    if (int rc = create_group(s, g, s->p.default_ttl_seconds, now)) return rc;
  g.expires = now + g.ttl;
  return DGDS_OK;
}

// ---------------------------------------------------------------------------
// Memory reclamation: a same-capacity rebuild drops the
// slots of retired groups (rebuild keeps live roots only), and the history arena is
// compacted to the live groups' tokens by a gather kernel.

namespace {

int compact_history(dgds_server* s) {
  std::vector<dgds::CopyPiece> pcs;
  uint64_t live = 0;
  for (auto& g : s->groups) {
    if (!g.alive) continue;
    for (LogRec& e : g.log) {
      pcs.push_back(dgds::CopyPiece{e.off, live, e.len, 0});
      e.off = live;
      live += e.len;
    }
  }
  const uint64_t cap = std::max<uint64_t>(1ull << 20, live + live / 2);
  int32_t* nb = nullptr;
  if (cudaMalloc(&nb, cap * sizeof(int32_t)) != cudaSuccess) return fail(DGDS_ENOMEM, "history arena allocation failed");
  if (!pcs.empty()) {
    if (int rc = s->d_blob_pieces.ensure(pcs.size() * sizeof(dgds::CopyPiece))) return rc;
    DGDS_CUDA(cudaMemcpyAsync(s->d_blob_pieces.p, pcs.data(), pcs.size() * sizeof(dgds::CopyPiece),
                              cudaMemcpyHostToDevice, s->st));
    DGDS_CUDA(dgds::launch_copy_pieces(static_cast<const dgds::CopyPiece*>(s->d_blob_pieces.p),
                                       static_cast<int64_t>(pcs.size()), s->d_hist, nb, s->st));
  }
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  cudaFree(s->d_hist);
  s->d_hist = nb;
  s->T.hist = nb;
  s->hist_cap = cap;
  s->hist_used = live;
  s->dead_hist_tokens = 0;
  return DGDS_OK;
}

int compact_memory(dgds_server* s) {
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  if (int rc = rebuild(s, s->T.cap)) return rc;
  if (int rc = compact_history(s)) return rc;
  s->compactions += 1;
  return DGDS_OK;
}

// after explicit retirements: compact once retired groups hold > 40% of the history
int maybe_compact(dgds_server* s) {
  if (s->dead_hist_tokens < (1ull << 12) || s->dead_hist_tokens * 10 < s->hist_used * 4) return DGDS_OK;
  return compact_memory(s);
}

}  // namespace

extern "C" {

int dgds_compact_memory(dgds_server* s) {
  if (!s) return fail(DGDS_EINVAL, "null server");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  return compact_memory(s);
}

int dgds_get_memory_stats(dgds_server* s, dgds_memory_stats* out) {
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  uint64_t used = 0;
  if (int rc = read_used(s, &used)) return rc;
  s->used_ub = used;
  out->slots = s->T.cap;
  out->used_slots = used;
  out->history_capacity = s->hist_cap;
  out->history_tokens = s->hist_used;
  out->dead_history_tokens = s->dead_hist_tokens;
  out->compactions = s->compactions;
  return DGDS_OK;
}

}  // extern "C"

extern "C" int dgds_debug_append_timing(dgds_server* s, uint64_t* out, int64_t n_warps) {  // [n][2] start, end (ns)
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  if (!s->T.dbg) return fail(DGDS_ESTATE, "set DGDS_APPEND_DBG before dgds_create");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  DGDS_CUDA(cudaMemcpy(out, s->T.dbg, std::min<int64_t>(n_warps, 65536) * 16, cudaMemcpyDeviceToHost));
  return DGDS_OK;
}

// server_internal.h — types and helpers shared by the server translation units
// (server.cpp: lifecycle, groups, updates; host_query.cpp: host-buffer and record
// query paths; replica.cpp: GDX1 replica sync and memory reclamation). Internal:
// not part of the C ABI in include/dgds_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <sys/resource.h>
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

namespace dgds_host {

inline thread_local std::string g_err;

inline int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define DGDS_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(DGDS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline uint64_t fnv1a64(const void* data, size_t n) {  // detail::fnv1a64 (bytes.hpp:89-96)
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

// Capacity for a growing staging buffer: 2x, and 25% headroom over the request. Batch sizes
// vary a little from call to call (a cluster splits each batch by owner), and every regrowth
// costs a cudaFreeHost / cudaFree (device-synchronizing) plus pinning or mapping fresh pages
// (measured: 30-80 ms per 18 MB pinned block on the 4-GPU box, i.e. 10x a tick).
inline size_t grown_cap(size_t bytes, size_t cap) {
  const size_t c = std::max<size_t>(bytes + bytes / 4, cap * 2);
  return (c + 65535) & ~size_t(65535);
}

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
    const size_t c = grown_cap(bytes, cap);
    if (cudaHostAlloc(&p, c, flags) != cudaSuccess) {
      p = nullptr;
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
    const size_t c = grown_cap(bytes, cap);
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

inline int host_threads() {
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
  uint64_t sh_base = 0;  // token extent in the stream-history arena (dgds_server::d_shist)
  uint64_t sh_cap = 0;   // its capacity (tokens); a full extent moves to one twice as large
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

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Debug: DGDS_HOST_TIMING=1 prints the host-path phases of each call to stderr.
struct PhaseClock {  // DGDS_HOST_TIMING: per-phase wall time (us) and the thread's minor faults
  bool on;
  const char* name;
  std::chrono::steady_clock::time_point t0, last;
  long flt0 = 0, flt = 0;
  std::string line;
  static long faults() {
    rusage u{};
    getrusage(RUSAGE_THREAD, &u);
    return u.ru_minflt;
  }
  explicit PhaseClock(const char* n) : on(std::getenv("DGDS_HOST_TIMING") != nullptr), name(n) {
    if (on) {
      t0 = last = std::chrono::steady_clock::now();
      flt0 = flt = faults();
    }
  }
  void mark(const char* phase) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    const long f = faults();
    line += std::string(" ") + phase + "=" +
            std::to_string(std::chrono::duration<double, std::micro>(t - last).count()).substr(0, 7);
    if (f != flt) line += "(" + std::to_string(f - flt) + "f)";
    last = t;
    flt = f;
  }
  ~PhaseClock() {
    if (on)
      std::fprintf(stderr, "[%s] total=%.1fus faults=%ld%s\n", name,
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(),
                   faults() - flt0, line.c_str());
  }
};

// Copy into pinned staging memory with non-temporal (streaming) stores. A staging block
// written by several threads with normal stores, then read by the device (DMA or a pull
// kernel), measured 8 GB/s on the GPU box instead of 52 GB/s: the device reads snoop
// lines still dirty in the writers' caches (tools/h2d_dirty.cu). The caller fences.
inline void nt_copy(void* dst, const void* src, size_t n) {
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

}  // namespace dgds_host

struct dgds_server;
namespace dgds_host {
int speculate_view_indexed(dgds_server* s, int64_t n, const int64_t* idx, const int32_t* handles,
                           const uint64_t* pat_offs, const int32_t* patterns, const dgds_spec_args* args,
                           int64_t args_stride, const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                           const int32_t* limit, dgds_result_view* out);
int flush_pending(dgds_server* s);  // launches a submitted query batch; before any later device work
int launch_batch(dgds_server* s, bool timed);
// one chunk of a staged host query batch: handles | pat_len | patterns | args | truth | truth_left | limit
// a history-log record planned but not yet appended to its group's log (materialize_logs)
struct DeferredLog {
  int32_t handle;
  LogRec rec;
};
struct QInBlock {
  int64_t q0 = 0, m = 0;
  size_t base = 0, o_len = 0, o_pat = 0, o_args = 0, o_tr = 0, o_tl = 0, o_lm = 0, bytes = 0;
};
// device outputs of a host query batch (internal strides) + compaction scratch
struct QOutLayout {
  size_t sc = 0, sp = 0, nc = 0, ln = 0, tk = 0, v = 0, bs = 0, tot = 0, cmeta = 0, ctoff = 0, ccoff = 0, ctok = 0;
};
}  // namespace dgds_host

using namespace dgds_host;  // the server translation units share these internal types

struct dgds_server {
  dgds_params p{};
  int32_t D = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t staging_free[2] = {nullptr, nullptr};  // h_stage[k]'s last H2D is done
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
  // asynchronous routed planning (dgds_update_plan_routed_async / _take): one server-owned
  // planner thread runs the jobs in submission order, each after its metadata-ready event
  struct PlanJob;
  std::thread planner;
  std::mutex pj_mu;
  std::condition_variable pj_cv, pj_done_cv;
  std::deque<std::shared_ptr<PlanJob>> pj_queue;
  std::map<uint64_t, std::shared_ptr<PlanJob>> pj_jobs;
  uint64_t pj_next = 0;
  bool pj_stop = false;
  // plans whose history-log records are not yet in their groups' logs (device / routed update
  // plans append them after their K1 launch, off the routed critical path); creation order
  std::vector<struct dgds_update_plan*> log_pending;
  int64_t par_plan_min = INT64_MAX;  // DGDS_PARALLEL_PLAN=<min records>: plan by group partition on the workers
  bool async_stage = true;  // DGDS_ASYNC_STAGE=0: submit stages synchronously
  dgds::DevTrie T{};
  unsigned long long* d_used = nullptr;
  uint64_t used_ub = 0;  // upper bound on occupied slots since the last exact read

  int32_t* d_hist = nullptr;  // append-only token history (GDX1 blobs); k_stage fills it
  uint64_t hist_cap = 0, hist_used = 0;
  // per-stream token extents (queries and K1's conversion walks read continuations there)
  int32_t* d_shist = nullptr;
  uint64_t shist_cap = 0, shist_used = 0;
  uint64_t dead_shist_tokens = 0;  // extents that were moved or whose stream was retired
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
  // slots of retired streams: reusable only after a rebuild has dropped their groups' entries
  // (entries name their stream; a reused slot would make a dead entry look alive)
  std::vector<uint32_t> retired_streams;

  std::unordered_map<std::string, int32_t> intern;
  std::vector<GroupRec> groups;
  std::vector<uint64_t> shard_counts;
  uint64_t batch_stamp = 0;

  // update / verify staging, double-buffered so the host can plan a batch ahead of the last
  // one's H2D (the single buffer made tick s+1's plan wait for tick s's copy)
  PinnedBuf h_stage[2], h_out;  // h_out: dgds_verify_batch results
  int stage_k = 0;
  // device update plans (segment / piece tables), by h_stage parity: copied in on copy_st as
  // soon as staged, so the H2D runs under the previous batch's kernels instead of between them
  DevBuf d_plan[2];
  cudaEvent_t plan_ready[2] = {nullptr, nullptr};  // d_plan[k] copied in
  cudaEvent_t plan_free[2] = {nullptr, nullptr};   // K1 of the last plan in d_plan[k] enqueued before this
  DevBuf d_stage, d_out;
  bool h2d_kernel = false;  // copy-engine H2D (no SMs taken from K1); DGDS_H2D=kernel: a pull kernel
  int h2d_blocks = 148;    // one CTA per SM (measured best); DGDS_H2D_BLOCKS
  std::unique_ptr<WorkerPool> pool;
  int pool_threads = 0;  // host workers incl. the caller; 0 = host_threads() (a cluster splits the cores)
  uint64_t plans_made = 0, plans_launched = 0;  // two-phase device updates (plan now, launch later)
  std::vector<struct dgds_update_plan*> plan_pool;  // recycled plans: their vectors keep capacity
  // planning scratch, reused across calls (per-call vectors of 16-130 KB were page-faulting)
  struct PlanScratch {
    std::vector<dgds::AppendSeg> segs;
    std::vector<dgds::AppendPiece> pieces;
    std::vector<dgds::CopyPiece> grow;
    std::vector<uint32_t> cnt, fill;
  } scratch;
  WorkerPool& workers() {
    if (!pool) pool = std::make_unique<WorkerPool>((pool_threads > 0 ? pool_threads : host_threads()) - 1);
    return *pool;
  }
  int32_t* d_err = nullptr;
  DevBuf d_count;  // node-count reduction
  DevBuf d_cplx;   // K2a -> K2b queue (dgds::CplxRec per query of a launch)
  unsigned long long* d_cplx_count = nullptr;  // [0] queue length, [1] K2b warp ticket
  unsigned long long* d_step_acc = nullptr;    // engine decode step accumulators [4]
  DevBuf d_step_args;                          // dgds_decode_step_device's lookup args
  uint64_t ev_cap = 0;  // K1 conversion-event queue (T.ev)
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

namespace dgds_host {

// server.cpp
cudaEvent_t pooled_event(dgds_server* s);
int set_root(dgds_server* s, int32_t handle, uint32_t root);
int alloc_stream_slot(dgds_server* s, uint32_t* out);
void retire_group(dgds_server* s, GroupRec& g);
int create_group(dgds_server* s, GroupRec& g, double ttl, double now);
bool live_entry(dgds_server* s, GroupRec& g, double now);
int check_handle(dgds_server* s, int32_t h);
// appends every pending plan's history-log records to the group logs, in plan order; anything
// that reads or resets group logs calls it first
void materialize_logs(dgds_server* s);
int check_args(const dgds_spec_args& a);
int read_used(dgds_server* s, uint64_t* out);
int rebuild(dgds_server* s, uint64_t new_cap);
int ensure_capacity(dgds_server* s, uint64_t worst_new, uint64_t nseg = 0);
int ensure_hist(dgds_server* s);
int ensure_shist(dgds_server* s);
// replica.cpp
int compact_memory(dgds_server* s);
int maybe_compact(dgds_server* s);

// Brackets one kernel launch with events on its stream when profiling is on.
// The next host staging buffer (alternating): waits for its previous H2D, sizes it; the caller
// records *ev on the stream of its copy out of it.
inline int next_stage(dgds_server* s, size_t bytes, char** h, cudaEvent_t* ev) {
  const int k = s->stage_k ^= 1;
  DGDS_CUDA(cudaEventSynchronize(s->staging_free[k]));
  if (int rc = s->h_stage[k].ensure(bytes)) return rc;
  *h = static_cast<char*>(s->h_stage[k].p);
  *ev = s->staging_free[k];
  return DGDS_OK;
}

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

}  // namespace dgds_host

// server.cpp: dgds_update_batch without the lock (also the replica path of dgds_apply_blob)
int update_batch_locked(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids, const uint64_t* prev,
                        const uint64_t* offs, const int32_t* tokens, double now, dgds_update_reply* rep);

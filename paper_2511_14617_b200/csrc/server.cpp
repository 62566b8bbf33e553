// server.cpp — host side of the B200 DGDS: the extern "C" ABI declared in
// include/dgds_b200.h over the sm_100a kernels in kernels.cu. This unit holds the
// server lifecycle, groups and the update paths; the query paths are in host_query.cpp,
// replica sync and memory reclamation in replica.cpp (shared types: server_internal.h).
//
// Host work here is O(records) bookkeeping that the reference performs per
// call under its shard mutex (proj/src/dgds.cpp:36-51,99-138): group lookup
// with lazy TTL expiry, auto-registration, per-stream gap check and version
// numbering in call order (cst.cpp:118-133). Record replies are therefore
// final before any device work completes. All trie work — insertion, suffix
// match, beam, verification — runs on the GPU; there is no CPU fallback: a
// missing device is an error.

#include "server_internal.h"

static void free_plan_pool(dgds_server* s);  // after dgds_update_plan is complete
static void recycle_launched(dgds_server* s);
static void stop_planner(dgds_server* s);    // asynchronous routed planning, below

namespace dgds_host {

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

// Stream tables (active, ov: [stream][32] entry ids; sinfo: extent + length + root), zeroed
// beyond the old capacity: ids of never-written lanes read as 0 (remapped safely by a rebuild).
int grow_streams(dgds_server* s, uint64_t nc) {
  if (nc > static_cast<uint64_t>(dgds::kStreamMask) + 1) return fail(DGDS_EUNSUPPORTED, "request streams exhausted (2^24)");
  uint32_t *na = nullptr, *no = nullptr;
  dgds::StreamInfo* ni = nullptr;
  DGDS_CUDA(cudaMalloc(&na, nc * dgds::kWarp * sizeof(uint32_t)));
  DGDS_CUDA(cudaMalloc(&no, nc * dgds::kWarp * sizeof(uint32_t)));
  DGDS_CUDA(cudaMalloc(&ni, nc * sizeof(dgds::StreamInfo)));
  DGDS_CUDA(cudaMemsetAsync(na, 0, nc * dgds::kWarp * sizeof(uint32_t), s->st));
  DGDS_CUDA(cudaMemsetAsync(no, 0, nc * dgds::kWarp * sizeof(uint32_t), s->st));
  DGDS_CUDA(cudaMemsetAsync(ni, 0, nc * sizeof(dgds::StreamInfo), s->st));
  if (s->T.active) {
    DGDS_CUDA(cudaMemcpyAsync(na, s->T.active, s->stream_cap * dgds::kWarp * sizeof(uint32_t),
                              cudaMemcpyDeviceToDevice, s->st));
    DGDS_CUDA(cudaMemcpyAsync(no, s->T.ov, s->stream_cap * dgds::kWarp * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                              s->st));
    DGDS_CUDA(cudaMemcpyAsync(ni, s->T.sinfo, s->stream_cap * sizeof(dgds::StreamInfo), cudaMemcpyDeviceToDevice,
                              s->st));
    DGDS_CUDA(cudaStreamSynchronize(s->st));
    cudaFree(s->T.active);
    cudaFree(s->T.ov);
    cudaFree(s->T.sinfo);
  }
  s->T.active = na;
  s->T.ov = no;
  s->T.sinfo = ni;
  s->stream_cap = nc;
  s->T.stream_cap = nc;
  return DGDS_OK;
}

int alloc_stream_slot(dgds_server* s, uint32_t* out) {
  if (!s->free_streams.empty()) {
    *out = s->free_streams.back();
    s->free_streams.pop_back();
    return DGDS_OK;
  }
  if (s->next_stream >= s->stream_cap) {
    if (int rc = flush_pending(s)) return rc;  // the stream tables change under a staged batch's launch
    if (int rc = grow_streams(s, std::max<uint64_t>(1024, s->stream_cap * 2))) return rc;
  }
  *out = s->next_stream++;
  return DGDS_OK;
}

void retire_group(dgds_server* s, GroupRec& g) {
  if (!g.alive) return;
  materialize_logs(s);
  for (const LogRec& e : g.log) s->dead_hist_tokens += e.len;
  g.streams.for_each([&](int32_t, StreamRec& r) {
    s->retired_streams.push_back(r.slot);
    s->dead_shist_tokens += r.sh_cap;
  });
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
  materialize_logs(s);
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
  std::vector<uint32_t> rows;  // stream rows to remap: live streams, and retired ones (-> 0)
  for (auto& g : s->groups) {
    if (!g.alive) continue;
    const uint32_t r = dgds::kRootTop - g.root;
    alive[r >> 5] |= 1u << (r & 31);
    g.streams.for_each([&](int32_t, StreamRec& r) { rows.push_back(r.slot); });
  }
  rows.insert(rows.end(), s->retired_streams.begin(), s->retired_streams.end());
  uint32_t *d_alive = nullptr, *d_remap = nullptr, *d_rows = nullptr;
  DGDS_CUDA(cudaMalloc(&d_alive, alive.size() * 4));
  DGDS_CUDA(cudaMalloc(&d_remap, s->T.cap * 4));
  DGDS_CUDA(cudaMalloc(&d_rows, std::max<size_t>(1, rows.size()) * 4));
  DGDS_CUDA(cudaMemcpyAsync(d_alive, alive.data(), alive.size() * 4, cudaMemcpyHostToDevice, s->st));
  DGDS_CUDA(cudaMemsetAsync(d_remap, 0, s->T.cap * 4, s->st));
  if (!rows.empty())
    DGDS_CUDA(cudaMemcpyAsync(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, s->st));
  DGDS_CUDA(dgds::launch_rebuild(s->T, to, d_alive, d_remap, s->st));
  DGDS_CUDA(dgds::launch_remap_active(s->T, d_rows, static_cast<int64_t>(rows.size()), d_remap, s->st, s->T.cap));
  DGDS_CUDA(cudaStreamSynchronize(s->st));  // host vectors above must outlive the copies
  cudaFree(d_alive);
  cudaFree(d_remap);
  cudaFree(d_rows);
  cudaFree(s->T.slots);
  cudaFree(s->d_used);
  s->T.slots = to.slots;
  s->T.cap = new_cap;
  s->T.used = d_used_new;
  s->d_used = d_used_new;
  // retired streams' entries are gone: their slots may now serve new streams
  s->free_streams.insert(s->free_streams.end(), s->retired_streams.begin(), s->retired_streams.end());
  s->retired_streams.clear();
  return read_used(s, &s->used_ub);
}

// K1's conversion-event queue: at most one event per window occurrence of the batch; warps take
// slots in chunks of 32, so the slots used are <= 2 x events + 32 x warps (kernels.cu, K1 queue).
int ensure_events(dgds_server* s, uint64_t worst_new, uint64_t nseg) {
  const uint64_t need = 2 * worst_new + 32 * (nseg + 64);
  if (need <= s->ev_cap) return DGDS_OK;
  const uint64_t nc = std::max<uint64_t>(need, s->ev_cap * 2);
  dgds::WalkEvent* nb = nullptr;
  DGDS_CUDA(cudaStreamSynchronize(s->st));  // a launch in flight may still use the old queue
  if (cudaMalloc(&nb, nc * sizeof(dgds::WalkEvent)) != cudaSuccess) return fail(DGDS_ENOMEM, "event queue allocation failed");
  cudaFree(s->T.ev);
  s->T.ev = nb;
  s->ev_cap = nc;
  s->T.ev_cap = nc;
  return DGDS_OK;
}

int ensure_capacity(dgds_server* s, uint64_t worst_new, uint64_t nseg) {
  if (int rc = flush_pending(s)) return rc;  // a submitted query reads the table as it was
  if (int rc = ensure_events(s, worst_new, nseg)) return rc;
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
  uint64_t pos;  // stream position of the record's first token
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
  s->T.hist_cap = nc;
  s->T.hist = nb;
  return DGDS_OK;
}

// Grow the stream-history arena to hold shist_used tokens. Offsets are kept (the old arena is
// copied whole), so extents planned but not yet staged stay valid.
int ensure_shist(dgds_server* s) {
  if (s->shist_used <= s->shist_cap) return DGDS_OK;
  if (s->shist_used >= (1ull << 32)) return fail(DGDS_ENOMEM, "stream-history arena exceeds 2^32 tokens");
  if (int rc = flush_pending(s)) return rc;  // T.shist changes under a staged batch's launch
  const uint64_t nc = std::min<uint64_t>(std::max<uint64_t>(s->shist_used, s->shist_cap * 2), (1ull << 32) - 1);
  int32_t* nb = nullptr;
  if (cudaMalloc(&nb, nc * sizeof(int32_t)) != cudaSuccess) return fail(DGDS_ENOMEM, "stream-history allocation failed");
  if (s->d_shist) {
    DGDS_CUDA(cudaStreamSynchronize(s->st));  // appends in flight finish writing the old arena
    DGDS_CUDA(cudaMemcpy(nb, s->d_shist, s->shist_cap * sizeof(int32_t), cudaMemcpyDeviceToDevice));
    cudaFree(s->d_shist);
  }
  s->d_shist = nb;
  s->shist_cap = nc;
  s->T.shist_cap = nc;
  s->T.shist = nb;
  return DGDS_OK;
}

// Shared host logic of update_batch / update_batch_device: replies in call
// order (DraftServer::update_cst, dgds.cpp:36-51 -> GroupDraftIndex::append,
// cst.cpp:118-133), plus the device segment table.
// Record i's tokens are tokens[tok_start(i) .. tok_start(i) + tok_count(i)).
int plan_updates(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids, const uint64_t* prev,
                 const uint64_t* offs, const uint64_t* counts, double now, dgds_update_reply* rep,
                 std::vector<dgds::AppendSeg>& segs, std::vector<dgds::AppendPiece>& pieces,
                 std::vector<dgds::CopyPiece>& grow, uint64_t* worst, std::vector<DeferredLog>* defer = nullptr) {
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
  grow.clear();
  *worst = 0;
  // Records of different groups are independent (version, streams and log are per group), so
  // large batches are planned in parallel with the groups partitioned over the host workers;
  // each worker walks the batch in call order for its groups. Global state (group roots,
  // stream slots) is touched under one mutex — only when a group or stream is created.
  // Measured: the pool wake-up and cross-core traffic on group/stream records cost more than
  // the planning saves at bench sizes (4096 records: 0.34 -> 0.61 ms per step), so the parallel
  // path is opt-in (DGDS_PARALLEL_PLAN=<min records>).
  WorkerPool& pool = s->workers();
  const int W = (n >= s->par_plan_min && pool.threads() > 1) ? pool.threads() : 1;
  if (!defer || W > 1) materialize_logs(s);  // this plan appends to the group logs directly
  struct Part {
    std::vector<dgds::AppendSeg> segs;
    std::vector<std::pair<int32_t, int32_t>> srec;  // (group handle, request id) of each segment
    std::vector<dgds::CopyPiece> grow;
    std::vector<PendingPiece> pend;
    uint64_t worst = 0;
    int rc = DGDS_OK;
    std::string msg;
  };
  thread_local std::vector<Part> tl_parts;  // kept across calls: capacity persists
  // the workers must use the CALLER's instance: a thread_local named inside the lambda would
  // resolve to each worker's own (empty) one
  std::vector<Part>& parts = tl_parts;
  parts.resize(W);
  for (Part& P : parts) {
    P.segs.clear();
    P.srec.clear();
    P.grow.clear();
    P.pend.clear();
    P.worst = 0;
    P.rc = DGDS_OK;
  }
  std::mutex gmu;
  std::atomic<uint64_t> hist_at{s->hist_used};
  uint64_t hist_one = s->hist_used;
  std::atomic<uint64_t> shist_at{s->shist_used};
  std::atomic<uint64_t> shist_dead{0};
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
        P.srec.emplace_back(handles[i], rids[i]);  // not &sr: a later insert may move it
      }
      uint64_t hoff;
      if (W == 1) {  // single planner: no locked read-modify-write per record
        hoff = hist_one;
        hist_one += cnt;
      } else {
        hoff = hist_at.fetch_add(cnt, std::memory_order_relaxed);
      }
      P.pend.push_back(PendingPiece{sr.batch_seg, tstart(i), hoff, sr.stored, static_cast<uint32_t>(cnt)});
      if (defer && W == 1)  // appended to the group log after the plan's K1 launch
        defer->push_back(DeferredLog{handles[i], LogRec{hoff, sr.stored, static_cast<uint32_t>(cnt), rids[i]}});
      else
        g.log.push_back(LogRec{hoff, sr.stored, static_cast<uint32_t>(cnt), rids[i]});
      P.worst += worst_windows(sr.stored, cnt, static_cast<uint64_t>(s->D));
      sr.stored += cnt;
      g.version += 1;
      rep[i] = dgds_update_reply{1, 0, g.version, sr.stored};
    }
    // each segment's stream extent: a full one moves to one twice as large (its stored tokens
    // are copied on the device before the batch is staged)
    for (size_t k = 0; k < P.segs.size(); ++k) {
      dgds::AppendSeg& sg = P.segs[k];
      StreamRec& sr = *s->groups[P.srec[k].first].streams.find(P.srec[k].second);
      sg.n = static_cast<uint32_t>(sr.stored - sg.start);
      if (sr.stored > sr.sh_cap) {
        const uint64_t nc = (std::max<uint64_t>({sr.stored, sr.sh_cap * 2, 64}) + 7) / 8 * 8;
        const uint64_t nb = shist_at.fetch_add(nc, std::memory_order_relaxed);
        for (uint64_t c = 0; c < sg.start; c += 128)  // 128-token chunks: one warp each, one pass, in k_stage
          P.grow.push_back(dgds::CopyPiece{sr.sh_base + c, nb + c, static_cast<uint32_t>(std::min<uint64_t>(128, sg.start - c)), 0});
        shist_dead.fetch_add(sr.sh_cap, std::memory_order_relaxed);
        sr.sh_base = nb;
        sr.sh_cap = nc;
      }
      sg.sh_base = sr.sh_base;
    }
  };
  pcl.mark("validate_setup");
  if (W > 1) pool.run(W, work);
  else work(0);
  pcl.mark("records");
  s->hist_used = W == 1 ? hist_one : hist_at.load();
  s->shist_used = shist_at.load();
  s->dead_shist_tokens += shist_dead.load();
  for (const Part& P : parts)
    if (P.rc) return fail(P.rc, P.msg);
  for (const Part& P : parts) grow.insert(grow.end(), P.grow.begin(), P.grow.end());
  // merge the workers' segments (pieces are independent copies: k_stage)
  if (W == 1) {
    Part& P = parts[0];
    segs.swap(P.segs);  // P.segs is cleared before its next use; both buffers keep their capacity
    *worst = P.worst;
    pieces.resize(P.pend.size());
    for (size_t k = 0; k < P.pend.size(); ++k) {
      const PendingPiece& pp = P.pend[k];
      pieces[k] = dgds::AppendPiece{pp.tok_off, pp.hist_off, segs[pp.seg].sh_base + pp.pos, pp.n, 0};
    }
    pcl.mark("pieces");
    return DGDS_OK;
  }
  std::vector<int64_t> base(W + 1, 0);
  for (int w = 0; w < W; ++w) base[w + 1] = base[w] + static_cast<int64_t>(parts[w].segs.size());
  segs.reserve(base[W]);
  for (int w = 0; w < W; ++w) segs.insert(segs.end(), parts[w].segs.begin(), parts[w].segs.end());
  size_t npend = 0;
  for (int w = 0; w < W; ++w) {
    *worst += parts[w].worst;
    npend += parts[w].pend.size();
  }
  // pieces are independent copies (k_stage); K1 reads each segment from its stream extent
  pieces.resize(npend);
  size_t at = 0;
  for (int w = 0; w < W; ++w)
    for (const auto& pp : parts[w].pend)
      pieces[at++] = dgds::AppendPiece{pp.tok_off, pp.hist_off, segs[base[w] + pp.seg].sh_base + pp.pos, pp.n, 0};
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

}  // namespace dgds_host

namespace dgds {
int set_error(int code, const std::string& msg) { return fail(code, msg); }  // shared with peer.cu
}  // namespace dgds

extern "C" {

const char* dgds_last_error(void) { return g_err.c_str(); }
const char* dgds_version_string(void) { return "dgds-b200 0.1 (sm_100a)"; }

uint64_t dgds_kernel_launches(void) { return dgds::g_kernel_launches.load(std::memory_order_relaxed); }

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
  for (auto& e : s->staging_free) DGDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : s->plan_ready) DGDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : s->plan_free) DGDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
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
  if (const char* e = std::getenv("DGDS_PARALLEL_PLAN")) s->par_plan_min = std::max<int64_t>(1, std::atoll(e));
  const uint64_t nodes = p.expected_nodes ? p.expected_nodes : (1ull << 20);
  double init_load = 0.35;  // expected_nodes is an upper bound, so the real load starts lower
  if (const char* e = std::getenv("DGDS_INIT_LOAD")) init_load = std::min(0.9, std::max(0.05, std::atof(e)));
  uint64_t cap = std::min(cap_for(nodes, init_load), kMaxCap);  // both multiples of the probe window
  s->T.cap = cap;
  s->T.depth_cap = s->D;
  s->T.lim_pattern = p.max_pattern_len;
  s->T.lim_spec = p.max_spec_len;
  s->T.dbg = nullptr;
  if (std::getenv("DGDS_APPEND_DBG")) {  // debug: per-warp K1 timing, read with dgds_debug_append_timing
    DGDS_CUDA(cudaMalloc(&s->T.dbg, 65536 * 2 * sizeof(unsigned long long)));
    DGDS_CUDA(cudaMemset(s->T.dbg, 0, 65536 * 2 * sizeof(unsigned long long)));
  }
  DGDS_CUDA(cudaMalloc(&s->T.slots, cap * sizeof(dgds::Slot)));
  DGDS_CUDA(cudaMemsetAsync(s->T.slots, 0, cap * sizeof(dgds::Slot), s->st));
  DGDS_CUDA(cudaMalloc(&s->d_used, dgds::kUsedParts * 8 * sizeof(unsigned long long)));
  DGDS_CUDA(cudaMemsetAsync(s->d_used, 0, dgds::kUsedParts * 8 * sizeof(unsigned long long), s->st));
  s->T.used = s->d_used;
  if (int rc = grow_streams(s.get(), std::max<uint64_t>(p.expected_streams ? p.expected_streams : 4096, 64))) return rc;
  DGDS_CUDA(cudaMalloc(&s->d_err, sizeof(int32_t)));
  DGDS_CUDA(cudaMemsetAsync(s->d_err, 0, sizeof(int32_t), s->st));
  s->T.err = s->d_err;
  DGDS_CUDA(cudaMalloc(&s->T.ev_count, 2 * sizeof(unsigned long long)));
  DGDS_CUDA(cudaMalloc(&s->d_cplx_count, 2 * sizeof(unsigned long long)));
  DGDS_CUDA(cudaMalloc(&s->d_step_acc, 4 * sizeof(unsigned long long)));
  if (std::getenv("DGDS_K1_STATS")) {  // debug: append-path counters, read with dgds_debug_dump(6)
    DGDS_CUDA(cudaMalloc(&s->T.k1_stats, 8 * sizeof(unsigned long long)));
    DGDS_CUDA(cudaMemsetAsync(s->T.k1_stats, 0, 8 * sizeof(unsigned long long), s->st));
  }
  DGDS_CUDA(cudaMemsetAsync(s->d_step_acc, 0, 4 * sizeof(unsigned long long), s->st));
  DGDS_CUDA(cudaMemsetAsync(s->d_cplx_count, 0, 2 * sizeof(unsigned long long), s->st));
  DGDS_CUDA(cudaMemsetAsync(s->T.ev_count, 0, 2 * sizeof(unsigned long long), s->st));
  s->hist_cap = std::max<uint64_t>(1ull << 20, nodes / 2);  // ~ tokens (entries per token ~ 1-3)
  DGDS_CUDA(cudaMalloc(&s->d_hist, s->hist_cap * sizeof(int32_t)));
  s->T.hist = s->d_hist;
  s->shist_cap = s->hist_cap * 2;  // extents: up to 2x their streams' lengths
  s->T.hist_cap = s->hist_cap;
  s->T.shist_cap = s->shist_cap;
  DGDS_CUDA(cudaMalloc(&s->d_shist, s->shist_cap * sizeof(int32_t)));
  s->T.shist = s->d_shist;
  // [kStatParts][8] counter partitions + the ticket of k_query's last-block fold
  DGDS_CUDA(cudaMalloc(&s->d_stat_part, (dgds::kStatParts * 8 + 1) * sizeof(unsigned long long)));
  DGDS_CUDA(cudaMemsetAsync(s->d_stat_part, 0, (dgds::kStatParts * 8 + 1) * sizeof(unsigned long long), s->st));
  s->root_of_cap = 1024;
  DGDS_CUDA(cudaMalloc(&s->d_root_of, s->root_of_cap * sizeof(uint32_t)));
  DGDS_CUDA(cudaMemsetAsync(s->d_root_of, 0, s->root_of_cap * sizeof(uint32_t), s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  *out = s.release();
  return DGDS_OK;
}

int dgds_destroy(dgds_server* s) {
  if (!s) return DGDS_OK;
  recycle_launched(s);
  stop_planner(s);  // jobs still queued are planned first (their inputs are the caller's)
  cudaSetDevice(s->p.device);
  flush_pending(s);  // a staged batch: its workers finish, its kernels run
  if (s->st) cudaStreamSynchronize(s->st);
  if (s->out_st) cudaStreamSynchronize(s->out_st);
  if (s->copy_st) cudaStreamSynchronize(s->copy_st);
  cudaFree(s->T.slots);
  cudaFree(s->T.active);
  cudaFree(s->T.ov);
  cudaFree(s->T.sinfo);
  cudaFree(s->d_shist);
  cudaFree(s->T.ev);
  cudaFree(s->T.ev_count);
  cudaFree(s->d_cplx_count);
  cudaFree(s->d_step_acc);
  if (s->T.k1_stats) cudaFree(s->T.k1_stats);
  cudaFree(s->d_used);
  cudaFree(s->d_root_of);
  cudaFree(s->d_err);
  cudaFree(s->d_stat_part);
  cudaFree(s->d_hist);
  free_plan_pool(s);
  for (auto e : s->staging_free)
    if (e) cudaEventDestroy(e);
  for (auto e : s->plan_ready)
    if (e) cudaEventDestroy(e);
  for (auto e : s->plan_free)
    if (e) cudaEventDestroy(e);
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
  // entries + the count-1 chains below leaves (k_node_count) + group roots, matching
  // nodes_.size() (root counted) per live group
  DevBuf& tmp = s->d_count;
  if (int rc = tmp.ensure(sizeof(unsigned long long))) return rc;
  DGDS_CUDA(cudaMemsetAsync(tmp.p, 0, sizeof(unsigned long long), s->st));
  DGDS_CUDA(dgds::launch_node_count(s->T, static_cast<unsigned long long*>(tmp.p), s->st));
  unsigned long long nodes = 0;
  DGDS_CUDA(cudaMemcpyAsync(&nodes, tmp.p, sizeof(nodes), cudaMemcpyDeviceToHost, s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  uint64_t roots = 0;
  for (const auto& g : s->groups) roots += g.alive ? 1 : 0;
  *out = nodes + roots;
  return DGDS_OK;
}

int dgds_entry_count(dgds_server* s, uint64_t* out) {
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  cudaSetDevice(s->p.device);
  if (int rc = read_used(s, out)) return rc;
  s->used_ub = *out;
  return DGDS_OK;
}

int dgds_device_error(dgds_server* s, int32_t* flags) {
  if (!s || !flags) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaSetDevice(s->p.device));
  DGDS_CUDA(cudaMemcpyAsync(flags, s->d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, s->st));
  DGDS_CUDA(cudaMemsetAsync(s->d_err, 0, sizeof(int32_t), s->st));
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  return DGDS_OK;
}

}  // extern "C"

// dgds_update_batch without the lock (also the replica path of dgds_apply_blob)
int update_batch_locked(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids,
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
  std::vector<dgds::CopyPiece>& grow = s->scratch.grow;
  uint64_t worst = 0;
  if (int rc = plan_updates(s, n, handles, rids, prev, offs, nullptr, now, rep, segs, pieces, grow, &worst)) return rc;
  pc.mark("plan");
  if (segs.empty()) return DGDS_OK;
  if (int rc = ensure_capacity(s, worst, segs.size())) return rc;
  if (int rc = ensure_hist(s)) return rc;
  if (int rc = ensure_shist(s)) return rc;
  // one pinned staging block -> one H2D copy: segs | pieces | extent moves | tokens
  const size_t b_seg = segs.size() * sizeof(dgds::AppendSeg);
  const size_t o_piece = align_up(b_seg, 256);
  const size_t b_piece = pieces.size() * sizeof(dgds::AppendPiece);
  const size_t o_grow = align_up(o_piece + b_piece, 256);
  const size_t b_grow = grow.size() * sizeof(dgds::CopyPiece);
  const size_t o_tok = align_up(o_grow + b_grow, 256);
  const size_t total = o_tok + ntok * sizeof(int32_t);
  char* h = nullptr;
  cudaEvent_t ev_free = nullptr;
  if (int rc = next_stage(s, total, &h, &ev_free)) return rc;
  const int k = s->stage_k;  // the parity next_stage chose (d_plan protocol: launch_plan)
  if (int rc = s->d_plan[k].ensure(total)) return rc;
  for (auto& pc : pieces) pc.tok_off -= offs[0];
  nt_copy(h, segs.data(), b_seg);
  nt_copy(h + o_piece, pieces.data(), b_piece);
  nt_copy(h + o_grow, grow.data(), b_grow);
  nt_copy(h + o_tok, tokens + offs[0], ntok * sizeof(int32_t));
  _mm_sfence();
  char* d = static_cast<char*>(s->d_plan[k].p);
  pc.mark("stage");
  if (int rc = flush_pending(s)) return rc;  // K1 after the query batch submitted before it
  // the copy runs on copy_st under the kernels already queued; K1 waits for it
  DGDS_CUDA(cudaStreamWaitEvent(s->copy_st, s->plan_free[k], 0));
  DGDS_CUDA(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s->copy_st));
  DGDS_CUDA(cudaEventRecord(ev_free, s->copy_st));
  DGDS_CUDA(cudaEventRecord(s->plan_ready[k], s->copy_st));
  DGDS_CUDA(cudaStreamWaitEvent(s->st, s->plan_ready[k], 0));
  {
    LaunchTimer lt(s, 0, s->st);
    DGDS_CUDA(dgds::launch_append(s->T, reinterpret_cast<const dgds::AppendSeg*>(d),
                                  static_cast<int64_t>(segs.size()), reinterpret_cast<const dgds::AppendPiece*>(d + o_piece),
                                  static_cast<int64_t>(pieces.size()), reinterpret_cast<const int32_t*>(d + o_tok),
                                  reinterpret_cast<const dgds::CopyPiece*>(d + o_grow),
                                  static_cast<int64_t>(grow.size()), s->st));
  }
  DGDS_CUDA(cudaEventRecord(s->plan_free[k], s->st));
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

// A planned device update: host bookkeeping done (replies final), device work pending.
struct dgds_update_plan {
  std::vector<dgds::AppendSeg> segs;
  std::vector<dgds::AppendPiece> pieces;
  std::vector<dgds::CopyPiece> grow;  // stream extents moved by this plan
  std::vector<DeferredLog> logs;  // history-log records, appended after the launch
  const int32_t* d_tokens = nullptr;
  uint64_t seq = 0;
  bool launched = false;  // queued by dgds_update_launch: recycled once its logs are materialized
};

namespace dgds_host {
void materialize_logs(dgds_server* s) {
  for (dgds_update_plan* p : s->log_pending) {
    for (const DeferredLog& d : p->logs) s->groups[d.handle].log.push_back(d.rec);
    p->logs.clear();
    if (p->launched) s->plan_pool.push_back(p);
  }
  s->log_pending.clear();
}

// The launched prefix only (plan order = log order): run by the routed planner thread while it
// waits for its next job's metadata, so the ~4,096 log appends per tick stay off the launching
// thread (measured 45 of update_launch's 90 us at 4,096 records).
void materialize_launched(dgds_server* s) {
  size_t k = 0;
  for (; k < s->log_pending.size() && s->log_pending[k]->launched; ++k) {
    dgds_update_plan* p = s->log_pending[k];
    for (const DeferredLog& d : p->logs) s->groups[d.handle].log.push_back(d.rec);
    p->logs.clear();
    s->plan_pool.push_back(p);
  }
  s->log_pending.erase(s->log_pending.begin(), s->log_pending.begin() + static_cast<std::ptrdiff_t>(k));
}
}  // namespace dgds_host

static void recycle_launched(dgds_server* s) {  // teardown: launched plans kept for their logs
  for (auto* pl : s->log_pending)
    if (pl->launched) s->plan_pool.push_back(pl);
  s->log_pending.clear();
}

static void free_plan_pool(dgds_server* s) {
  for (auto* pl : s->plan_pool) delete pl;
  s->plan_pool.clear();
}

// Host half: validation, bookkeeping (replies, versions, history log), capacity. Plans must be
// launched in the order they were made (K1 of a later plan reads the stream rows K1 of an
// earlier one writes), which dgds_update_launch checks.
// defer_logs = false (a plan launched within the same locked call): history-log records go
// straight to the group logs instead of through the plan.
static int plan_device(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* rids, const uint64_t* prev,
                       const uint64_t* offs, const uint64_t* counts, const int32_t* d_tokens, double now,
                       dgds_update_reply* rep, dgds_update_plan* plan, bool defer_logs = true) {
  uint64_t worst = 0;
  const int prc = plan_updates(s, n, handles, rids, prev, offs, counts, now, rep, plan->segs, plan->pieces,
                               plan->grow, &worst, defer_logs ? &plan->logs : nullptr);
  if (!plan->logs.empty()) s->log_pending.push_back(plan);  // accepted records, even on a later error
  if (prc) return prc;
  if (plan->segs.empty()) return DGDS_OK;
  if (int rc = ensure_capacity(s, worst, plan->segs.size())) return rc;
  if (int rc = ensure_hist(s)) return rc;
  if (int rc = ensure_shist(s)) return rc;
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
  const size_t o_grow = align_up(o_piece + plan->pieces.size() * sizeof(dgds::AppendPiece), 256);
  const size_t total = o_grow + plan->grow.size() * sizeof(dgds::CopyPiece);
  char* h = nullptr;
  cudaEvent_t ev_free = nullptr;
  if (int rc = next_stage(s, total, &h, &ev_free)) return rc;
  pc.mark("staging_wait");
  const int k = s->stage_k;  // the parity next_stage chose
  if (int rc = s->d_plan[k].ensure(total)) return rc;  // growth: cudaFree waits for the device
  nt_copy(h, plan->segs.data(), b_seg);
  nt_copy(h + o_piece, plan->pieces.data(), plan->pieces.size() * sizeof(dgds::AppendPiece));
  nt_copy(h + o_grow, plan->grow.data(), plan->grow.size() * sizeof(dgds::CopyPiece));
  _mm_sfence();
  pc.mark("stage");
  char* d = static_cast<char*>(s->d_plan[k].p);
  DGDS_CUDA(cudaStreamWaitEvent(s->copy_st, s->plan_free[k], 0));  // its last readers were enqueued
  DGDS_CUDA(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s->copy_st));
  DGDS_CUDA(cudaEventRecord(ev_free, s->copy_st));
  DGDS_CUDA(cudaEventRecord(s->plan_ready[k], s->copy_st));
  DGDS_CUDA(cudaStreamWaitEvent(join.stream(), s->plan_ready[k], 0));
  {
    LaunchTimer lt(s, 0, join.stream());
    DGDS_CUDA(dgds::launch_append(s->T, reinterpret_cast<const dgds::AppendSeg*>(d),
                                  static_cast<int64_t>(plan->segs.size()),
                                  reinterpret_cast<const dgds::AppendPiece*>(d + o_piece),
                                  static_cast<int64_t>(plan->pieces.size()), plan->d_tokens,
                                  reinterpret_cast<const dgds::CopyPiece*>(d + o_grow),
                                  static_cast<int64_t>(plan->grow.size()), join.stream()));
  }
  DGDS_CUDA(cudaEventRecord(s->plan_free[k], join.stream()));
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
  plan.grow.clear();
  if (int rc = plan_device(s, n, handles, rids, prev, offs, counts, d_tokens, now, rep, &plan, false)) {
    materialize_logs(s);
    return rc;
  }
  pc.mark("plan");
  const int rc = launch_plan(s, &plan, stream, pc);
  materialize_logs(s);  // after K1 is queued
  return rc;
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

namespace dgds_host {
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
}  // namespace dgds_host

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
  plan->grow.clear();
  plan->logs.clear();
  plan->d_tokens = nullptr;
  plan->seq = 0;
  plan->launched = false;
  if (n > 0) {
    thread_local RoutedScratch r;
    if (int rc = fill_routed(r, n, n_seg, seg_rows, h_counts, h_meta, meta_stride, row_words)) return rc;
    std::lock_guard<std::mutex> lk(s->mu);
    if (int rc_ = flush_pending(s)) return rc_;
    DGDS_CUDA(cudaSetDevice(s->p.device));
    if (int rc = plan_device(s, n, r.handles.data(), r.rids.data(), r.prev.data(), r.starts.data(), r.counts.data(),
                             d_rows, now, r.rep.data(), plan.get())) {
      materialize_logs(s);  // before the plan (holding accepted records' logs) is destroyed
      return rc;
    }
    if (n_rejected) {
      int64_t bad = 0;
      for (int64_t k = 0; k < n; ++k) bad += r.rep[k].ok ? 0 : 1;
      *n_rejected = bad;
    }
  }
  *out = plan.release();
  return DGDS_OK;
}

}  // extern "C"

struct dgds_server::PlanJob {
  cudaEvent_t ready = nullptr;
  int32_t n_seg = 0;
  int64_t seg_rows = 0;
  const int32_t* h_counts = nullptr;
  const int32_t* h_meta = nullptr;
  int32_t meta_stride = 0;
  const int32_t* d_rows = nullptr;
  int32_t row_words = 0;
  double now = 0.0;
  bool done = false;
  int rc = DGDS_OK;
  std::string msg;
  int64_t n_rejected = 0;
  dgds_update_plan* plan = nullptr;
};

static void planner_loop(dgds_server* s) {
  cudaSetDevice(s->p.device);
  for (;;) {
    std::shared_ptr<dgds_server::PlanJob> j;
    {
      std::unique_lock<std::mutex> lk(s->pj_mu);
      s->pj_cv.wait(lk, [&] { return s->pj_stop || !s->pj_queue.empty(); });
      if (s->pj_queue.empty()) return;  // stopping
      j = s->pj_queue.front();
      s->pj_queue.pop_front();
    }
    {
      std::lock_guard<std::mutex> lk(s->mu);
      materialize_launched(s);  // earlier plans' logs, before waiting for this job's metadata
    }
    int rc = DGDS_OK;
    if (j->ready && cudaEventSynchronize(j->ready) != cudaSuccess)
      rc = fail(DGDS_ECUDA, "metadata event of a routed plan failed");
    if (rc == DGDS_OK)
      rc = dgds_update_plan_routed(s, j->n_seg, j->seg_rows, j->h_counts, j->h_meta, j->meta_stride, j->d_rows,
                                   j->row_words, j->now, &j->n_rejected, &j->plan);
    {
      std::lock_guard<std::mutex> lk(s->pj_mu);
      j->rc = rc;
      if (rc) j->msg = dgds_last_error();
      j->done = true;
    }
    s->pj_done_cv.notify_all();
  }
}

static void stop_planner(dgds_server* s) {
  {
    std::lock_guard<std::mutex> lk(s->pj_mu);
    s->pj_stop = true;
  }
  s->pj_cv.notify_all();
  if (s->planner.joinable()) s->planner.join();
  for (auto& kv : s->pj_jobs) delete kv.second->plan;  // planned but never taken
  s->pj_jobs.clear();
}

extern "C" {

int dgds_update_plan_routed_async(dgds_server* s, void* ready_event, int32_t n_seg, int64_t seg_rows,
                                  const int32_t* h_counts, const int32_t* h_meta, int32_t meta_stride,
                                  const int32_t* d_rows, int32_t row_words, double now, uint64_t* job) {
  if (!s || !job || !d_rows) return fail(DGDS_EINVAL, "bad routed append arguments");
  auto j = std::make_shared<dgds_server::PlanJob>();
  j->ready = static_cast<cudaEvent_t>(ready_event);
  j->n_seg = n_seg;
  j->seg_rows = seg_rows;
  j->h_counts = h_counts;
  j->h_meta = h_meta;
  j->meta_stride = meta_stride;
  j->d_rows = d_rows;
  j->row_words = row_words;
  j->now = now;
  {
    std::lock_guard<std::mutex> lk(s->pj_mu);
    if (!s->planner.joinable()) s->planner = std::thread(planner_loop, s);
    *job = ++s->pj_next;
    s->pj_jobs[*job] = j;
    s->pj_queue.push_back(j);
  }
  s->pj_cv.notify_one();
  return DGDS_OK;
}

int dgds_update_plan_take(dgds_server* s, uint64_t job, int64_t* n_rejected, dgds_update_plan** out) {
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  *out = nullptr;
  std::shared_ptr<dgds_server::PlanJob> j;
  {
    std::unique_lock<std::mutex> lk(s->pj_mu);
    auto it = s->pj_jobs.find(job);
    if (it == s->pj_jobs.end()) return fail(DGDS_EINVAL, "unknown plan job");
    j = it->second;
    s->pj_done_cv.wait(lk, [&] { return j->done; });
    s->pj_jobs.erase(it);
  }
  if (n_rejected) *n_rejected = j->n_rejected;
  if (j->rc) return fail(j->rc, j->msg);
  *out = j->plan;
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
  // its history-log records are materialized later (the planner thread, or any reader of the
  // logs); a plan without pending records is recycled now (the staging copy keeps no references)
  plan->launched = true;
  if (plan->logs.empty()) s->plan_pool.push_back(plan);
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

extern "C" {

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

// Debug: copy device state into out (host): which 0 = slot table, 1 = stream table (StreamInfo),
// 2 = active rows, 3 = ov rows, 4 = the stream-history arena, 5 = event queue. At most `bytes`.
extern "C" int dgds_debug_dump(dgds_server* s, int32_t which, void* out, uint64_t bytes) {
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  const void* src = nullptr;
  uint64_t have = 0;
  switch (which) {
    case 0: src = s->T.slots; have = s->T.cap * sizeof(dgds::Slot); break;
    case 1: src = s->T.sinfo; have = s->stream_cap * sizeof(dgds::StreamInfo); break;
    case 2: src = s->T.active; have = s->stream_cap * dgds::kWarp * 4; break;
    case 3: src = s->T.ov; have = s->stream_cap * dgds::kWarp * 4; break;
    case 4: src = s->d_shist; have = s->shist_cap * 4; break;
    case 5: src = s->T.ev; have = s->ev_cap * sizeof(dgds::WalkEvent); break;
    case 6: src = s->T.k1_stats; have = s->T.k1_stats ? 8 * sizeof(unsigned long long) : 0; break;
    default: return fail(DGDS_EINVAL, "bad dump selector");
  }
  DGDS_CUDA(cudaMemcpy(out, src, std::min(bytes, have), cudaMemcpyDeviceToHost));
  return DGDS_OK;
}

extern "C" int dgds_debug_append_timing(dgds_server* s, uint64_t* out, int64_t n_warps) {  // [n][2] start, end (ns)
  if (!s || !out) return fail(DGDS_EINVAL, "null argument");
  if (!s->T.dbg) return fail(DGDS_ESTATE, "set DGDS_APPEND_DBG before dgds_create");
  std::lock_guard<std::mutex> lk(s->mu);
  if (int rc_ = flush_pending(s)) return rc_;
  DGDS_CUDA(cudaStreamSynchronize(s->st));
  DGDS_CUDA(cudaMemcpy(out, s->T.dbg, std::min<int64_t>(n_warps, 65536) * 16, cudaMemcpyDeviceToHost));
  return DGDS_OK;
}

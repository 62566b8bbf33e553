// cluster.cpp — N GPUs behind one draft server (dgds_cluster_*, include/dgds_b200.h).
//
// The reference routes every call by shard behind one DraftServer API: shard = shard_of_group
// (fnv1a64(group_id) % shard_count, dgds.cpp:10-14), each shard owning its groups' indexes
// under its own mutex (dgds.cpp:36-51,130-138). Here a shard is a GPU: one dgds_server per
// device, group g owned by GPU fnv1a64(g) % n. A batch call splits its records / queries by
// owner (stable, so every owner sees its records in call order — versions and gap checks are
// per group, and a group lives on one owner), runs the owners' batches concurrently on one
// host thread per GPU (each bound to its device), and scatters the replies back in call order.
// Records arrive on the host, so they go straight to their owner's GPU with one H2D each; no
// device-to-device exchange is needed on this path (the NVLink peer exchange, csrc/peer.cu,
// serves ranks whose inputs are already on their GPUs).
#include "server_internal.h"

namespace {

// One persistent host thread per GPU; run(f) calls f(g) for every GPU in parallel.
class GpuThreads {
 public:
  explicit GpuThreads(const std::vector<int>& devices) : dev_(devices) {
    for (size_t g = 0; g < dev_.size(); ++g) th_.emplace_back([this, g] { loop(static_cast<int>(g)); });
  }
  ~GpuThreads() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void run(const std::function<void(int)>& f) {
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &f;
    left_ = static_cast<int>(dev_.size());
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [this] { return left_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int g) {
    cudaSetDevice(dev_[g]);
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = fn_;
      }
      (*f)(g);
      std::lock_guard<std::mutex> lk(mu_);
      if (--left_ == 0) done_.notify_all();
    }
  }
  std::vector<int> dev_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int left_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace

struct dgds_cluster {
  std::vector<dgds_server*> srv;
  std::vector<int> devices;
  std::unique_ptr<GpuThreads> threads;
  std::unordered_map<std::string, int32_t> intern;
  std::vector<std::pair<int32_t, int32_t>> owner_of;  // cluster handle -> (gpu, server handle)
  std::mutex mu;
  // per-GPU scratch of a batch call (kept: capacities persist)
  struct Part {
    std::vector<int64_t> idx;
    std::vector<int32_t> handles, rids;
    std::vector<uint64_t> prev, offs;
    std::vector<int32_t> tokens;
    std::vector<dgds_update_reply> rep;
    dgds_result_view view{};
    int rc = DGDS_OK;
    std::string msg;
  };
  std::vector<Part> part;
  std::vector<std::pair<int32_t, uint32_t>> where;  // per call item: (owner, index within the owner's part)
  std::vector<int64_t> cnt, bad;                     // partition scratch: [range][owner] counts, first bad item
};

namespace {

// resize a per-GPU scratch vector, growing its capacity with headroom: batch sizes per owner
// vary from call to call, and every reallocation of a multi-MB buffer maps and faults fresh
// pages (measured: ~5,000 minor faults per 4-GPU tick when sized exactly, ~10x the tick time)
template <class T>
void sized(std::vector<T>& v, size_t n) {
  if (n > v.capacity()) v.reserve(n + n / 2);
  v.resize(n);
}

int owner_check(dgds_cluster* c, int32_t h) {
  if (!c) return fail(DGDS_EINVAL, "null cluster");
  if (h < 0 || static_cast<size_t>(h) >= c->owner_of.size()) return fail(DGDS_EINVAL, "bad group handle");
  return DGDS_OK;
}

// Run f(gpu, Part&) on every GPU that has work; the first failure is returned.
int run_parts(dgds_cluster* c, const std::function<int(int, dgds_cluster::Part&)>& f) {
  for (auto& p : c->part) p.rc = DGDS_OK;
  c->threads->run([&](int g) {
    dgds_cluster::Part& p = c->part[g];
    if (p.idx.empty()) return;
    PhaseClock pc("cluster_part");
    p.rc = f(g, p);
    if (p.rc) p.msg = dgds_last_error();
    pc.mark("owner_batch");
  });
  for (auto& p : c->part)
    if (p.rc) return fail(p.rc, p.msg);
  return DGDS_OK;
}

// Copy the owners' replies back in call order. GPU thread g takes the contiguous call range
// [g*n/N, (g+1)*n/N): scattering by owner instead made every thread write interleaved items of
// the caller's arrays, and the shared cache lines cost ~100 ns per query (measured, 4 GPUs).
// Each range is split further over that GPU's server host workers (idle between its calls).
void scatter(dgds_cluster* c, int64_t n, const std::function<void(int64_t, dgds_cluster::Part&, uint32_t)>& f) {
  const int64_t N = static_cast<int64_t>(c->part.size());
  c->threads->run([&](int g) {
    const int64_t a = n * g / N, b = n * (g + 1) / N;
    WorkerPool& pool = c->srv[g]->workers();
    const int tasks = b - a >= 8192 ? 2 * pool.threads() : 1;
    pool.run(tasks, [&](int t) {
      for (int64_t i = a + (b - a) * t / tasks; i < a + (b - a) * (t + 1) / tasks; ++i)
        f(i, c->part[c->where[i].first], c->where[i].second);
    });
  });
}

// Split a batch by owner in parallel: GPU thread g scans the call range [g*n/N, (g+1)*n/N) twice —
// counting its items per owner (and validating them), then, at the offsets the counts give,
// writing each item's call index and server handle into its owner's part and its (owner, index
// within the part) into c->where. Every thread writes contiguous runs, and owners see their
// items in call order. Returns the first invalid item's error, as a serial scan would.
int partition(dgds_cluster* c, int64_t n, const int32_t* handles, const uint64_t* offs, const char* offs_msg) {
  const int N = static_cast<int>(c->part.size());
  if (N == 1) {  // one GPU: only the handles are mapped (the owner validates the rest)
    dgds_cluster::Part& p = c->part[0];
    sized(p.handles, n);
    sized(p.idx, n);  // only its size is read: it marks the single owner's part as the whole call
    for (int64_t i = 0; i < n; ++i) {
      if (int rc = owner_check(c, handles[i])) return rc;
      p.handles[i] = c->owner_of[handles[i]].second;
    }
    return DGDS_OK;
  }
  sized(c->where, n);
  c->cnt.assign(static_cast<size_t>(N) * N, 0);
  c->bad.assign(N, INT64_MAX);
  c->threads->run([&](int g) {
    int64_t* cnt = c->cnt.data() + static_cast<size_t>(g) * N;
    for (int64_t i = n * g / N; i < n * (g + 1) / N; ++i) {
      const int32_t h = handles[i];
      if (h < 0 || static_cast<size_t>(h) >= c->owner_of.size() || offs[i + 1] < offs[i]) {
        c->bad[g] = i;
        return;
      }
      ++cnt[c->owner_of[h].first];
    }
  });
  for (int g = 0; g < N; ++g)
    if (c->bad[g] != INT64_MAX) {
      const int64_t i = c->bad[g];
      if (int rc = owner_check(c, handles[i])) return rc;
      return fail(DGDS_EINVAL, offs_msg);
    }
  for (int o = 0; o < N; ++o) {  // cnt[g][o] -> start of range g's items in part o
    int64_t at = 0;
    for (int g = 0; g < N; ++g) {
      const int64_t k = c->cnt[static_cast<size_t>(g) * N + o];
      c->cnt[static_cast<size_t>(g) * N + o] = at;
      at += k;
    }
    sized(c->part[o].idx, at);
    sized(c->part[o].handles, at);
  }
  c->threads->run([&](int g) {
    int64_t* at = c->cnt.data() + static_cast<size_t>(g) * N;
    for (int64_t i = n * g / N; i < n * (g + 1) / N; ++i) {
      const auto& ow = c->owner_of[handles[i]];
      dgds_cluster::Part& p = c->part[ow.first];
      const int64_t k = at[ow.first]++;
      p.idx[k] = i;
      p.handles[k] = ow.second;
      c->where[i] = {ow.first, static_cast<uint32_t>(k)};
    }
  });
  return DGDS_OK;
}

}  // namespace

extern "C" {

int dgds_cluster_create(const dgds_params* params, int32_t n_gpus, const int32_t* devices, dgds_cluster** out) {
  if (!params || !out || n_gpus < 1 || n_gpus > 64) return fail(DGDS_EINVAL, "bad cluster arguments");
  *out = nullptr;
  auto c = std::make_unique<dgds_cluster>();
  for (int32_t g = 0; g < n_gpus; ++g) {
    dgds_params p = *params;
    p.device = devices ? devices[g] : g;
    dgds_server* s = nullptr;
    if (int rc = dgds_create(&p, &s)) {
      for (auto* x : c->srv) dgds_destroy(x);
      return rc;
    }
    c->srv.push_back(s);
    c->devices.push_back(p.device);
  }
  // the owners' batches run at once, so each server's host worker pool gets its share of the cores
  // (measured on a 4-GPU box: 4 servers x 8 workers oversubscribed the host and stalled calls by ms)
  const int hw = std::max(1, static_cast<int>(std::thread::hardware_concurrency()));
  for (auto* s : c->srv) s->pool_threads = std::max(1, std::min(host_threads(), hw / n_gpus - 1));
  c->part.resize(n_gpus);
  c->threads = std::make_unique<GpuThreads>(c->devices);
  *out = c.release();
  return DGDS_OK;
}

int dgds_cluster_destroy(dgds_cluster* c) {
  if (!c) return DGDS_OK;
  c->threads.reset();
  for (auto* s : c->srv) dgds_destroy(s);
  delete c;
  return DGDS_OK;
}

int32_t dgds_cluster_size(dgds_cluster* c) { return c ? static_cast<int32_t>(c->srv.size()) : 0; }

dgds_server* dgds_cluster_server(dgds_cluster* c, int32_t gpu) {
  return (c && gpu >= 0 && static_cast<size_t>(gpu) < c->srv.size()) ? c->srv[gpu] : nullptr;
}

int dgds_cluster_intern(dgds_cluster* c, const char* gid, size_t len, int32_t* handle) {
  if (!c || !gid || !handle) return fail(DGDS_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  std::string key(gid, len);
  auto it = c->intern.find(key);
  if (it != c->intern.end()) {
    *handle = it->second;
    return DGDS_OK;
  }
  const int32_t g = static_cast<int32_t>(fnv1a64(gid, len) % c->srv.size());  // shard_of_group (dgds.cpp:10-14)
  int32_t local = 0;
  if (int rc = dgds_intern(c->srv[g], gid, len, &local)) return rc;
  const int32_t h = static_cast<int32_t>(c->owner_of.size());
  c->owner_of.emplace_back(g, local);
  c->intern.emplace(std::move(key), h);
  *handle = h;
  return DGDS_OK;
}

int dgds_cluster_owner(dgds_cluster* c, int32_t handle, int32_t* gpu) {
  if (int rc = owner_check(c, handle)) return rc;
  *gpu = c->owner_of[handle].first;
  return DGDS_OK;
}

int dgds_cluster_register_group(dgds_cluster* c, int32_t h, double ttl, double now) {
  if (int rc = owner_check(c, h)) return rc;
  return dgds_register_group(c->srv[c->owner_of[h].first], c->owner_of[h].second, ttl, now);
}
int dgds_cluster_drop_group(dgds_cluster* c, int32_t h) {
  if (int rc = owner_check(c, h)) return rc;
  return dgds_drop_group(c->srv[c->owner_of[h].first], c->owner_of[h].second);
}
int dgds_cluster_sweep_expired(dgds_cluster* c, double now) {
  if (!c) return fail(DGDS_EINVAL, "null cluster");
  for (auto* s : c->srv)
    if (int rc = dgds_sweep_expired(s, now)) return rc;
  return DGDS_OK;
}
int dgds_cluster_has_group(dgds_cluster* c, int32_t h, int32_t* out) {
  if (int rc = owner_check(c, h)) return rc;
  return dgds_has_group(c->srv[c->owner_of[h].first], c->owner_of[h].second, out);
}
int dgds_cluster_group_version(dgds_cluster* c, int32_t h, uint64_t* out) {
  if (int rc = owner_check(c, h)) return rc;
  return dgds_group_version(c->srv[c->owner_of[h].first], c->owner_of[h].second, out);
}
int dgds_cluster_stored_tokens(dgds_cluster* c, int32_t h, int32_t rid, uint64_t* out) {
  if (int rc = owner_check(c, h)) return rc;
  return dgds_stored_tokens(c->srv[c->owner_of[h].first], c->owner_of[h].second, rid, out);
}
int dgds_cluster_shard_group_count(dgds_cluster* c, int32_t shard, uint64_t* out) {
  if (!c || !out) return fail(DGDS_EINVAL, "null argument");
  uint64_t t = 0;
  for (auto* s : c->srv) {  // logical shards span the GPUs: every server counts its own groups
    uint64_t x = 0;
    if (int rc = dgds_shard_group_count(s, shard, &x)) return rc;
    t += x;
  }
  *out = t;
  return DGDS_OK;
}
int dgds_cluster_node_count(dgds_cluster* c, uint64_t* out) {
  if (!c || !out) return fail(DGDS_EINVAL, "null argument");
  uint64_t t = 0;
  for (auto* s : c->srv) {
    uint64_t x = 0;
    if (int rc = dgds_node_count(s, &x)) return rc;
    t += x;
  }
  *out = t;
  return DGDS_OK;
}

int dgds_cluster_update_batch(dgds_cluster* c, int64_t n, const int32_t* handles, const int32_t* rids,
                              const uint64_t* prev, const uint64_t* offs, const int32_t* tokens, double now,
                              dgds_update_reply* rep) {
  if (!c || n < 0 || (n > 0 && (!handles || !rids || !prev || !offs || !tokens || !rep)))
    return fail(DGDS_EINVAL, "null argument");
  if (n == 0) return DGDS_OK;
  std::lock_guard<std::mutex> lk(c->mu);
  if (int rc = partition(c, n, handles, offs, "token offsets must be nondecreasing")) return rc;
  for (size_t g = 0; g < c->part.size(); ++g)  // one owner: the caller's batch in place
    if (static_cast<int64_t>(c->part[g].idx.size()) == n)
      return dgds_update_batch(c->srv[g], n, c->part[g].handles.data(), rids, prev, offs, tokens, now, rep);
  const int rc = run_parts(c, [&](int g, dgds_cluster::Part& p) {
    const size_t m = p.idx.size();
    sized(p.rids, m);
    sized(p.prev, m);
    sized(p.offs, m + 1);
    sized(p.rep, m);
    size_t ntok = 0;
    for (size_t k = 0; k < m; ++k) ntok += offs[p.idx[k] + 1] - offs[p.idx[k]];
    sized(p.tokens, ntok);
    p.offs[0] = 0;
    for (size_t k = 0; k < m; ++k) {
      const int64_t i = p.idx[k];
      p.rids[k] = rids[i];
      p.prev[k] = prev[i];
      std::memcpy(p.tokens.data() + p.offs[k], tokens + offs[i], (offs[i + 1] - offs[i]) * sizeof(int32_t));
      p.offs[k + 1] = p.offs[k] + (offs[i + 1] - offs[i]);
    }
    return dgds_update_batch(c->srv[g], static_cast<int64_t>(m), p.handles.data(), p.rids.data(), p.prev.data(),
                             p.offs.data(), p.tokens.data(), now, p.rep.data());
  });
  if (rc) return rc;
  scatter(c, n, [&](int64_t i, dgds_cluster::Part& p, uint32_t k) { rep[i] = p.rep[k]; });
  return DGDS_OK;
}

int dgds_cluster_speculate_verify_batch(dgds_cluster* c, int64_t n, const int32_t* handles,
                                        const uint64_t* pat_offsets, const int32_t* patterns,
                                        const dgds_spec_args* args, int64_t args_stride, const int32_t* truth_next,
                                        int32_t truth_stride, const int32_t* truth_left, const int32_t* limit,
                                        dgds_candidates* out, dgds_verify_out* vout) {
  if (!c || n < 0 || (n > 0 && (!handles || !pat_offsets || !patterns || !args || !out)))
    return fail(DGDS_EINVAL, "null argument");
  if (vout && (!truth_next || !truth_left || !limit)) return fail(DGDS_EINVAL, "verify needs truth inputs");
  if (n == 0) return DGDS_OK;
  std::lock_guard<std::mutex> lk(c->mu);
  if (int rc = partition(c, n, handles, pat_offsets, "pattern offsets must be nondecreasing")) return rc;
  const int32_t K = out->k_stride, S = out->s_stride;
  for (size_t g = 0; g < c->part.size(); ++g)  // every query is owned by one GPU: its batch is the caller's, in place
    if (static_cast<int64_t>(c->part[g].idx.size()) == n)
      return dgds_speculate_verify_batch(c->srv[g], n, c->part[g].handles.data(), pat_offsets, patterns, args,
                                         args_stride, truth_next, truth_stride, truth_left, limit, out, vout);
  for (int64_t i = 0; i < (args_stride ? n : 1); ++i) {  // the owners' results are scattered at these strides
    const dgds_spec_args& a = args[i * args_stride];
    if (a.top_k > K || std::min(a.max_spec_tokens, c->srv[0]->p.max_spec_len) > S)
      return fail(DGDS_EBUFFER, "candidate buffer strides too small");
  }
  // each owner stages its rows straight from the caller's arrays (idx), on its own host workers;
  // its results stay in its mapped result slot (valid until its next-but-one batch; the cluster
  // lock is held until they are scattered below)
  const int rc = run_parts(c, [&](int g, dgds_cluster::Part& p) {
    return dgds_host::speculate_view_indexed(c->srv[g], static_cast<int64_t>(p.idx.size()), p.idx.data(),
                                             p.handles.data(), pat_offsets, patterns, args, args_stride,
                                             vout ? truth_next : nullptr, truth_stride, truth_left, limit, &p.view);
  });
  if (rc) return rc;
  scatter(c, n, [&](int64_t i, dgds_cluster::Part& p, uint32_t k) {
    const dgds_result_view& v = p.view;
    const int64_t c0 = v.cand_off[k], c1 = v.cand_off[k + 1];
    out->n_cands[i] = static_cast<int32_t>(c1 - c0);
    for (int64_t j = c0; j < c1; ++j) {
      const int64_t di = i * K + (j - c0);
      const dgds_cand_meta& m = v.cands[j];
      out->lens[di] = m.len;
      out->scores[di] = m.score;
      out->supports[di] = m.support;
      std::memcpy(out->tokens + di * S, v.tokens + v.tok_off[j], static_cast<size_t>(m.len) * sizeof(int32_t));
    }
    if (vout) {
      vout->drafted[i] = v.drafted[k];
      vout->accepted[i] = v.accepted[k];
      vout->emitted[i] = v.emitted[k];
    }
  });
  return DGDS_OK;
}

}  // extern "C"

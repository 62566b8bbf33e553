// dgds_b200.hpp — C++ facade of the B200 draft server over the C ABI (dgds_b200.h).
//
// Mirrors the reference C++ API so a rollout engine can switch by changing the
// include and namespace:
//   rollsim::DraftServer      (proj/include/rollsim/dgds.hpp:51-91)   -> dgds_b200::DraftServer
//   rollsim::DraftTransport / LocalTransport (dgds.hpp:93-116)      -> same names
//   rollsim::DraftClient      (dgds.hpp:128-162)                      -> dgds_b200::DraftClient
//     DraftClient(DraftTransport&, DgdsParams) as in the reference; replicas of the queried /
//     active groups are GPU-resident (GDX1 blobs, cst.cpp:233-329)
//   rollsim::SpeculationSource (engine.hpp:67-74, never implemented
//                               in the reference)                    -> dgds_b200::GpuSpeculationSource
//   SpeculationArgs / DraftCandidate / UpdateReply / DgdsParams / SpecQuery
//                              (cst.hpp:16-29, dgds.hpp:18-43,118-122) -> same names, same defaults
// Errors follow the reference: std::invalid_argument where it throws that
// (bad args, negative request id or token), std::runtime_error otherwise.
// Header-only; link against paper_2511_14617_b200/libdgds_b200.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "dgds_b200.h"

namespace dgds_b200 {

using Token = std::int32_t;
using TokenSeq = std::vector<Token>;
using SimTime = double;

struct SpeculationArgs {  // cst.hpp:16-23
  int max_spec_tokens = 8;
  int pattern_lookup_max = 6;
  int pattern_lookup_min = 1;
  int top_k = 1;
  double min_step_freq = 0.25;
  long long min_support = 1;
};

struct DraftCandidate {  // cst.hpp:25-29
  TokenSeq tokens;
  double score = 0.0;
  long long support = 0;
};

struct Limits {  // GroupDraftIndex::Limits, cst.hpp:44-47
  int max_pattern_len = 8;
  int max_spec_len = 16;
};

struct DgdsParams {  // dgds.hpp:18-24 (+ device placement)
  int shard_count = 1;
  double fetch_period = 0.2;
  int append_batch_tokens = 16;
  double default_ttl_seconds = 600.0;
  Limits limits;
  int device = 0;
  std::uint64_t expected_nodes = 0;
  std::uint64_t expected_streams = 0;
};

struct UpdateReply {  // dgds.hpp:39-43
  bool ok = false;
  std::uint64_t version = 0;
  std::uint64_t acked_tokens = 0;
};

struct DraftCacheInfo {  // dgds.hpp:26-29
  std::string group_id;
  std::uint64_t cached_version = 0;  // 0 = no local replica
};

enum class FetchKind : std::uint8_t { UpToDate = 0, Delta = 1, Full = 2, UnknownGroup = 3 };  // dgds.hpp:31

struct FetchReply {  // dgds.hpp:33-37
  FetchKind kind = FetchKind::UnknownGroup;
  std::uint64_t version = 0;
  std::vector<std::uint8_t> blob;
};

struct SpecQuery {  // dgds.hpp:118-122
  std::string group_id;
  TokenSeq pattern;
  SpeculationArgs args;
};

namespace detail {
inline void check(int rc) {
  if (rc == DGDS_OK) return;
  const std::string msg = dgds_last_error();
  if (rc == DGDS_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("dgds: " + msg);
}
inline dgds_spec_args c_args(const SpeculationArgs& a) {
  return dgds_spec_args{a.max_spec_tokens, a.pattern_lookup_max, a.pattern_lookup_min, a.top_k, a.min_step_freq,
                        a.min_support};
}
}  // namespace detail

// shard_of_group (dgds.cpp:10-14)
inline int shard_of_group(const std::string& group_id, int shard_count) {
  const int r = dgds_shard_of_group(group_id.data(), group_id.size(), shard_count);
  if (r < 0) throw std::invalid_argument("shard_count must be >= 1");
  return r;
}

class DraftServer {
 public:
  explicit DraftServer(DgdsParams params = {}) : params_(params) {
    dgds_params p{};
    p.shard_count = params.shard_count;
    p.append_batch_tokens = params.append_batch_tokens;
    p.fetch_period = params.fetch_period;
    p.default_ttl_seconds = params.default_ttl_seconds;
    p.max_pattern_len = params.limits.max_pattern_len;
    p.max_spec_len = params.limits.max_spec_len;
    p.device = params.device;
    p.expected_nodes = params.expected_nodes;
    p.expected_streams = params.expected_streams;
    detail::check(dgds_create(&p, &s_));
  }
  ~DraftServer() { dgds_destroy(s_); }
  DraftServer(const DraftServer&) = delete;
  DraftServer& operator=(const DraftServer&) = delete;

  UpdateReply update_cst(const std::string& group_id, int request_id, std::uint64_t prev_token_count,
                         std::span<const Token> new_tokens, SimTime now) {
    const std::int32_t h = handle(group_id);
    const std::uint64_t offs[2] = {0, new_tokens.size()};
    dgds_update_reply r{};
    detail::check(dgds_update_batch(s_, 1, &h, &request_id, &prev_token_count, offs, new_tokens.data(), now, &r));
    return UpdateReply{r.ok != 0, r.version, r.acked_tokens};
  }

  // n update_cst calls in call order, one device launch.
  std::vector<UpdateReply> update_batch(std::span<const std::string> group_ids, std::span<const int> request_ids,
                                        std::span<const std::uint64_t> prev_counts,
                                        std::span<const TokenSeq> tokens, SimTime now) {
    const std::size_t n = group_ids.size();
    std::vector<std::int32_t> hs(n);
    std::vector<std::uint64_t> offs(n + 1, 0);
    TokenSeq flat;
    for (std::size_t i = 0; i < n; ++i) {
      hs[i] = handle(group_ids[i]);
      offs[i + 1] = offs[i] + tokens[i].size();
      flat.insert(flat.end(), tokens[i].begin(), tokens[i].end());
    }
    std::vector<dgds_update_reply> r(n);
    std::vector<std::int32_t> rids(request_ids.begin(), request_ids.end());
    detail::check(dgds_update_batch(s_, static_cast<int64_t>(n), hs.data(), rids.data(), prev_counts.data(),
                                    offs.data(), flat.data(), now, r.data()));
    std::vector<UpdateReply> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = UpdateReply{r[i].ok != 0, r[i].version, r[i].acked_tokens};
    return out;
  }

  void register_group(const std::string& group_id, double ttl_seconds, SimTime now) {
    detail::check(dgds_register_group(s_, handle(group_id), ttl_seconds, now));
  }
  void drop_group(const std::string& group_id) { detail::check(dgds_drop_group(s_, handle(group_id))); }
  void sweep_expired(SimTime now) { detail::check(dgds_sweep_expired(s_, now)); }

  std::vector<DraftCandidate> speculate(const std::string& group_id, std::span<const Token> pattern,
                                        const SpeculationArgs& args) {
    SpecQuery q{group_id, TokenSeq(pattern.begin(), pattern.end()), args};
    return batch_speculate(std::span<const SpecQuery>(&q, 1))[0];
  }

  // DraftClient::batch_speculate with fetch_period 0 (dgds.cpp:274-292): one device launch.
  std::vector<std::vector<DraftCandidate>> batch_speculate(std::span<const SpecQuery> queries) {
    const std::size_t n = queries.size();
    std::vector<std::vector<DraftCandidate>> out(n);
    if (n == 0) return out;
    std::vector<std::int32_t> hs(n);
    std::vector<std::uint64_t> offs(n + 1, 0);
    TokenSeq flat;
    std::vector<dgds_spec_args> args(n);
    int k = 1, s = 1;
    for (std::size_t i = 0; i < n; ++i) {
      hs[i] = handle(queries[i].group_id);
      offs[i + 1] = offs[i] + queries[i].pattern.size();
      flat.insert(flat.end(), queries[i].pattern.begin(), queries[i].pattern.end());
      args[i] = detail::c_args(queries[i].args);
      k = std::max(k, queries[i].args.top_k);
      s = std::max(s, std::min(queries[i].args.max_spec_tokens, params_.limits.max_spec_len));
    }
    std::vector<std::int32_t> nc(n), lens(n * k), toks(n * k * s);
    std::vector<double> scores(n * k);
    std::vector<std::int64_t> sup(n * k);
    dgds_candidates c{k, s, nc.data(), lens.data(), scores.data(), sup.data(), toks.data()};
    detail::check(dgds_speculate_batch(s_, static_cast<int64_t>(n), hs.data(), offs.data(), flat.data(), args.data(),
                                       1, &c));
    for (std::size_t q = 0; q < n; ++q)
      for (int j = 0; j < nc[q]; ++j) {
        const std::size_t i = q * k + j;
        out[q].push_back(DraftCandidate{TokenSeq(toks.begin() + i * s, toks.begin() + i * s + lens[i]), scores[i],
                                        static_cast<long long>(sup[i])});
      }
    return out;
  }

  // Asynchronous batch_speculate (dgds_speculate_submit / dgds_speculate_wait): the batch is
  // staged on the server's host workers and queued behind every update made before the call;
  // speculate_wait returns its results. The PendingBatch owns the flattened inputs the staging
  // reads, so it must outlive the wait; two batches can be in flight.
  class PendingBatch {
   public:
    std::uint64_t ticket() const { return ticket_; }
    std::size_t size() const { return in_ ? in_->hs.size() : 0; }

   private:
    friend class DraftServer;
    struct Inputs {
      std::vector<std::int32_t> hs;
      std::vector<std::uint64_t> offs;
      TokenSeq flat;
      std::vector<dgds_spec_args> args;
    };
    std::unique_ptr<Inputs> in_;  // stable addresses while the server stages them
    std::uint64_t ticket_ = 0;
  };

  PendingBatch speculate_submit(std::span<const SpecQuery> queries) {
    if (queries.empty()) throw std::invalid_argument("speculate_submit: empty batch");
    PendingBatch b;
    b.in_ = std::make_unique<PendingBatch::Inputs>();
    auto& in = *b.in_;
    const std::size_t n = queries.size();
    in.hs.resize(n);
    in.offs.assign(n + 1, 0);
    in.args.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
      in.hs[i] = handle(queries[i].group_id);
      in.offs[i + 1] = in.offs[i] + queries[i].pattern.size();
      in.flat.insert(in.flat.end(), queries[i].pattern.begin(), queries[i].pattern.end());
      in.args[i] = detail::c_args(queries[i].args);
    }
    detail::check(dgds_speculate_submit(s_, static_cast<int64_t>(n), in.hs.data(), in.offs.data(), in.flat.data(),
                                        in.args.data(), 1, nullptr, 0, nullptr, nullptr, &b.ticket_));
    return b;
  }

  std::vector<std::vector<DraftCandidate>> speculate_wait(const PendingBatch& b) {
    dgds_result_view v{};
    detail::check(dgds_speculate_wait(s_, b.ticket_, &v));
    std::vector<std::vector<DraftCandidate>> out(static_cast<std::size_t>(v.n_queries));
    for (int64_t q = 0; q < v.n_queries; ++q)
      for (int64_t c = v.cand_off[q]; c < v.cand_off[q + 1]; ++c)
        out[q].push_back(DraftCandidate{TokenSeq(v.tokens + v.tok_off[c], v.tokens + v.tok_off[c + 1]),
                                        v.cands[c].score, static_cast<long long>(v.cands[c].support)});
    return out;
  }

  // fetch_cst (dgds.cpp:53-97): UpToDate / Delta / Full / UnknownGroup per group.
  std::vector<FetchReply> fetch_cst(std::span<const std::string> group_ids, std::span<const DraftCacheInfo> infos,
                                    SimTime now) {
    if (group_ids.size() != infos.size())
      throw std::invalid_argument("fetch_cst: group_ids and draft_cache_infos must have equal length");
    const std::size_t n = group_ids.size();
    std::vector<FetchReply> out(n);
    if (n == 0) return out;
    std::vector<std::int32_t> hs(n);
    std::vector<std::uint64_t> cv(n);
    for (std::size_t i = 0; i < n; ++i) {
      hs[i] = handle(group_ids[i]);
      cv[i] = infos[i].cached_version;
    }
    std::vector<dgds_fetch_reply> r(n);
    const std::uint8_t* blobs = nullptr;
    detail::check(dgds_fetch_cst(s_, static_cast<int64_t>(n), hs.data(), cv.data(), now, r.data(), &blobs));
    for (std::size_t i = 0; i < n; ++i) {
      out[i].kind = static_cast<FetchKind>(r[i].kind);
      out[i].version = r[i].version;
      if (r[i].blob_len) out[i].blob.assign(blobs + r[i].blob_off, blobs + r[i].blob_off + r[i].blob_len);
    }
    return out;
  }
  void compact_group(const std::string& group_id, std::uint64_t before_version) {
    detail::check(dgds_compact_group(s_, handle(group_id), before_version));
  }
  // GroupDraftIndex::apply_blob on this server's copy of the group (a replica); returns its version.
  std::uint64_t apply_blob(const std::string& group_id, std::span<const std::uint8_t> blob, SimTime now = 0.0) {
    std::uint64_t v = 0;
    detail::check(dgds_apply_blob(s_, handle(group_id), blob.data(), blob.size(), now, &v));
    return v;
  }

  int shard_count() const { return params_.shard_count; }
  const DgdsParams& params() const { return params_; }
  bool has_group(const std::string& group_id) {
    std::int32_t r = 0;
    detail::check(dgds_has_group(s_, handle(group_id), &r));
    return r != 0;
  }
  std::uint64_t node_count() {  // the reference's node count over live groups (roots included)
    std::uint64_t v = 0;
    detail::check(dgds_node_count(s_, &v));
    return v;
  }
  std::uint64_t group_version(const std::string& group_id) {
    std::uint64_t v = 0;
    detail::check(dgds_group_version(s_, handle(group_id), &v));
    return v;
  }
  std::uint64_t stored_tokens(const std::string& group_id, int request_id) {
    std::uint64_t v = 0;
    detail::check(dgds_stored_tokens(s_, handle(group_id), request_id, &v));
    return v;
  }
  std::size_t shard_group_count(int shard) {
    std::uint64_t v = 0;
    detail::check(dgds_shard_group_count(s_, shard, &v));
    return static_cast<std::size_t>(v);
  }
  dgds_server* raw() { return s_; }

 private:
  std::int32_t handle(const std::string& gid) {
    auto it = handles_.find(gid);
    if (it != handles_.end()) return it->second;
    std::int32_t h = -1;
    detail::check(dgds_intern(s_, gid.data(), gid.size(), &h));
    handles_.emplace(gid, h);
    return h;
  }

  DgdsParams params_;
  dgds_server* s_ = nullptr;
  std::unordered_map<std::string, std::int32_t> handles_;
};

// N GPUs behind one DraftServer API: the reference's shards (dgds.cpp:10-51) as GPUs
// (dgds_cluster_*). Group g lives on GPU shard_of_group(g, n); batch calls run the GPUs
// concurrently and keep call order. Drop-in for rollsim::DraftServer's update / speculate /
// group calls with shard_count = the number of GPUs.
class ClusterServer {
 public:
  ClusterServer(DgdsParams params, std::vector<int> devices) : params_(params) {
    dgds_params p{};
    p.shard_count = params.shard_count;
    p.append_batch_tokens = params.append_batch_tokens;
    p.fetch_period = params.fetch_period;
    p.default_ttl_seconds = params.default_ttl_seconds;
    p.max_pattern_len = params.limits.max_pattern_len;
    p.max_spec_len = params.limits.max_spec_len;
    p.expected_nodes = params.expected_nodes;
    p.expected_streams = params.expected_streams;
    detail::check(dgds_cluster_create(&p, static_cast<std::int32_t>(devices.size()), devices.data(), &c_));
  }
  ~ClusterServer() { dgds_cluster_destroy(c_); }
  ClusterServer(const ClusterServer&) = delete;
  ClusterServer& operator=(const ClusterServer&) = delete;

  std::int32_t handle(const std::string& group_id) {
    auto it = handles_.find(group_id);
    if (it != handles_.end()) return it->second;
    std::int32_t h = 0;
    detail::check(dgds_cluster_intern(c_, group_id.data(), group_id.size(), &h));
    handles_.emplace(group_id, h);
    return h;
  }
  int owner_gpu(const std::string& group_id) {
    std::int32_t g = 0;
    detail::check(dgds_cluster_owner(c_, handle(group_id), &g));
    return g;
  }
  UpdateReply update_cst(const std::string& group_id, int request_id, std::uint64_t prev_token_count,
                         std::span<const Token> new_tokens, SimTime now) {
    const std::int32_t h = handle(group_id);
    const std::uint64_t offs[2] = {0, new_tokens.size()};
    dgds_update_reply r{};
    detail::check(dgds_cluster_update_batch(c_, 1, &h, &request_id, &prev_token_count, offs, new_tokens.data(), now,
                                            &r));
    return UpdateReply{r.ok != 0, r.version, r.acked_tokens};
  }
  void register_group(const std::string& group_id, double ttl_seconds, SimTime now) {
    detail::check(dgds_cluster_register_group(c_, handle(group_id), ttl_seconds, now));
  }
  void drop_group(const std::string& group_id) { detail::check(dgds_cluster_drop_group(c_, handle(group_id))); }
  void sweep_expired(SimTime now) { detail::check(dgds_cluster_sweep_expired(c_, now)); }
  bool has_group(const std::string& group_id) {
    std::int32_t v = 0;
    detail::check(dgds_cluster_has_group(c_, handle(group_id), &v));
    return v != 0;
  }
  std::uint64_t group_version(const std::string& group_id) {
    std::uint64_t v = 0;
    detail::check(dgds_cluster_group_version(c_, handle(group_id), &v));
    return v;
  }
  std::vector<DraftCandidate> speculate(const std::string& group_id, std::span<const Token> pattern,
                                        const SpeculationArgs& args) {
    SpecQuery q{group_id, TokenSeq(pattern.begin(), pattern.end()), args};
    return batch_speculate(std::span<const SpecQuery>(&q, 1))[0];
  }
  std::vector<std::vector<DraftCandidate>> batch_speculate(std::span<const SpecQuery> queries) {
    const std::size_t n = queries.size();
    std::vector<std::vector<DraftCandidate>> out(n);
    if (n == 0) return out;
    std::vector<std::int32_t> hs(n);
    std::vector<std::uint64_t> offs(n + 1, 0);
    std::vector<Token> pats;
    std::vector<dgds_spec_args> args(n);
    int K = 1, S = 1;
    for (std::size_t i = 0; i < n; ++i) {
      hs[i] = handle(queries[i].group_id);
      pats.insert(pats.end(), queries[i].pattern.begin(), queries[i].pattern.end());
      offs[i + 1] = pats.size();
      args[i] = detail::c_args(queries[i].args);
      K = std::max(K, queries[i].args.top_k);
      S = std::max(S, std::min(queries[i].args.max_spec_tokens, params_.limits.max_spec_len));
    }
    std::vector<std::int32_t> nc(n), lens(n * K), toks(n * K * S);
    std::vector<double> sc(n * K);
    std::vector<std::int64_t> sp(n * K);
    dgds_candidates c{K, S, nc.data(), lens.data(), sc.data(), sp.data(), toks.data()};
    detail::check(dgds_cluster_speculate_verify_batch(c_, static_cast<std::int64_t>(n), hs.data(), offs.data(),
                                                      pats.data(), args.data(), 1, nullptr, 0, nullptr, nullptr, &c,
                                                      nullptr));
    for (std::size_t i = 0; i < n; ++i)
      for (int j = 0; j < nc[i]; ++j) {
        const std::size_t at = i * K + j;
        DraftCandidate d;
        d.tokens.assign(toks.begin() + at * S, toks.begin() + at * S + lens[at]);
        d.score = sc[at];
        d.support = sp[at];
        out[i].push_back(std::move(d));
      }
    return out;
  }
  std::uint64_t node_count() {
    std::uint64_t v = 0;
    detail::check(dgds_cluster_node_count(c_, &v));
    return v;
  }

 private:
  DgdsParams params_;
  dgds_cluster* c_ = nullptr;
  std::unordered_map<std::string, std::int32_t> handles_;
};

// Transport seam between DraftClient and the server (dgds.hpp:93-116): in-process calls
// (LocalTransport) or any other implementation (e.g. the framed wire protocol).
class DraftTransport {
 public:
  virtual ~DraftTransport() = default;
  virtual UpdateReply update_cst(const std::string& group_id, int request_id, std::uint64_t prev_token_count,
                                 std::span<const Token> new_tokens, SimTime now) = 0;
  virtual std::vector<FetchReply> fetch_cst(std::span<const std::string> group_ids,
                                            std::span<const DraftCacheInfo> infos, SimTime now) = 0;
  virtual void register_group(const std::string& group_id, double ttl_seconds, SimTime now) = 0;
};

class LocalTransport final : public DraftTransport {  // dgds.hpp:105-116
 public:
  explicit LocalTransport(DraftServer& server) : server_(server) {}
  UpdateReply update_cst(const std::string& group_id, int request_id, std::uint64_t prev_token_count,
                         std::span<const Token> new_tokens, SimTime now) override {
    return server_.update_cst(group_id, request_id, prev_token_count, new_tokens, now);
  }
  std::vector<FetchReply> fetch_cst(std::span<const std::string> group_ids, std::span<const DraftCacheInfo> infos,
                                    SimTime now) override {
    return server_.fetch_cst(group_ids, infos, now);
  }
  void register_group(const std::string& group_id, double ttl_seconds, SimTime now) override {
    server_.register_group(group_id, ttl_seconds, now);
  }
  DraftServer& server() { return server_; }

 private:
  DraftServer& server_;
};

// DraftClient (dgds.hpp:128-162, dgds.cpp:186-297) over a DraftTransport. note_tokens batches
// appends per (group, request) and flushes at append_batch_tokens with the resync rules of
// push_stream (dgds.cpp:193-217). batch_speculate answers from replicas of the queried groups,
// kept in a GPU replica server and synced with GDX1 delta / full blobs (cst.cpp:233-329):
// - fetch_period == 0 (always fresh): the queried groups are fetched first on every call;
// - fetch_period > 0: fetch_active() syncs the active groups (stale between fetches, as in the
//   paper's periodic fetch).
// Over a LocalTransport in fresh mode the just-fetched replica would equal the server's own
// index, so the server answers directly (same results, no blob round trip).
class DraftClient {
 public:
  DraftClient(DraftTransport& transport, DgdsParams params) : transport_(transport), params_(params) {
    local_ = dynamic_cast<LocalTransport*>(&transport_);
    if (params_.fetch_period > 0.0 || !local_) {
      DgdsParams rp = params_;
      rp.default_ttl_seconds = 1e300;  // replicas live until dropped or told UnknownGroup
      replica_ = std::make_unique<DraftServer>(rp);
    }
  }
  // Convenience: a client of a server in this process (owns its LocalTransport).
  DraftClient(DraftServer& server, DgdsParams params)
      : own_(std::make_unique<LocalTransport>(server)), transport_(*own_), params_(params) {
    local_ = own_.get();
    if (params_.fetch_period > 0.0) {
      DgdsParams rp = params_;
      rp.default_ttl_seconds = 1e300;
      replica_ = std::make_unique<DraftServer>(rp);
    }
  }

  void register_group(const std::string& group_id, double ttl_seconds, SimTime now) {
    transport_.register_group(group_id, ttl_seconds, now);
  }
  void note_tokens(const std::string& group_id, int request_id, std::span<const Token> tokens, SimTime now) {
    if (tokens.empty()) return;
    Pending& ps = pending_[{group_id, request_id}];
    ps.buf.insert(ps.buf.end(), tokens.begin(), tokens.end());
    if (ps.buf.size() - ps.acked >= static_cast<std::size_t>(params_.append_batch_tokens))
      push(group_id, request_id, ps, now);
  }
  void flush(SimTime now) {
    for (auto& [key, ps] : pending_)
      if (ps.acked < ps.buf.size()) push(key.first, key.second, ps, now);
  }

  void set_active_groups(std::vector<std::string> group_ids) {  // dgds.cpp:224-228
    std::sort(group_ids.begin(), group_ids.end());
    group_ids.erase(std::unique(group_ids.begin(), group_ids.end()), group_ids.end());
    active_ = std::move(group_ids);
  }
  bool fetch_due(SimTime now) const {  // dgds.cpp:230-233
    if (active_.empty()) return false;
    return last_fetch_ < 0.0 || now - last_fetch_ >= params_.fetch_period;
  }
  void fetch_active(SimTime now) {  // dgds.cpp:265-268
    fetch_groups(active_, now);
    last_fetch_ = now;
  }
  void drop_replica(const std::string& group_id) {
    cached_.erase(group_id);
    if (replica_) replica_->drop_group(group_id);
  }
  std::uint64_t cached_version(const std::string& group_id) const {
    auto it = cached_.find(group_id);
    return it == cached_.end() ? 0 : it->second;
  }
  const DgdsParams& params() const { return params_; }

  std::vector<std::vector<DraftCandidate>> batch_speculate(std::span<const SpecQuery> queries, SimTime now) {
    std::vector<std::vector<DraftCandidate>> out(queries.size());
    if (queries.empty()) return out;
    if (params_.fetch_period <= 0.0) {  // fresh mode: sync the queried groups first (dgds.cpp:277-282)
      std::vector<std::string> ids;
      for (const auto& q : queries) ids.push_back(q.group_id);
      std::sort(ids.begin(), ids.end());
      ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
      if (local_ && !replica_) {  // the server's own index is what the replica would hold
        std::vector<DraftCacheInfo> infos;
        for (const auto& g : ids) infos.push_back(DraftCacheInfo{g, local_->server().group_version(g)});
        auto reps = local_->fetch_cst(ids, infos, now);  // lazy expiry + TTL refresh, no blob (up to date)
        std::vector<SpecQuery> live;
        std::vector<std::size_t> where;
        for (std::size_t i = 0; i < queries.size(); ++i) {
          const auto k = std::lower_bound(ids.begin(), ids.end(), queries[i].group_id) - ids.begin();
          if (reps[k].kind == FetchKind::UnknownGroup) continue;  // no replica -> empty candidates
          cached_[queries[i].group_id] = reps[k].version;
          live.push_back(queries[i]);
          where.push_back(i);
        }
        auto got = local_->server().batch_speculate(live);
        for (std::size_t j = 0; j < where.size(); ++j) out[where[j]] = std::move(got[j]);
        for (std::size_t k = 0; k < ids.size(); ++k)
          if (reps[k].kind == FetchKind::UnknownGroup) cached_.erase(ids[k]);
        return out;
      }
      fetch_groups(ids, now);
    }
    std::vector<SpecQuery> have;
    std::vector<std::size_t> where;
    for (std::size_t i = 0; i < queries.size(); ++i) {
      if (!cached_.count(queries[i].group_id)) continue;  // no replica -> empty candidates
      have.push_back(queries[i]);
      where.push_back(i);
    }
    auto got = replica_->batch_speculate(have);
    for (std::size_t j = 0; j < where.size(); ++j) out[where[j]] = std::move(got[j]);
    return out;
  }

 private:
  struct Pending {
    TokenSeq buf;
    std::uint64_t acked = 0;
  };
  void fetch_groups(const std::vector<std::string>& ids, SimTime now) {  // dgds.cpp:235-263
    if (ids.empty()) return;
    std::vector<DraftCacheInfo> infos;
    for (const auto& g : ids) infos.push_back(DraftCacheInfo{g, cached_version(g)});
    auto reps = transport_.fetch_cst(ids, infos, now);
    for (std::size_t i = 0; i < ids.size(); ++i) {
      FetchReply& r = reps[i];
      switch (r.kind) {
        case FetchKind::UpToDate:
          break;
        case FetchKind::UnknownGroup:
          drop_replica(ids[i]);
          break;
        case FetchKind::Delta:
          if (!cached_.count(ids[i])) throw std::runtime_error("delta for group without replica: " + ids[i]);
          cached_[ids[i]] = replica_ ? replica_->apply_blob(ids[i], r.blob, now) : r.version;
          break;
        case FetchKind::Full:
          cached_[ids[i]] = replica_ ? replica_->apply_blob(ids[i], r.blob, now) : r.version;
          break;
      }
    }
  }
  void push(const std::string& gid, int rid, Pending& ps, SimTime now) {  // push_stream, dgds.cpp:193-208
    while (ps.acked < ps.buf.size()) {
      std::span<const Token> chunk(ps.buf.data() + ps.acked, ps.buf.size() - ps.acked);
      UpdateReply rep = transport_.update_cst(gid, rid, ps.acked, chunk, now);
      if (rep.ok) {
        ps.acked = rep.acked_tokens;
      } else if (rep.acked_tokens > ps.acked && rep.acked_tokens <= ps.buf.size()) {
        ps.acked = rep.acked_tokens;
      } else if (rep.acked_tokens < ps.acked) {
        ps.acked = rep.acked_tokens;
      } else {
        throw std::runtime_error("draft append resync cannot make progress for group " + gid);
      }
    }
  }
  std::unique_ptr<LocalTransport> own_;  // the DraftServer& constructor's transport
  DraftTransport& transport_;
  LocalTransport* local_ = nullptr;
  DgdsParams params_;
  std::unique_ptr<DraftServer> replica_;  // GPU-resident replicas
  std::map<std::pair<std::string, int>, Pending> pending_;
  std::vector<std::string> active_;
  SimTime last_fetch_ = -1.0;
  std::map<std::string, std::uint64_t> cached_;
};

// The engine seam the reference declares but never implements (engine.hpp:67-74).
class GpuSpeculationSource {
 public:
  explicit GpuSpeculationSource(DraftClient& client) : client_(client) {}
  std::vector<std::vector<DraftCandidate>> batch(std::span<const SpecQuery> queries, SimTime now) {
    return client_.batch_speculate(queries, now);
  }
  void on_emitted(const std::string& group_id, int request_id, std::span<const Token> tokens, SimTime now) {
    client_.note_tokens(group_id, request_id, tokens, now);
  }

 private:
  DraftClient& client_;
};

}  // namespace dgds_b200

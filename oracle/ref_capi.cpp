// ref_capi.cpp — extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. Compiled together with /root/reference/proj/src/*.cpp
// by oracle/Makefile into oracle/_ref/libdgds_ref.so; it lets the Python tests,
// golden-fixture generator and bench.py's reference arm call the reference's own
// GroupDraftIndex / speculate_oracle / DraftServer / DraftClient / Instance /
// generate_workload through plain C types. No reference logic is restated here:
// every computation is a call into the reference code.

#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oracle_capi.h"
#include "rollsim/cst.hpp"
#include "rollsim/detail/bytes.hpp"
#include "rollsim/detail/rng.hpp"
#include "rollsim/dgds.hpp"
#include "rollsim/dgds_wire.hpp"
#include "rollsim/engine.hpp"
#include "rollsim/kvpool.hpp"
#include "rollsim/workload.hpp"

using namespace rollsim;

namespace {

thread_local std::string g_err;

SpeculationArgs to_args(const orc_args* a) {
  SpeculationArgs s;
  s.max_spec_tokens = a->max_spec_tokens;
  s.pattern_lookup_max = a->pattern_lookup_max;
  s.pattern_lookup_min = a->pattern_lookup_min;
  s.top_k = a->top_k;
  s.min_step_freq = a->min_step_freq;
  s.min_support = a->min_support;
  return s;
}

int write_cands(const std::vector<DraftCandidate>& c, orc_cands* out) {
  out->n = 0;
  for (const auto& d : c) {
    if (out->n >= out->k_cap || static_cast<int>(d.tokens.size()) > out->s_cap) {
      g_err = "candidate buffer too small";
      return -1;
    }
    int i = out->n++;
    std::memcpy(out->tokens + static_cast<std::size_t>(i) * out->s_cap, d.tokens.data(),
                d.tokens.size() * sizeof(int32_t));
    out->lens[i] = static_cast<int32_t>(d.tokens.size());
    out->scores[i] = d.score;
    out->supports[i] = d.support;
  }
  return 0;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // namespace

namespace {
struct GroupSet {
  std::vector<std::unique_ptr<GroupDraftIndex>> idx;
};

template <class F>
void for_groups(int64_t n, const int32_t* group, int32_t ngroups, int32_t threads, F&& f) {
  const int T = std::max(1, std::min<int32_t>(threads, ngroups));
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (int64_t i = 0; i < n; ++i)
        if (group[i] % T == t) f(i);
    });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// GroupDraftIndex

void* orc_index_new(const char* group_id, int32_t max_pattern_len, int32_t max_spec_len) {
  try {
    GroupDraftIndex::Limits lim;
    lim.max_pattern_len = max_pattern_len;
    lim.max_spec_len = max_spec_len;
    return new GroupDraftIndex(group_id, lim);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_index_free(void* idx) { delete static_cast<GroupDraftIndex*>(idx); }

int orc_index_append(void* idx, int32_t request_id, uint64_t prev, const int32_t* toks, uint64_t n,
                     int32_t* ok, uint64_t* version, uint64_t* acked) {
  return guarded([&] {
    auto r = static_cast<GroupDraftIndex*>(idx)->append(request_id, prev, std::span<const Token>(toks, n));
    *ok = r.ok ? 1 : 0;
    *version = r.version;
    *acked = r.acked_tokens;
    return 0;
  });
}

int orc_index_speculate(const void* idx, const int32_t* pattern, uint64_t plen, const orc_args* args,
                        orc_cands* out) {
  return guarded([&] {
    auto c = static_cast<const GroupDraftIndex*>(idx)->speculate(std::span<const Token>(pattern, plen),
                                                                  to_args(args));
    return write_cands(c, out);
  });
}

uint64_t orc_index_version(const void* idx) { return static_cast<const GroupDraftIndex*>(idx)->version(); }
uint64_t orc_index_node_count(const void* idx) {
  return static_cast<const GroupDraftIndex*>(idx)->node_count();
}
uint64_t orc_index_stored_tokens(const void* idx, int32_t request_id) {
  return static_cast<const GroupDraftIndex*>(idx)->stored_tokens(request_id);
}

int orc_oracle_speculate(const int32_t* toks, const uint64_t* offsets, uint64_t nseq, const int32_t* pattern,
                         uint64_t plen, const orc_args* args, orc_cands* out) {
  return guarded([&] {
    std::vector<TokenSeq> seqs(nseq);
    for (uint64_t i = 0; i < nseq; ++i) seqs[i].assign(toks + offsets[i], toks + offsets[i + 1]);
    auto c = speculate_oracle(seqs, std::span<const Token>(pattern, plen), to_args(args));
    return write_cands(c, out);
  });
}

// The instrumented variant exists only in the restatement.
int orc_index_speculate_stats(const void*, const int32_t*, uint64_t, const orc_args*, orc_cands*, orc_qstats*) {
  g_err = "speculate_stats is provided by liboracle.so only";
  return -1;
}

// ---------------------------------------------------------------------------
// A set of GroupDraftIndex objects driven in bulk (scale parity tests): records and queries
// of different groups are independent, so they are split over threads by group; inside a
// group the records apply in array order, exactly as sequential append calls would.

void* orc_ref_gset_new(int32_t ngroups, const char* const* gids, int32_t max_pattern_len, int32_t max_spec_len) {
  try {
    auto* g = new GroupSet;
    GroupDraftIndex::Limits lim;
    lim.max_pattern_len = max_pattern_len;
    lim.max_spec_len = max_spec_len;
    for (int32_t i = 0; i < ngroups; ++i) g->idx.push_back(std::make_unique<GroupDraftIndex>(gids[i], lim));
    return g;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_ref_gset_free(void* g) { delete static_cast<GroupSet*>(g); }

int orc_ref_gset_append(void* gs, int64_t n, const int32_t* group, const int32_t* rid, const uint64_t* prev,
                        const uint64_t* offs, const int32_t* tokens, int32_t threads, int32_t* ok,
                        uint64_t* version, uint64_t* acked) {
  auto* g = static_cast<GroupSet*>(gs);
  std::atomic<int> bad{0};
  for_groups(n, group, static_cast<int32_t>(g->idx.size()), threads, [&](int64_t i) {
    try {
      auto r = g->idx[group[i]]->append(rid[i], prev[i], std::span<const Token>(tokens + offs[i], offs[i + 1] - offs[i]));
      ok[i] = r.ok ? 1 : 0;
      version[i] = r.version;
      acked[i] = r.acked_tokens;
    } catch (const std::exception&) {
      bad = 1;
    }
  });
  if (bad) {
    g_err = "reference append threw";
    return -1;
  }
  return 0;
}

int orc_ref_gset_speculate(void* gs, int64_t n, const int32_t* group, const uint64_t* pat_offs, const int32_t* pats,
                           const orc_args* args, int32_t threads, int32_t k_cap, int32_t s_cap, int32_t* n_cands,
                           int32_t* lens, double* scores, int64_t* supports, int32_t* tokens) {
  auto* g = static_cast<GroupSet*>(gs);
  std::atomic<int> bad{0};
  for_groups(n, group, static_cast<int32_t>(g->idx.size()), threads, [&](int64_t i) {
    try {
      auto c = g->idx[group[i]]->speculate(std::span<const Token>(pats + pat_offs[i], pat_offs[i + 1] - pat_offs[i]),
                                            to_args(args + i));
      orc_cands out{tokens + i * static_cast<int64_t>(k_cap) * s_cap, lens + i * static_cast<int64_t>(k_cap),
                    scores + i * static_cast<int64_t>(k_cap), supports + i * static_cast<int64_t>(k_cap), k_cap,
                    s_cap, 0};
      if (write_cands(c, &out)) bad = 1;
      n_cands[i] = out.n;
    } catch (const std::exception&) {
      bad = 1;
    }
  });
  if (bad) {
    g_err = "reference speculate threw or overflowed the candidate buffer";
    return -1;
  }
  return 0;
}

uint64_t orc_ref_gset_node_count(const void* gs) {
  uint64_t n = 0;
  for (const auto& x : static_cast<const GroupSet*>(gs)->idx) n += x->node_count();
  return n;
}

// ---------------------------------------------------------------------------
// DraftServer (dgds.hpp:51-91)

int32_t orc_ref_shard_of_group(const char* gid, int32_t shard_count) {
  try {
    return shard_of_group(gid, shard_count);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

uint64_t orc_ref_fnv1a64(const void* data, uint64_t n) { return detail::fnv1a64(data, n); }

void* orc_ref_server_new(int32_t shard_count, double fetch_period, int32_t append_batch_tokens, double ttl,
                         int32_t max_pattern_len, int32_t max_spec_len) {
  try {
    DgdsParams p;
    p.shard_count = shard_count;
    p.fetch_period = fetch_period;
    p.append_batch_tokens = append_batch_tokens;
    p.default_ttl_seconds = ttl;
    p.limits.max_pattern_len = max_pattern_len;
    p.limits.max_spec_len = max_spec_len;
    return new DraftServer(p);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_ref_server_free(void* s) { delete static_cast<DraftServer*>(s); }

int orc_ref_server_update(void* s, const char* gid, int32_t rid, uint64_t prev, const int32_t* toks, uint64_t n,
                          double now, int32_t* ok, uint64_t* version, uint64_t* acked) {
  return guarded([&] {
    auto r = static_cast<DraftServer*>(s)->update_cst(gid, rid, prev, std::span<const Token>(toks, n), now);
    *ok = r.ok ? 1 : 0;
    *version = r.version;
    *acked = r.acked_tokens;
    return 0;
  });
}

int orc_ref_server_speculate(const void* s, const char* gid, const int32_t* pattern, uint64_t plen,
                             const orc_args* args, orc_cands* out) {
  return guarded([&] {
    auto c = static_cast<const DraftServer*>(s)->speculate(gid, std::span<const Token>(pattern, plen),
                                                           to_args(args));
    return write_cands(c, out);
  });
}

int orc_ref_server_register(void* s, const char* gid, double ttl, double now) {
  return guarded([&] {
    static_cast<DraftServer*>(s)->register_group(gid, ttl, now);
    return 0;
  });
}

int orc_ref_server_drop(void* s, const char* gid) {
  return guarded([&] {
    static_cast<DraftServer*>(s)->drop_group(gid);
    return 0;
  });
}

int orc_ref_server_sweep(void* s, double now) {
  return guarded([&] {
    static_cast<DraftServer*>(s)->sweep_expired(now);
    return 0;
  });
}

int32_t orc_ref_server_has_group(const void* s, const char* gid) {
  return static_cast<const DraftServer*>(s)->has_group(gid) ? 1 : 0;
}

uint64_t orc_ref_server_group_version(const void* s, const char* gid) {
  return static_cast<const DraftServer*>(s)->group_version(gid);
}

uint64_t orc_ref_server_shard_group_count(const void* s, int32_t shard) {
  return static_cast<const DraftServer*>(s)->shard_group_count(shard);
}

// ---------------------------------------------------------------------------
// replica sync (GDX1 blobs): fetch_cst / compact_group on the server, and
// full_snapshot / delta_since / apply_blob on a GroupDraftIndex. Blobs are
// copied into caller buffers; *len is always the full size (-2 = too small).

namespace {
int copy_blob(const std::vector<std::uint8_t>& b, uint8_t* buf, uint64_t cap, uint64_t* len) {
  *len = b.size();
  if (b.size() > cap) {
    g_err = "blob buffer too small";
    return -2;
  }
  if (!b.empty()) std::memcpy(buf, b.data(), b.size());
  return 0;
}
}  // namespace

int orc_ref_server_fetch(void* s, const char* gid, uint64_t cached, double now, int32_t* kind, uint64_t* version,
                         uint8_t* buf, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    std::string id(gid);
    DraftCacheInfo info{id, cached};
    auto r = static_cast<DraftServer*>(s)->fetch_cst(std::span<const std::string>(&id, 1),
                                                     std::span<const DraftCacheInfo>(&info, 1), now);
    *kind = static_cast<int32_t>(r[0].kind);
    *version = r[0].version;
    return copy_blob(r[0].blob, buf, cap, len);
  });
}

int orc_ref_server_compact(void* s, const char* gid, uint64_t before) {
  return guarded([&] {
    static_cast<DraftServer*>(s)->compact_group(gid, before);
    return 0;
  });
}

int orc_index_full_snapshot(const void* idx, uint8_t* buf, uint64_t cap, uint64_t* len) {
  return guarded([&] { return copy_blob(static_cast<const GroupDraftIndex*>(idx)->full_snapshot(), buf, cap, len); });
}

int orc_index_delta_since(const void* idx, uint64_t since, int32_t* available, uint8_t* buf, uint64_t cap,
                          uint64_t* len) {
  return guarded([&] {
    auto d = static_cast<const GroupDraftIndex*>(idx)->delta_since(since);
    *available = d.has_value() ? 1 : 0;
    *len = 0;
    return d.has_value() ? copy_blob(*d, buf, cap, len) : 0;
  });
}

int orc_index_apply_blob(void* idx, const uint8_t* blob, uint64_t len, uint64_t* version) {
  return guarded([&] {
    *version = static_cast<GroupDraftIndex*>(idx)->apply_blob(std::span<const std::uint8_t>(blob, len));
    return 0;
  });
}

int orc_index_compact(void* idx, uint64_t before) {
  return guarded([&] {
    static_cast<GroupDraftIndex*>(idx)->compact_log(before);
    return 0;
  });
}

// ---------------------------------------------------------------------------
// framed wire protocol (dgds_wire.cpp): serve_payload, the TcpTransport client and
// the TcpDraftService, to check our service and client against the reference.

int orc_ref_wire_serve(void* s, const uint8_t* payload, uint64_t len, double now, uint8_t* out, uint64_t cap,
                       uint64_t* out_len) {
  return guarded([&] {
    auto r = wire::serve_payload(*static_cast<DraftServer*>(s), std::span<const std::uint8_t>(payload, len), now);
    return copy_blob(r, out, cap, out_len);
  });
}

void* orc_ref_tcp_new(const char* host, int32_t port) {
  try {
    return new wire::TcpTransport(host, port);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_ref_tcp_free(void* t) { delete static_cast<wire::TcpTransport*>(t); }

int orc_ref_tcp_update(void* t, const char* gid, int32_t rid, uint64_t prev, const int32_t* toks, uint64_t n,
                       int32_t* ok, uint64_t* version, uint64_t* acked) {
  return guarded([&] {
    auto r = static_cast<wire::TcpTransport*>(t)->update_cst(gid, rid, prev, std::span<const Token>(toks, n), 0.0);
    *ok = r.ok ? 1 : 0;
    *version = r.version;
    *acked = r.acked_tokens;
    return 0;
  });
}

int orc_ref_tcp_fetch(void* t, const char* gid, uint64_t cached, int32_t* kind, uint64_t* version, uint8_t* buf,
                      uint64_t cap, uint64_t* len) {
  return guarded([&] {
    std::string id(gid);
    DraftCacheInfo info{id, cached};
    auto r = static_cast<wire::TcpTransport*>(t)->fetch_cst(std::span<const std::string>(&id, 1),
                                                            std::span<const DraftCacheInfo>(&info, 1), 0.0);
    *kind = static_cast<int32_t>(r[0].kind);
    *version = r[0].version;
    return copy_blob(r[0].blob, buf, cap, len);
  });
}

int orc_ref_tcp_register(void* t, const char* gid, double ttl) {
  return guarded([&] {
    static_cast<wire::TcpTransport*>(t)->register_group(gid, ttl, 0.0);
    return 0;
  });
}

void* orc_ref_service_new(int32_t port) {
  try {
    return new wire::TcpDraftService(DgdsParams{}, port);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int32_t orc_ref_service_port(void* sv) { return static_cast<wire::TcpDraftService*>(sv)->port(); }

void orc_ref_service_free(void* sv) { delete static_cast<wire::TcpDraftService*>(sv); }

// ---------------------------------------------------------------------------
// generate_workload (workload.cpp:51-103)

typedef struct orc_wcfg {
  int32_t num_groups;
  int32_t group_size;
  int32_t length_family;  // 0 lognormal, 1 pareto
  int32_t vocab_size;
  double location;
  double scale;
  double group_correlation;
  double noise_base;
  double pattern_similarity;
  double prompt_mean;
  double prompt_spread;
  int32_t max_tokens;
  int32_t pad_;
  uint64_t seed;
} orc_wcfg;

struct RefTrace {
  std::vector<PromptGroup> groups;
};

void* orc_ref_workload_new(const orc_wcfg* c) {
  try {
    WorkloadConfig w;
    w.num_groups = c->num_groups;
    w.group_size = c->group_size;
    w.length_model.family = c->length_family == 0 ? LengthFamily::Lognormal : LengthFamily::Pareto;
    w.length_model.location = c->location;
    w.length_model.scale = c->scale;
    w.length_model.group_correlation = c->group_correlation;
    w.length_model.noise_base = c->noise_base;
    w.pattern_similarity = c->pattern_similarity;
    w.vocab_size = c->vocab_size;
    w.max_tokens = c->max_tokens;
    w.prompt_len_model.mean = c->prompt_mean;
    w.prompt_len_model.spread = c->prompt_spread;
    w.seed = c->seed;
    auto* t = new RefTrace;
    t->groups = generate_workload(w);
    return t;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_ref_workload_free(void* t) { delete static_cast<RefTrace*>(t); }
int32_t orc_ref_workload_num_groups(const void* t) {
  return static_cast<int32_t>(static_cast<const RefTrace*>(t)->groups.size());
}
const char* orc_ref_workload_group_id(const void* t, int32_t g) {
  return static_cast<const RefTrace*>(t)->groups[g].group_id.c_str();
}
int32_t orc_ref_workload_prompt_len(const void* t, int32_t g) {
  return static_cast<const RefTrace*>(t)->groups[g].prompt_len;
}
int32_t orc_ref_workload_group_size(const void* t, int32_t g) {
  return static_cast<int32_t>(static_cast<const RefTrace*>(t)->groups[g].outputs.size());
}
int64_t orc_ref_workload_output_len(const void* t, int32_t g, int32_t i) {
  return static_cast<int64_t>(static_cast<const RefTrace*>(t)->groups[g].outputs[i].size());
}
const int32_t* orc_ref_workload_output(const void* t, int32_t g, int32_t i) {
  return static_cast<const RefTrace*>(t)->groups[g].outputs[i].data();
}
uint64_t orc_ref_workload_fingerprint(const void* t) {
  return trace_fingerprint(static_cast<const RefTrace*>(t)->groups);
}

// ---------------------------------------------------------------------------
// Staggered engine replay through the reference Instance::decode_step
// (engine.cpp:69-167) with the reference DraftClient (fetch_period 0) over a
// LocalTransport to a reference DraftServer as the SpeculationSource — the
// adapter the reference declares (engine.hpp:67-74) but never ships.

namespace {

class ClientSource final : public SpeculationSource {
 public:
  explicit ClientSource(DraftClient& c) : client_(c) {}
  std::vector<std::vector<DraftCandidate>> batch(std::span<const SpecQuery> q, SimTime now) override {
    queries_ += q.size();
    return client_.batch_speculate(q, now);
  }
  void on_emitted(const std::string& gid, int rid, std::span<const Token> toks, SimTime now) override {
    client_.note_tokens(gid, rid, toks, now);
  }
  uint64_t queries_ = 0;

 private:
  DraftClient& client_;
};

}  // namespace

typedef struct orc_replay_cfg {
  int32_t stagger_steps;        // request r of every group is admitted at step r*stagger
  int32_t append_batch_tokens;  // DraftClient flush threshold (dgds.hpp:21)
  int32_t batch_token_budget;   // AdaptiveSpecPolicy (engine.hpp:28-33)
  int32_t per_request_cap;
  int32_t adaptive_enabled;
  int32_t multi_path_k;
  int32_t max_pattern_len;  // Limits
  int32_t max_spec_len;
  int32_t max_steps;
  int32_t pad_;
  orc_args args;  // lookup bounds and cutoffs (max_spec_tokens/top_k overridden per step)
} orc_replay_cfg;

// Output: per step the batch size; per (step, running request) the record
// {slot, drafted, accepted, emitted}. Returns the number of steps, or -1.
int64_t orc_ref_replay(const void* trace, const orc_replay_cfg* cfg, int32_t* step_batch, int64_t step_cap,
                       int32_t* rec, int64_t rec_cap, int64_t* n_rec, uint64_t* n_queries) {
  try {
    const auto& groups = static_cast<const RefTrace*>(trace)->groups;
    KvParams kp;
    kp.instance_capacity_tokens = 1ull << 50;
    kp.dram_capacity_tokens = 1ull << 50;
    kp.ssd_capacity_tokens = 1ull << 50;
    KvPool pool(kp, 1);
    StepTimeModel sm;
    sm.batch_cap = 1 << 30;
    Instance inst(0, sm, 1ull << 50, pool, /*divided=*/false);

    DgdsParams dp;
    dp.fetch_period = 0.0;
    dp.append_batch_tokens = cfg->append_batch_tokens;
    dp.limits.max_pattern_len = cfg->max_pattern_len;
    dp.limits.max_spec_len = cfg->max_spec_len;
    DraftServer server(dp);
    LocalTransport lt(server);
    DraftClient client(lt, dp);
    ClientSource src(client);

    SpecConfig spec;
    spec.sd_enabled = true;
    spec.adaptive.batch_token_budget = cfg->batch_token_budget;
    spec.adaptive.per_request_cap = cfg->per_request_cap;
    spec.adaptive.enabled = cfg->adaptive_enabled != 0;
    spec.adaptive.multi_path_k = cfg->multi_path_k;
    spec.args = to_args(&cfg->args);

    std::vector<std::unique_ptr<SimRequest>> reqs;
    int max_g = 0;
    for (const auto& g : groups) max_g = std::max<int>(max_g, static_cast<int>(g.outputs.size()));
    for (std::size_t gi = 0; gi < groups.size(); ++gi) {
      for (std::size_t i = 0; i < groups[gi].outputs.size(); ++i) {
        auto r = std::make_unique<SimRequest>();
        r->meta.group_id = groups[gi].group_id;
        r->meta.request_index = static_cast<int>(i);
        r->meta.prompt_len = groups[gi].prompt_len;
        r->meta.ori_max_tokens = groups[gi].max_tokens;
        r->truth = &groups[gi].outputs[i];
        r->slot = static_cast<int>(gi * max_g + i);
        reqs.push_back(std::move(r));
      }
    }
    SimTime now = 0.0;
    int64_t steps = 0, nrec = 0;
    std::size_t finished = 0;
    while (finished < reqs.size() && steps < cfg->max_steps) {
      for (auto& r : reqs) {
        if (r->meta.state == RequestState::Pending &&
            static_cast<int64_t>(r->meta.request_index) * cfg->stagger_steps == steps) {
          double delay = 0;
          if (inst.admit(*r, static_cast<int>(r->truth->size()), now, &delay) != Instance::AdmitOutcome::Accept)
            throw std::runtime_error("replay admit refused");
          inst.make_ready(*r);
        }
      }
      if (inst.running().empty()) {
        ++steps;
        if (steps <= step_cap) step_batch[steps - 1] = 0;
        continue;
      }
      StepReport rep = inst.decode_step(&src, spec, now);
      now += rep.duration;
      if (steps < step_cap) step_batch[steps] = rep.batch;
      for (const auto& p : rep.per_request) {
        if (nrec < rec_cap) {
          rec[4 * nrec + 0] = p.slot;
          rec[4 * nrec + 1] = p.drafted;
          rec[4 * nrec + 2] = p.accepted;
          rec[4 * nrec + 3] = p.emitted;
        }
        ++nrec;
      }
      std::vector<SimRequest*> running(inst.running().begin(), inst.running().end());
      for (SimRequest* r : running) {
        if (r->remaining_truth() == 0 || r->remaining_chunk() == 0) {
          inst.finish_or_requeue(*r, now);
          if (r->meta.state == RequestState::Finished) ++finished;
        }
      }
      ++steps;
    }
    *n_rec = nrec;
    *n_queries = src.queries_;
    return steps;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"

extern "C" {

// ---------------------------------------------------------------------------
// CPU baseline: the reference GroupDraftIndex driven thread-per-shard over the
// host cores: groups are partitioned by the reference
// shard_of_group(gid, T); every thread owns its shard's indexes, so there is no
// locking. Phases per step: append (one record per stream) then queries with
// verification (engine.cpp:115-143 rule), each bracketed by a barrier and
// timed with steady_clock.

typedef struct orc_bench_cfg {
  int32_t threads;
  int32_t n_streams;      // streams in the sample (group-major)
  int32_t group_size;
  int32_t steps;          // timed + warmup steps provided in the schedule
  int32_t record_tokens;  // tokens per append record (DraftClient flush size)
  int32_t queries_per_step;
  int32_t max_pattern_len, max_spec_len;  // Limits
  int32_t pad_;
  orc_args args;
} orc_bench_cfg;

// out[0] prefill seconds, out[1] prefill tokens, then per step s:
// out[2+4s] append seconds, out[3+4s] tokens appended, out[4+4s] query seconds, out[5+4s] queries
int orc_ref_bench(const orc_bench_cfg* cfg, const char* const* gids, const int32_t* tokens, const int64_t* offsets,
                  const int64_t* prefill, const int32_t* q_stream, const int64_t* q_pos, double* out) {
  try {
    const int T = std::max(1, cfg->threads);
    const int S = cfg->n_streams, G = cfg->group_size;
    const int ngroups = S / G;
    GroupDraftIndex::Limits lim;
    lim.max_pattern_len = cfg->max_pattern_len;
    lim.max_spec_len = cfg->max_spec_len;
    std::vector<std::unique_ptr<GroupDraftIndex>> idx(ngroups);
    std::vector<int> owner(ngroups);
    std::vector<std::vector<int>> mine(T);
    for (int g = 0; g < ngroups; ++g) {
      idx[g] = std::make_unique<GroupDraftIndex>(gids[g], lim);
      owner[g] = shard_of_group(gids[g], T);
      mine[owner[g]].push_back(g);
    }
    const SpeculationArgs a = to_args(&cfg->args);
    const int rt = cfg->record_tokens;
    std::vector<int64_t> pos(prefill, prefill + S);
    // queries of each step bucketed by owner thread (outside the timed phases)
    std::vector<std::vector<std::vector<int64_t>>> qb(cfg->steps, std::vector<std::vector<int64_t>>(T));
    for (int s = 0; s < cfg->steps; ++s)
      for (int i = 0; i < cfg->queries_per_step; ++i) {
        const int64_t k = static_cast<int64_t>(s) * cfg->queries_per_step + i;
        qb[s][owner[q_stream[k] / G]].push_back(k);
      }
    std::barrier sync(T + 1);
    std::atomic<int64_t> appended{0};
    std::atomic<int64_t> sink{0};
    auto worker = [&](int t) {
      // prefill: records of rt tokens, round-robin over the thread's streams
      sync.arrive_and_wait();
      for (int g : mine[t]) {
        for (int r = 0; r < G; ++r) {
          const int st = g * G + r;
          for (int64_t p = 0; p < prefill[st]; p += rt) {
            const int64_t n = std::min<int64_t>(rt, prefill[st] - p);
            idx[g]->append(r, static_cast<uint64_t>(p), std::span<const Token>(tokens + offsets[st] + p, n));
          }
        }
      }
      sync.arrive_and_wait();
      for (int s = 0; s < cfg->steps; ++s) {
        sync.arrive_and_wait();  // append phase
        int64_t app = 0;
        for (int g : mine[t])
          for (int r = 0; r < G; ++r) {
            const int st = g * G + r;
            const int64_t len = offsets[st + 1] - offsets[st];
            const int64_t p = pos[st];
            const int64_t n = std::min<int64_t>(rt, len - p);
            if (n <= 0) continue;
            idx[g]->append(r, static_cast<uint64_t>(p), std::span<const Token>(tokens + offsets[st] + p, n));
            pos[st] = p + n;
            app += n;
          }
        appended += app;
        sync.arrive_and_wait();
        sync.arrive_and_wait();  // query phase
        int64_t acc_sum = 0;
        for (int64_t k : qb[s][t]) {
          const int st = q_stream[k];
          const int64_t p = q_pos[k];
          const int64_t plen = std::min<int64_t>(a.pattern_lookup_max, p);
          auto c = idx[st / G]->speculate(std::span<const Token>(tokens + offsets[st] + p - plen, plen), a);
          const int64_t len = offsets[st + 1] - offsets[st];
          const int truth_left = static_cast<int>(len - p);
          int acc = 0;
          for (const auto& d : c) {
            int m = 0;
            const int cap = std::min<int>(static_cast<int>(d.tokens.size()), truth_left);
            while (m < cap && d.tokens[m] == tokens[offsets[st] + p + m]) ++m;
            acc = std::max(acc, m);
          }
          acc_sum += std::min(acc + 1, truth_left);
        }
        sink += acc_sum;
        sync.arrive_and_wait();
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(worker, t);
    using clk = std::chrono::steady_clock;
    auto secs = [](clk::time_point a0, clk::time_point b0) { return std::chrono::duration<double>(b0 - a0).count(); };
    sync.arrive_and_wait();
    auto t0 = clk::now();
    sync.arrive_and_wait();
    out[0] = secs(t0, clk::now());
    int64_t pre = 0;
    for (int st = 0; st < S; ++st) pre += prefill[st];
    out[1] = static_cast<double>(pre);
    for (int s = 0; s < cfg->steps; ++s) {
      appended = 0;
      auto a0 = clk::now();
      sync.arrive_and_wait();
      sync.arrive_and_wait();
      auto a1 = clk::now();
      sync.arrive_and_wait();
      sync.arrive_and_wait();
      auto a2 = clk::now();
      out[2 + 4 * s] = secs(a0, a1);
      out[3 + 4 * s] = static_cast<double>(appended.load());
      out[4 + 4 * s] = secs(a1, a2);
      out[5 + 4 * s] = static_cast<double>(cfg->queries_per_step);
    }
    for (auto& x : th) x.join();
    return sink.load() >= 0 ? 0 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C" (bench)

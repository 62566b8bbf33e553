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

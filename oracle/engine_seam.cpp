// engine_seam.cpp — the reference engine driving the B200 draft server through its own seam.
//
// TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/engine_seam from the
// unmodified reference sources plus this file, linked against paper_2511_14617_b200/libdgds_b200.so).
//
// The reference's Instance::decode_step (proj/src/engine.cpp:69-167) asks a SpeculationSource
// (engine.hpp:67-74) for drafts and reports emitted tokens back. The reference ships no
// implementation of that seam; DgdsSource below is the one INTEGRATION.md §3 describes: a
// rollsim::SpeculationSource over dgds_b200::GpuSpeculationSource, i.e. a dgds_b200::DraftClient
// (note_tokens batching, fetch_period 0) over a dgds_b200::LocalTransport to the GPU
// dgds_b200::DraftServer. The same staggered replay is run twice — once with the reference's own
// DraftClient / LocalTransport / DraftServer behind the seam, once with DgdsSource — and every
// StepReport (batch, drafted, accepted, emitted, per-request slot/drafted/accepted/emitted,
// step duration) must be identical.
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgds_b200.hpp"
#include "rollsim/dgds.hpp"
#include "rollsim/engine.hpp"
#include "rollsim/kvpool.hpp"
#include "rollsim/workload.hpp"

using namespace rollsim;

namespace {

class RefSource final : public SpeculationSource {  // the reference's own stack behind the seam
 public:
  explicit RefSource(DraftClient& c) : client_(c) {}
  std::vector<std::vector<DraftCandidate>> batch(std::span<const SpecQuery> q, SimTime now) override {
    return client_.batch_speculate(q, now);
  }
  void on_emitted(const std::string& gid, int rid, std::span<const Token> toks, SimTime now) override {
    client_.note_tokens(gid, rid, toks, now);
  }

 private:
  DraftClient& client_;
};

// the adapter a maintainer adds to the reference engine.
class DgdsSource final : public SpeculationSource {
 public:
  explicit DgdsSource(dgds_b200::GpuSpeculationSource& src) : src_(src) {}
  std::vector<std::vector<DraftCandidate>> batch(std::span<const SpecQuery> queries, SimTime now) override {
    std::vector<dgds_b200::SpecQuery> q(queries.size());
    for (std::size_t i = 0; i < queries.size(); ++i) {
      const auto& a = queries[i].args;
      q[i].group_id = queries[i].group_id;
      q[i].pattern.assign(queries[i].pattern.begin(), queries[i].pattern.end());
      q[i].args = dgds_b200::SpeculationArgs{a.max_spec_tokens, a.pattern_lookup_max, a.pattern_lookup_min,
                                             a.top_k, a.min_step_freq, a.min_support};
    }
    auto got = src_.batch(q, now);
    std::vector<std::vector<DraftCandidate>> out(got.size());
    for (std::size_t i = 0; i < got.size(); ++i)
      for (auto& c : got[i]) {
        DraftCandidate d;
        d.tokens.assign(c.tokens.begin(), c.tokens.end());
        d.score = c.score;
        d.support = c.support;
        out[i].push_back(std::move(d));
      }
    return out;
  }
  void on_emitted(const std::string& gid, int rid, std::span<const Token> toks, SimTime now) override {
    src_.on_emitted(gid, rid, std::span<const dgds_b200::Token>(toks.data(), toks.size()), now);
  }

 private:
  dgds_b200::GpuSpeculationSource& src_;
};

// A transport that is not a LocalTransport: the client then keeps GPU replicas and syncs them
// with GDX1 blobs before every batch (fresh mode), as it would over the wire protocol.
class ForwardingTransport final : public dgds_b200::DraftTransport {
 public:
  explicit ForwardingTransport(dgds_b200::DraftTransport& t) : t_(t) {}
  dgds_b200::UpdateReply update_cst(const std::string& g, int r, std::uint64_t p, std::span<const dgds_b200::Token> x,
                                    SimTime now) override {
    return t_.update_cst(g, r, p, x, now);
  }
  std::vector<dgds_b200::FetchReply> fetch_cst(std::span<const std::string> ids,
                                               std::span<const dgds_b200::DraftCacheInfo> infos,
                                               SimTime now) override {
    return t_.fetch_cst(ids, infos, now);
  }
  void register_group(const std::string& g, double ttl, SimTime now) override { t_.register_group(g, ttl, now); }

 private:
  dgds_b200::DraftTransport& t_;
};

struct Run {
  std::vector<StepReport> steps;
};

Run replay(const std::vector<PromptGroup>& groups, SpeculationSource& src, const SpecConfig& spec, int stagger) {
  KvParams kp;
  kp.instance_capacity_tokens = 1ull << 50;
  kp.dram_capacity_tokens = 1ull << 50;
  kp.ssd_capacity_tokens = 1ull << 50;
  KvPool pool(kp, 1);
  StepTimeModel sm;
  sm.batch_cap = 1 << 30;
  Instance inst(0, sm, 1ull << 50, pool, /*divided=*/false);
  std::vector<std::unique_ptr<SimRequest>> reqs;
  int max_g = 0;
  for (const auto& g : groups) max_g = std::max<int>(max_g, static_cast<int>(g.outputs.size()));
  for (std::size_t gi = 0; gi < groups.size(); ++gi)
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
  Run run;
  SimTime now = 0.0;
  std::size_t finished = 0;
  for (long long step = 0; finished < reqs.size() && step < 100000; ++step) {
    for (auto& r : reqs)
      if (r->meta.state == RequestState::Pending && static_cast<long long>(r->meta.request_index) * stagger == step) {
        double delay = 0;
        if (inst.admit(*r, static_cast<int>(r->truth->size()), now, &delay) != Instance::AdmitOutcome::Accept)
          throw std::runtime_error("admit refused");
        inst.make_ready(*r);
      }
    if (inst.running().empty()) continue;
    StepReport rep = inst.decode_step(&src, spec, now);
    now += rep.duration;
    run.steps.push_back(rep);
    std::vector<SimRequest*> running(inst.running().begin(), inst.running().end());
    for (SimRequest* r : running)
      if (r->remaining_truth() == 0 || r->remaining_chunk() == 0) {
        inst.finish_or_requeue(*r, now);
        if (r->meta.state == RequestState::Finished) ++finished;
      }
  }
  return run;
}

}  // namespace

int main(int argc, char** argv) {
  const int k = argc > 1 ? std::atoi(argv[1]) : 1;                          // multi_path_k
  const bool via_replicas = argc > 2 && std::string(argv[2]) == "replicas";  // blob-synced GPU replicas
  WorkloadConfig w;
  w.num_groups = 6;
  w.group_size = 4;
  w.length_model.location = 600.0;
  w.length_model.scale = 0.3;
  w.pattern_similarity = 0.8;
  w.vocab_size = 300;
  w.max_tokens = 1200;
  w.seed = 17;
  const auto groups = generate_workload(w);
  SpecConfig spec;
  spec.sd_enabled = true;
  spec.adaptive.enabled = true;
  spec.adaptive.batch_token_budget = 48;
  spec.adaptive.per_request_cap = 8;
  spec.adaptive.multi_path_k = k;
  const int stagger = 64;

  DgdsParams dp;
  dp.fetch_period = 0.0;
  DraftServer ref_server(dp);
  LocalTransport ref_lt(ref_server);
  DraftClient ref_client(ref_lt, dp);
  RefSource ref_src(ref_client);
  const Run a = replay(groups, ref_src, spec, stagger);

  dgds_b200::DgdsParams gp;
  gp.fetch_period = 0.0;
  dgds_b200::DraftServer gpu_server(gp);
  dgds_b200::LocalTransport gpu_lt(gpu_server);
  ForwardingTransport fwd(gpu_lt);
  dgds_b200::DraftClient gpu_client(via_replicas ? static_cast<dgds_b200::DraftTransport&>(fwd)
                                                 : static_cast<dgds_b200::DraftTransport&>(gpu_lt),
                                    gp);
  dgds_b200::GpuSpeculationSource gpu_src(gpu_client);
  DgdsSource seam(gpu_src);
  const Run b = replay(groups, seam, spec, stagger);

  if (a.steps.size() != b.steps.size()) {
    std::fprintf(stderr, "step count differs: %zu vs %zu\n", a.steps.size(), b.steps.size());
    return 1;
  }
  long long drafted = 0, accepted = 0, records = 0;
  for (std::size_t i = 0; i < a.steps.size(); ++i) {
    const StepReport& x = a.steps[i];
    const StepReport& y = b.steps[i];
    bool same = x.batch == y.batch && x.drafted == y.drafted && x.accepted == y.accepted && x.emitted == y.emitted &&
                x.duration == y.duration && x.per_request.size() == y.per_request.size();
    for (std::size_t j = 0; same && j < x.per_request.size(); ++j) {
      const auto& p = x.per_request[j];
      const auto& q = y.per_request[j];
      same = p.slot == q.slot && p.drafted == q.drafted && p.accepted == q.accepted && p.emitted == q.emitted;
    }
    if (!same) {
      std::fprintf(stderr, "step %zu differs: drafted %lld/%lld accepted %lld/%lld emitted %lld/%lld\n", i,
                   x.drafted, y.drafted, x.accepted, y.accepted, x.emitted, y.emitted);
      return 1;
    }
    drafted += x.drafted;
    accepted += x.accepted;
    records += static_cast<long long>(x.per_request.size());
  }
  if (drafted == 0 || accepted == 0) {
    std::fprintf(stderr, "degenerate replay: nothing drafted or accepted\n");
    return 1;
  }
  std::printf("engine seam ok: %zu steps, %lld request-steps, drafted %lld, accepted %lld (k=%d, %s)\n",
              a.steps.size(), records, drafted, accepted, k, via_replicas ? "GPU replicas" : "server");
  return 0;
}

// facade_test.cpp — the C++ facade (include/dgds_b200.hpp) used the way a C++
// rollout engine would use rollsim::DraftServer; answers pinned to SPEC.md.
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgds_b200.hpp"

using namespace dgds_b200;

#define EXPECT(c)                                                          \
  do {                                                                     \
    if (!(c)) {                                                            \
      std::fprintf(stderr, "FAILED %s at line %d\n", #c, __LINE__);        \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main() {
  DraftServer server(DgdsParams{});
  // [1,2,3,4,5], pattern [2,3], k=1 -> [[4,5]] score 1.0
  TokenSeq s1{1, 2, 3, 4, 5};
  UpdateReply r = server.update_cst("g1", 1, 0, s1, 0.0);
  EXPECT(r.ok && r.version == 1 && r.acked_tokens == 5);
  auto c = server.speculate("g1", TokenSeq{2, 3}, SpeculationArgs{8, 6, 1, 1});
  EXPECT(c.size() == 1 && c[0].tokens == (TokenSeq{4, 5}) && c[0].score == 1.0 && c[0].support == 1);
  // [1,2,3] + [1,2,4], pattern [1,2], k=2 -> [3], [4] each 0.5
  server.update_cst("g2", 1, 0, TokenSeq{1, 2, 3}, 0.0);
  server.update_cst("g2", 2, 0, TokenSeq{1, 2, 4}, 0.0);
  c = server.speculate("g2", TokenSeq{1, 2}, SpeculationArgs{8, 6, 1, 2});
  EXPECT(c.size() == 2 && c[0].tokens == TokenSeq{3} && c[1].tokens == TokenSeq{4} && c[0].score == 0.5);
  // gap -> out-of-order value with the acknowledged count
  r = server.update_cst("g1", 1, 9, TokenSeq{7}, 0.0);
  EXPECT(!r.ok && r.acked_tokens == 5 && r.version == 1);
  // invalid args throw std::invalid_argument, as the reference does
  bool threw = false;
  try {
    server.speculate("g1", TokenSeq{1}, SpeculationArgs{8, 6, 0, 1});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  // engine seam: SpeculationSource over an always-fresh DraftClient (16-token flush)
  DgdsParams p;
  p.fetch_period = 0.0;
  DraftClient client(server, p);
  GpuSpeculationSource src(client);
  TokenSeq emitted;
  for (int i = 0; i < 20; ++i) emitted.push_back(100 + i % 5);
  src.on_emitted("g3", 0, std::span<const Token>(emitted.data(), 20), 0.0);  // >= 16 pending -> flushed
  EXPECT(server.stored_tokens("g3", 0) == 20);
  std::vector<SpecQuery> qs{{"g3", TokenSeq{100, 101}, SpeculationArgs{4, 6, 1, 1}}, {"nope", TokenSeq{1}, {}}};
  auto res = src.batch(qs, 0.0);
  EXPECT(res.size() == 2 && res[1].empty() && res[0].size() == 1 && res[0][0].tokens == (TokenSeq{102, 103, 104, 100}));
  EXPECT(shard_of_group("g00000", 8) == shard_of_group("g00000", 8));

  // replica sync: fetch_cst blobs restore a replica server; periodic client mode
  std::vector<std::string> ids{"g1"};
  std::vector<DraftCacheInfo> infos{{"g1", 0}};
  auto f = server.fetch_cst(ids, infos, 0.0);
  EXPECT(f.size() == 1 && f[0].kind == FetchKind::Full && f[0].version == 1 && f[0].blob.size() > 4);
  DraftServer replica(DgdsParams{});
  EXPECT(replica.apply_blob("g1", f[0].blob) == 1);
  EXPECT(replica.speculate("g1", TokenSeq{2, 3}, SpeculationArgs{8, 6, 1, 1})[0].tokens == (TokenSeq{4, 5}));
  infos[0].cached_version = 1;
  EXPECT(server.fetch_cst(ids, infos, 0.0)[0].kind == FetchKind::UpToDate);

  DgdsParams pp;  // fetch_period 0.2 (reference default): answers from GPU replicas, stale between fetches
  DraftClient periodic(server, pp);
  periodic.set_active_groups({"g3", "g2"});
  EXPECT(periodic.fetch_due(0.0));
  EXPECT(periodic.batch_speculate(qs, 0.0)[0].empty());  // no replica yet
  periodic.fetch_active(0.0);
  EXPECT(!periodic.fetch_due(0.1) && periodic.fetch_due(0.25));
  EXPECT(periodic.cached_version("g3") == server.group_version("g3"));
  auto pr = periodic.batch_speculate(qs, 0.1);
  EXPECT(pr[0].size() == 1 && pr[0][0].tokens == (TokenSeq{102, 103, 104, 100}) && pr[1].empty());
  TokenSeq more{100, 101, 7, 7, 7, 7, 7, 7, 7, 7, 7, 7, 7, 7, 7, 7};
  server.update_cst("g3", 1, 0, more, 0.2);  // the server moves on; the replica is stale until fetched
  auto stale = periodic.batch_speculate(qs, 0.2);
  EXPECT(stale[0].size() == pr[0].size() && stale[0][0].tokens == pr[0][0].tokens &&
         stale[0][0].score == pr[0][0].score);
  periodic.fetch_active(0.3);  // delta
  auto fresh = periodic.batch_speculate(qs, 0.3);
  auto direct = server.speculate("g3", TokenSeq{100, 101}, SpeculationArgs{4, 6, 1, 1});
  EXPECT(fresh[0].size() == direct.size() && fresh[0][0].tokens == direct[0].tokens &&
         fresh[0][0].score == direct[0].score);
  EXPECT(periodic.cached_version("g3") == server.group_version("g3"));
  // asynchronous batches see exactly the updates made before their submit
  DraftServer as;
  as.update_cst("ga", 0, 0, TokenSeq{1, 2, 3, 4, 5}, 0.0);
  std::vector<SpecQuery> aq{{"ga", TokenSeq{1, 2}, SpeculationArgs{4, 6, 1, 2}}};
  auto b1 = as.speculate_submit(aq);
  as.update_cst("ga", 1, 0, TokenSeq{1, 2, 9}, 0.0);
  auto b2 = as.speculate_submit(aq);
  auto r2 = as.speculate_wait(b2);
  auto r1 = as.speculate_wait(b1);
  EXPECT(r1[0].size() == 1 && r1[0][0].tokens == (TokenSeq{3, 4, 5}) && r1[0][0].score == 1.0);
  auto now = as.batch_speculate(aq);
  EXPECT(r2[0].size() == 2 && now[0].size() == 2);
  for (int j = 0; j < 2; ++j)
    EXPECT(r2[0][j].tokens == now[0][j].tokens && r2[0][j].score == now[0][j].score &&
           r2[0][j].support == now[0][j].support);
  // the cluster form (shards as GPUs; here three shards on device 0) answers like one server
  ClusterServer cl(DgdsParams{}, std::vector<int>{0, 0, 0});
  DraftServer one;
  for (int g = 0; g < 6; ++g) {
    const std::string gid = "k" + std::to_string(g);
    for (int r = 0; r < 3; ++r) {
      TokenSeq t{1, 2, 3 + (r + g) % 3, 4, 5 + r};
      EXPECT(cl.update_cst(gid, r, 0, t, 0.0).version == one.update_cst(gid, r, 0, t, 0.0).version);
    }
    EXPECT(cl.owner_gpu(gid) == shard_of_group(gid, 3));
  }
  std::vector<SpecQuery> cq;
  for (int g = 0; g < 6; ++g) cq.push_back({"k" + std::to_string(g), TokenSeq{1, 2}, SpeculationArgs{4, 6, 1, 3}});
  auto x = cl.batch_speculate(cq);
  auto y = one.batch_speculate(cq);
  for (std::size_t i = 0; i < cq.size(); ++i) {
    EXPECT(x[i].size() == y[i].size());
    for (std::size_t j = 0; j < x[i].size(); ++j)
      EXPECT(x[i][j].tokens == y[i][j].tokens && x[i][j].score == y[i][j].score && x[i][j].support == y[i][j].support);
  }
  EXPECT(cl.node_count() == one.node_count());
  // DraftClient over a transport that is not local: GPU replicas synced by blobs
  struct Fwd final : DraftTransport {
    LocalTransport& t;
    explicit Fwd(LocalTransport& x) : t(x) {}
    UpdateReply update_cst(const std::string& g, int r, std::uint64_t p, std::span<const Token> v, SimTime n) override {
      return t.update_cst(g, r, p, v, n);
    }
    std::vector<FetchReply> fetch_cst(std::span<const std::string> ids, std::span<const DraftCacheInfo> in,
                                      SimTime n) override {
      return t.fetch_cst(ids, in, n);
    }
    void register_group(const std::string& g, double ttl, SimTime n) override { t.register_group(g, ttl, n); }
  };
  LocalTransport lt(one);
  Fwd fwd(lt);
  DgdsParams fresh_p;
  fresh_p.fetch_period = 0.0;
  DraftClient rc(fwd, fresh_p);
  auto z = rc.batch_speculate(cq, 1.0);
  for (std::size_t i = 0; i < cq.size(); ++i) {
    EXPECT(z[i].size() == y[i].size());
    for (std::size_t j = 0; j < z[i].size(); ++j) EXPECT(z[i][j].tokens == y[i][j].tokens && z[i][j].score == y[i][j].score);
  }
  std::printf("facade ok\n");
  return 0;
}

// facade_test.cpp — the C++ facade (include/dgds_b200.hpp) used the way a C++
// rollout engine would use rollsim::DraftServer; answers pinned to SPEC.md.
#include <cstdio>
#include <stdexcept>
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
  // engine seam: SpeculationSource over a DraftClient (16-token flush)
  DgdsParams p;
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
  std::printf("facade ok\n");
  return 0;
}

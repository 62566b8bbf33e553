// workload_gen.cpp — synthetic grouped-rollout traces for the benchmark and the tests (a tools
// library, not part of the draft server: tools/workload/libdgds_workload.so).
//
// Restates generate_workload (proj/src/workload.cpp:51-103) and the
// self-contained splitmix64 Rng it draws from (proj/include/rollsim/detail/
// rng.hpp:8-65) so bench.py can build the reference's exact inputs on the GPU
// box, where the reference does not exist. Bit-identical output is checked by
// tests/test_workload.py against the compiled reference (golden fingerprints).
// Same libm calls in the same order as the reference, so traces match on the
// same platform.

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "workload_gen.h"

namespace {

uint64_t mix64(uint64_t x) {  // splitmix64 finaliser (rng.hpp:8-13)
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t substream(uint64_t seed, uint64_t stream) {  // mix_seed (rng.hpp:18-20)
  return mix64(seed ^ (0x9E3779B97F4A7C15ull * (stream + 1)));
}

class Draws {  // Rng (rng.hpp:25-65)
 public:
  explicit Draws(uint64_t s) : state_(s) {}
  uint64_t u64() {
    state_ += 0x9E3779B97F4A7C15ull;
    uint64_t x = state_;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return static_cast<uint64_t>((static_cast<unsigned __int128>(u64()) * n) >> 64); }
  double gauss(double mean, double sigma) {  // Box-Muller, no cached spare
    if (sigma == 0.0) return mean;
    const double u1 = (static_cast<double>(u64() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = unit();
    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
    return mean + sigma * z;
  }
  double lognormal(double mu, double sigma) { return std::exp(gauss(mu, sigma)); }
  double pareto(double xm, double alpha) {
    const double u = 1.0 - unit();
    return xm / std::pow(u, 1.0 / alpha);
  }

 private:
  uint64_t state_;
};

int round_clamp(double v, int hi) {  // clamp_len (workload.cpp:41-47)
  if (!(v > 0.5)) return 1;
  const double r = std::floor(v + 0.5);
  if (r < 1.0) return 1;
  if (r > static_cast<double>(hi)) return hi;
  return static_cast<int>(r);
}

bool valid(const dgds_workload_cfg& c) {  // validate_config (workload.cpp:21-39)
  if (c.num_groups < 1 || c.group_size < 1 || c.vocab_size < 2 || c.max_tokens < 1) return false;
  if (!(c.location > 0.0) || !(c.scale >= 0.0)) return false;
  if (c.length_family == 1 && !(c.scale > 0.0)) return false;
  if (!(c.group_correlation >= 0.0 && c.group_correlation <= 1.0)) return false;
  if (!(c.noise_base >= 0.0)) return false;
  if (!(c.pattern_similarity >= 0.0 && c.pattern_similarity <= 1.0)) return false;
  if (!(c.prompt_mean >= 1.0) || !(c.prompt_spread >= 0.0)) return false;
  return true;
}

}  // namespace

extern "C" int dgds_generate_workload(const dgds_workload_cfg* cfg, int64_t* lengths, int32_t* prompt_lens,
                                      int32_t* tokens) {
  if (!cfg || !lengths || !valid(*cfg)) return -1;
  const dgds_workload_cfg& c = *cfg;
  int64_t out_off = 0;
  std::vector<int> len(c.group_size);
  std::vector<int32_t> tmpl;
  for (int g = 0; g < c.num_groups; ++g) {
    Draws rng(substream(c.seed, static_cast<uint64_t>(g)));
    const int plen = round_clamp(rng.gauss(c.prompt_mean, c.prompt_spread), std::numeric_limits<int>::max());
    if (prompt_lens) prompt_lens[g] = plen;
    double target = c.length_family == 0 ? rng.lognormal(std::log(c.location), c.scale)
                                         : rng.pareto(c.location, c.scale);
    if (target > static_cast<double>(c.max_tokens)) target = c.max_tokens;
    const double spread = (1.0 - c.group_correlation) * c.noise_base;
    int longest = 1;
    for (int i = 0; i < c.group_size; ++i) {
      const double eps = rng.gauss(0.0, spread);
      len[i] = round_clamp(target * (1.0 + eps), c.max_tokens);
      if (len[i] > longest) longest = len[i];
    }
    tmpl.resize(longest);
    for (int j = 0; j < longest; ++j) tmpl[j] = static_cast<int32_t>(rng.below(static_cast<uint64_t>(c.vocab_size)));
    for (int i = 0; i < c.group_size; ++i) {
      lengths[static_cast<int64_t>(g) * c.group_size + i] = len[i];
      if (!tokens) continue;  // lengths are drawn before any token of the group
      int32_t* out = tokens + out_off;
      for (int j = 0; j < len[i]; ++j)
        out[j] = (rng.unit() < c.pattern_similarity)
                     ? tmpl[j]
                     : static_cast<int32_t>(rng.below(static_cast<uint64_t>(c.vocab_size)));
      out_off += len[i];
    }
  }
  return 0;
}

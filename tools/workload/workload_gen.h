/* workload_gen.h — synthetic grouped-rollout traces for the benchmark and the tests (not part of the
 * draft-server library: built into tools/workload/libdgds_workload.so by paper_2511_14617_b200/build.py). */
#ifndef DGDS_WORKLOAD_GEN_H
#define DGDS_WORKLOAD_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synthetic grouped-rollout traces (generate_workload, workload.cpp:51-103) ---- */
typedef struct dgds_workload_cfg {
  int32_t num_groups;
  int32_t group_size;
  int32_t length_family; /* 0 lognormal, 1 pareto (workload.hpp:19-25) */
  int32_t vocab_size;
  double location;
  double scale;
  double group_correlation;
  double noise_base;
  double pattern_similarity;
  double prompt_mean;
  double prompt_spread;
  int32_t max_tokens;
  int32_t reserved0;
  uint64_t seed;
} dgds_workload_cfg;

/* Pass 1 (tokens == NULL): fills lengths[num_groups*group_size] and prompt_lens[num_groups] (may be NULL).
 * Pass 2: also writes all outputs back to back (group-major, request-minor) into tokens. */
/* returns 0, or -1 on an invalid configuration */
int dgds_generate_workload(const dgds_workload_cfg* cfg, int64_t* lengths, int32_t* prompt_lens, int32_t* tokens);

#ifdef __cplusplus
}
#endif

#endif

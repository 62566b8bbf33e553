/* oracle_capi.h — C ABI shared by the two CPU checkers under oracle/.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py. Never linked into the
 * product library (paper_2511_14617_b200/).
 *
 *   liboracle.so         our restatement (cst_oracle.cpp)
 *   _ref/libdgds_ref.so  the reference sources compiled in place (ref_capi.cpp)
 *
 * Both export the orc_index_* / orc_oracle_* subset with identical meaning so
 * the parity tests can run the same case through either; the reference build
 * additionally exports the server / workload / engine-replay / bench entry
 * points (orc_ref_*).
 */
#ifndef ORACLE_CAPI_H
#define ORACLE_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors rollsim::SpeculationArgs (proj/include/rollsim/cst.hpp:16-23). */
typedef struct orc_args {
  int32_t max_spec_tokens;
  int32_t pattern_lookup_max;
  int32_t pattern_lookup_min;
  int32_t top_k;
  double min_step_freq;
  int64_t min_support;
} orc_args;

/* Caller-owned candidate buffers: tokens[k_cap * s_cap], lens/scores/supports[k_cap]. */
typedef struct orc_cands {
  int32_t* tokens;
  int32_t* lens;
  double* scores;
  int64_t* supports;
  int32_t k_cap;
  int32_t s_cap;
  int32_t n; /* out: candidates written */
} orc_cands;

/* Work counters of one sequential speculate (SURVEY.md §8(d) B_q terms). */
typedef struct orc_qstats {
  int64_t suffix_lookups; /* F: child_of calls in the longest-suffix loop (cst.cpp:160-178) */
  int64_t expansions;     /* beam paths expanded (cst.cpp:196-215, outer loop body) */
  int64_t children;       /* Σ child-list entries visited over all expansions */
  int64_t child_sectors;  /* Σ ceil(8 * c / 32) over expansions */
  int64_t cand_tokens;    /* Σ |tokens| over returned candidates */
  int64_t cands;          /* returned candidates */
} orc_qstats;

const char* orc_last_error(void);

/* ---- GroupDraftIndex (cst.hpp:42-138) ---- */
void* orc_index_new(const char* group_id, int32_t max_pattern_len, int32_t max_spec_len);
void orc_index_free(void* idx);
/* returns 0, or -1 when the reference throws (message in orc_last_error) */
int orc_index_append(void* idx, int32_t request_id, uint64_t prev_token_count, const int32_t* toks,
                     uint64_t n, int32_t* ok, uint64_t* version, uint64_t* acked);
int orc_index_speculate(const void* idx, const int32_t* pattern, uint64_t plen, const orc_args* args,
                        orc_cands* out);
uint64_t orc_index_version(const void* idx);
uint64_t orc_index_node_count(const void* idx);
uint64_t orc_index_stored_tokens(const void* idx, int32_t request_id);

/* ---- speculate_oracle (cst.cpp:386-453): brute force over explicit sequences ---- */
int orc_oracle_speculate(const int32_t* toks, const uint64_t* offsets, uint64_t nseq,
                         const int32_t* pattern, uint64_t plen, const orc_args* args, orc_cands* out);

/* ---- restatement-only: instrumented speculate (liboracle.so) ---- */
int orc_index_speculate_stats(const void* idx, const int32_t* pattern, uint64_t plen,
                              const orc_args* args, orc_cands* out, orc_qstats* stats);

/* ---- reference-only: many indexes driven in bulk, threads split by group (scale parity) ---- */
void* orc_ref_gset_new(int32_t ngroups, const char* const* gids, int32_t max_pattern_len, int32_t max_spec_len);
void orc_ref_gset_free(void* gset);
int orc_ref_gset_append(void* gset, int64_t n, const int32_t* group, const int32_t* rid, const uint64_t* prev,
                        const uint64_t* offs, const int32_t* tokens, int32_t threads, int32_t* ok,
                        uint64_t* version, uint64_t* acked);
/* candidates of query i at [i][k_cap][s_cap] (tokens) / [i][k_cap] (lens, scores, supports) */
int orc_ref_gset_speculate(void* gset, int64_t n, const int32_t* group, const uint64_t* pat_offs,
                           const int32_t* pats, const orc_args* args, int32_t threads, int32_t k_cap,
                           int32_t s_cap, int32_t* n_cands, int32_t* lens, double* scores, int64_t* supports,
                           int32_t* tokens);
uint64_t orc_ref_gset_node_count(const void* gset);

#ifdef __cplusplus
}
#endif

#endif

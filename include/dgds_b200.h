/* dgds_b200.h — C ABI of the B200-native Distributed Grouped Draft Server (DGDS).
 *
 * Drop-in boundary for the reference draft-server hot path
 * (/root/reference/proj/include/rollsim/dgds.hpp:51-162, cst.hpp:16-138,
 *  engine.hpp:28-92). Plain pointers and sizes only; no C++ or torch types.
 * Host buffers unless a function says "device". Every function returns an int
 * status (DGDS_OK or a negative code; message via dgds_last_error()) and never
 * throws across the boundary.
 *
 * Reference interface each entry point replaces:
 *   dgds_create / dgds_destroy      DraftServer::DraftServer(DgdsParams)       dgds.hpp:53, dgds.cpp:19-23
 *   dgds_shard_of_group             shard_of_group                             dgds.hpp:46, dgds.cpp:10-14
 *   dgds_intern                     (group-id string -> handle; the reference keys std::map by string)
 *   dgds_register_group             DraftServer::register_group                dgds.hpp:59, dgds.cpp:99-110
 *   dgds_drop_group                 DraftServer::drop_group                    dgds.hpp:60, dgds.cpp:112-116
 *   dgds_sweep_expired              DraftServer::sweep_expired                 dgds.hpp:61, dgds.cpp:118-128
 *   dgds_has_group / dgds_group_version / dgds_stored_tokens / dgds_shard_group_count
 *                                   DraftServer::has_group/group_version, GroupDraftIndex::stored_tokens,
 *                                   DraftServer::shard_group_count             dgds.hpp:69-72, cst.hpp:75
 *   dgds_update_batch               DraftServer::update_cst x n (call order)   dgds.hpp:55-56, dgds.cpp:36-51
 *                                    -> GroupDraftIndex::append                 cst.cpp:118-133
 *   dgds_speculate_batch            DraftServer::speculate x n /               dgds.hpp:64-65, dgds.cpp:130-138
 *                                   DraftClient::batch_speculate (fetch_period 0) dgds.cpp:274-292
 *                                    -> GroupDraftIndex::speculate              cst.cpp:153-228
 *   dgds_verify_batch               Instance::decode_step verification          engine.cpp:115-143
 *   dgds_draft_len                  Instance::decode_step draft-length policy   engine.cpp:78-85
 *   dgds_*_device                   zero-copy forms of the batch calls over device buffers and a
 *                                   cudaStream_t (PAPER.md:359 batch_speculate(..., void* pattern_buffer_ptr,
 *                                   void* output_buffer_ptr, ...); SPEC.md:263 leaves it to us).
 *
 * Semantics are the reference's, record by record, including: an out-of-order
 * append is a VALUE (ok=0, acked=stored count) and still creates the request's
 * stream; an empty append is ok without a version bump; update auto-registers an
 * unknown or expired group with the default TTL; speculate on an unknown group
 * yields zero candidates and does not check expiry. Deliberate divergence: a
 * batch is validated as a whole before anything is applied (negative request id
 * or token, bad args -> DGDS_EINVAL and no effect), where the reference throws
 * after partially applying (cst.cpp:120,126-128).
 */
#ifndef DGDS_B200_H
#define DGDS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGDS_OK 0
#define DGDS_EINVAL (-1)      /* std::invalid_argument in the reference */
#define DGDS_ECUDA (-2)       /* CUDA runtime error */
#define DGDS_ENOMEM (-3)      /* device or host allocation failed */
#define DGDS_EUNSUPPORTED (-4) /* outside this build's device limits (see DGDS_MAX_*) */
#define DGDS_EBUFFER (-5)     /* caller output buffer too small */
#define DGDS_ESTATE (-6)      /* bad handle / call order */
#define DGDS_EBLOB (-7)       /* malformed or inapplicable GDX1 blob (std::runtime_error in the reference) */

#define DGDS_MAX_DEPTH 32 /* max_pattern_len + max_spec_len (one warp lane per trie level) */
#define DGDS_MAX_TOP_K 32

typedef struct dgds_server dgds_server;

/* DgdsParams (dgds.hpp:18-24) + Limits (cst.hpp:44-47) + device capacity plan. */
typedef struct dgds_params {
  int32_t shard_count;         /* logical shards for shard_group_count(); >= 1 */
  int32_t append_batch_tokens; /* kept for the client facade (dgds.hpp:21) */
  double fetch_period;         /* kept for the client facade (dgds.hpp:20) */
  double default_ttl_seconds;  /* auto-registration TTL (dgds.hpp:22) */
  int32_t max_pattern_len;     /* Limits (cst.hpp:45) */
  int32_t max_spec_len;        /* Limits (cst.hpp:46) */
  int32_t device;              /* CUDA device ordinal */
  int32_t reserved0;
  uint64_t expected_nodes;     /* initial trie capacity in nodes (0 = 1<<20); grows by rebuild */
  uint64_t expected_streams;   /* initial request-stream capacity (0 = 4096) */
} dgds_params;

/* SpeculationArgs (cst.hpp:16-23); 32 bytes. */
typedef struct dgds_spec_args {
  int32_t max_spec_tokens;
  int32_t pattern_lookup_max;
  int32_t pattern_lookup_min;
  int32_t top_k;
  double min_step_freq;
  int64_t min_support;
} dgds_spec_args;

/* UpdateReply (dgds.hpp:39-43). */
typedef struct dgds_update_reply {
  int32_t ok;
  int32_t reserved0;
  uint64_t version;
  uint64_t acked_tokens;
} dgds_update_reply;

/* Caller-owned candidate buffers for n queries: query q, candidate c in
 * [0, n_cands[q]) has lens[q*k_stride+c] tokens at tokens[(q*k_stride+c)*s_stride ...],
 * score scores[q*k_stride+c] (IEEE double, bit-exact with DraftCandidate::score) and
 * support supports[q*k_stride+c]. Candidates are in candidate_before order
 * (cst.cpp:29-33). k_stride >= max top_k, s_stride >= max min(max_spec_tokens, max_spec_len). */
typedef struct dgds_candidates {
  int32_t k_stride;
  int32_t s_stride;
  int32_t* n_cands;
  int32_t* lens;
  double* scores;
  int64_t* supports;
  int32_t* tokens;
} dgds_candidates;

/* Verification outputs per request (StepReport::PerRequest, engine.hpp:85-90). */
typedef struct dgds_verify_out {
  int32_t* drafted;
  int32_t* accepted; /* emitted - 1 */
  int32_t* emitted;
} dgds_verify_out;

/* Device-side counters of one query launch, for SURVEY.md §8(d)'s algorithmic
 * bytes: B_q = 4|p| + 32 + 32F + sum_exp(32 + 32 ceil(8c/32)) + sum_cand(4|tokens| + 16). */
typedef struct dgds_query_stats {
  uint64_t queries;
  uint64_t pattern_tokens;
  uint64_t suffix_lookups; /* F */
  uint64_t expansions;
  uint64_t child_sectors;  /* sum ceil(8c/32) */
  uint64_t cands;
  uint64_t cand_tokens;
  uint64_t algorithmic_bytes;
} dgds_query_stats;

const char* dgds_last_error(void);
/* Index / query / compaction kernels this process has enqueued (append: k_stage + K1 + K1b;
 * query: K2a + K2b or K2; compaction; copy-out; verify) — bench.py's gpu_launches. */
uint64_t dgds_kernel_launches(void);
const char* dgds_version_string(void);

uint64_t dgds_fnv1a64(const void* data, size_t n); /* detail::fnv1a64 (bytes.hpp:89-96) */
int32_t dgds_shard_of_group(const char* group_id, size_t len, int32_t shard_count);

int dgds_create(const dgds_params* params, dgds_server** out);
int dgds_destroy(dgds_server* s);
/* The CUDA stream (cudaStream_t) the server orders its work on. */
void* dgds_cuda_stream(dgds_server* s);

/* Group-id string -> stable handle (interned; no registration side effect). */
int dgds_intern(dgds_server* s, const char* group_id, size_t len, int32_t* handle);

int dgds_register_group(dgds_server* s, int32_t handle, double ttl_seconds, double now);
int dgds_drop_group(dgds_server* s, int32_t handle);
int dgds_sweep_expired(dgds_server* s, double now);
int dgds_has_group(dgds_server* s, int32_t handle, int32_t* out);
int dgds_group_version(dgds_server* s, int32_t handle, uint64_t* out);
int dgds_stored_tokens(dgds_server* s, int32_t handle, int32_t request_id, uint64_t* out);
int dgds_shard_group_count(dgds_server* s, int32_t shard, uint64_t* out);
/* Device-side trie size: the reference's node count (nodes_.size(), root included) summed over
 * live groups; counts entries plus the implicit count-1 chains below leaves (synchronises). */
int dgds_node_count(dgds_server* s, uint64_t* out);
/* Table entries in use (materialised windows: nodes with count >= 2 and leaves). */
int dgds_entry_count(dgds_server* s, uint64_t* out);
/* Reads and clears the device error flags (synchronises): bit 0 a device-API query with invalid
 * arguments (it returned no candidates), bit 1 a negative token in a device-path update batch
 * (that batch and every later one inserted nothing; its replies were already returned), bits
 * 2-4 internal invariants (never expected). Returns DGDS_OK with *flags = 0 when clean. */
int dgds_device_error(dgds_server* s, int32_t* flags);
/* Slots of the open-addressing node table (load factor = stored nodes / slots). */
int dgds_index_slots(dgds_server* s, uint64_t* slots);

/* n update_cst calls, applied in array order. Record i appends
 * tokens[tok_offsets[i] .. tok_offsets[i+1]) for (handles[i], request_ids[i]).
 * Host buffers; returns after the replies are final (the device insertion is
 * enqueued on the server stream and ordered before any later query). */
int dgds_update_batch(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* request_ids,
                      const uint64_t* prev_counts, const uint64_t* tok_offsets, const int32_t* tokens, double now,
                      dgds_update_reply* replies);

/* Same, with the token payload already in device memory (d_tokens, record order);
 * metadata stays on the host. The kernel is enqueued on `stream` (NULL = the legacy default stream). */
int dgds_update_batch_device(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* request_ids,
                             const uint64_t* prev_counts, const uint64_t* tok_offsets, const int32_t* d_tokens,
                             double now, dgds_update_reply* replies, void* stream);

/* Same as dgds_update_batch_device with record i's tokens at d_tokens[tok_starts[i] .. + tok_counts[i])
 * (host arrays) — e.g. fixed-size routed records with the tokens inline. */
int dgds_update_batch_device_strided(dgds_server* s, int64_t n, const int32_t* handles, const int32_t* request_ids,
                                     const uint64_t* prev_counts, const uint64_t* tok_starts,
                                     const uint64_t* tok_counts, const int32_t* d_tokens, double now,
                                     dgds_update_reply* replies, void* stream);

/* n speculate calls. Query q uses patterns[pat_offsets[q] .. pat_offsets[q+1]) and
 * args[q * args_stride] (args_stride 0 = one shared args). Host buffers; blocks until done.
 */
int dgds_speculate_batch(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offsets,
                         const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                         dgds_candidates* out);

/* Zero-copy query over device buffers, enqueued on `stream` (NULL = the legacy default stream), no sync.
 * d_handles[n], d_pat_len[n], d_patterns[n * pat_stride] (the LAST d_pat_len[q] tokens of each
 * pattern, left-aligned; only the last max_pattern_len can matter), d_args[q * args_stride].
 * max_top_k bounds args.top_k and max_spec bounds min(args.max_spec_tokens, max_spec_len) over the
 * batch (they select the kernel instance; max_spec <= 0 means max_spec_len). A query outside the
 * bounds returns no candidates and raises the server's device error flag.
 * Optional fused verify: d_truth (n * truth_stride next ground-truth tokens), d_truth_left[n],
 * d_limit[n] -> d_vout (all device) — may be NULL. Optional d_stats accumulates counters. */
int dgds_speculate_device(dgds_server* s, int64_t n, const int32_t* d_handles, const int32_t* d_pat_len,
                          const int32_t* d_patterns, int32_t pat_stride, const dgds_spec_args* d_args,
                          int64_t args_stride, int32_t max_top_k, int32_t max_spec, const dgds_candidates* d_out,
                          const int32_t* d_truth, int32_t truth_stride, const int32_t* d_truth_left,
                          const int32_t* d_limit, const dgds_verify_out* d_vout, dgds_query_stats* d_stats,
                          void* stream);

/* The draft-budget policy of the engine (AdaptiveSpecPolicy + SpecConfig::sd_enabled,
 * engine.hpp:28-40). feedback 0 = the reference policy, d = min(cap, budget / n_running)
 * (engine.cpp:78-85), which has no acceptance feedback (the paper claims one);
 * feedback 1 = an acceptance-scaled extension: d_next = min(d_reference, ceil(mean accepted) + 1). */
typedef struct dgds_spec_policy {
  int32_t sd_enabled;
  int32_t adaptive;
  int32_t batch_token_budget;
  int32_t per_request_cap;
  int32_t multi_path_k;
  int32_t feedback;
} dgds_spec_policy;

/* Instance::decode_step's draft path for one step of n running requests, entirely on the device
 * (engine.cpp:69-143): per request, spec_len = min(d, limit - 1), pat_len = min(pattern_lookup_max,
 * generated), no query when spec_len <= 0 or pat_len < pattern_lookup_min; top_k =
 * max(1, multi_path_k); the draft query; verification against the next truth tokens
 * (d_vout: drafted / accepted / emitted). d is *d_draft_len (device scalar, e.g. the previous step's
 * d_next_draft_len) or, when that is NULL, draft_len. d_ctx rows (ctx_stride >= max_pattern_len)
 * hold each request's last min(generated, ctx_stride) tokens, left-aligned. The step's last warp
 * writes d_next_draft_len (the policy over the requests still running after this step, i.e.
 * limit - emitted > 0) and d_totals[4] = {still running, drafted, accepted, emitted} (both
 * optional, device memory). args: lookup bounds and cutoffs (max_spec_tokens / top_k are set per
 * request). Stream-ordered like dgds_speculate_device. */
int dgds_decode_step_device(dgds_server* s, int64_t n, const int32_t* d_handles, const int32_t* d_ctx,
                            int32_t ctx_stride, const int32_t* d_generated, const int32_t* d_limit,
                            const int32_t* d_truth, int32_t truth_stride, const int32_t* d_truth_left,
                            const dgds_spec_args* args, const dgds_spec_policy* policy,
                            const int32_t* d_draft_len, int32_t draft_len, const dgds_candidates* d_out,
                            const dgds_verify_out* d_vout, int32_t* d_next_draft_len, int64_t* d_totals,
                            void* stream);

/* dgds_speculate_batch + fused verification (engine.cpp:115-143) in one host call:
 * truth_next[q*truth_stride ..], truth_left[q], limit[q] -> vout (host buffers). */
int dgds_speculate_verify_batch(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offsets,
                                const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                                const int32_t* truth_next, int32_t truth_stride, const int32_t* truth_left,
                                const int32_t* limit, dgds_candidates* out, dgds_verify_out* vout);

/* Fixed-size query / reply records (e.g. traffic routed between GPUs). Offsets in 32-bit words.
 * Query record: group handle (-1 = empty slot: answered with nothing), pattern length, the last
 * <= rec_words - off_pattern pattern tokens, truth_left, limit, next truth tokens.
 * Reply record: n_cands, lens[k], scores[k] (f64), supports[k] (i64), tokens[k][max_spec],
 * drafted/accepted/emitted (off_verify < 0: no verification). 8-byte fields need even offsets and an
 * even reply width. */
typedef struct dgds_query_record_layout {
  int32_t rec_words;
  int32_t off_handle;
  int32_t off_pat_len;
  int32_t off_pattern;
  int32_t off_truth_left;
  int32_t off_limit;
  int32_t off_truth;
  int32_t reply_words;
  int32_t off_n_cands;
  int32_t off_lens;
  int32_t off_scores;
  int32_t off_supports;
  int32_t off_tokens;
  int32_t off_verify;
} dgds_query_record_layout;

/* K2 + fused K3 directly over device query records, writing device reply records (zero-copy,
 * enqueued on `stream`). max_spec also fixes the reply's per-candidate token stride. */
int dgds_speculate_records(dgds_server* s, int64_t n, const int32_t* d_records, const dgds_query_record_layout* layout,
                           const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k, int32_t max_spec,
                           int32_t* d_replies, dgds_query_stats* d_stats, void* stream);

/* Appends delivered by owner routing (dgds_px_send): n_seg sender segments of seg_rows rows;
 * segment g holds h_counts[g] valid rows. Row r = [handle, request_id, prev_lo, prev_hi, n,
 * tokens[n] ...] of row_words int32 — metadata read from host memory h_meta (row r at
 * h_meta + r * meta_stride), tokens from device memory d_rows. Same semantics as
 * dgds_update_batch_device_strided; *n_rejected = replies with ok == false. */
int dgds_update_batch_routed(dgds_server* s, int32_t n_seg, int64_t seg_rows, const int32_t* h_counts,
                             const int32_t* h_meta, int32_t meta_stride, const int32_t* d_rows, int32_t row_words,
                             double now, int64_t* n_rejected, void* stream);
/* Two-phase form of dgds_update_batch_routed: the plan call does all host work (validation,
 * replies, versions, history log, capacity) and returns a plan; dgds_update_launch later
 * enqueues the device part (H2D of the segment tables + the append kernel) on `stream` and
 * frees the plan. Lets a driver plan tick s+1 while the GPU runs tick s. Plans must be
 * launched in the order they were made (DGDS_ESTATE otherwise); d_rows must stay valid
 * until the launched kernel has run. */
typedef struct dgds_update_plan dgds_update_plan;
int dgds_update_plan_routed(dgds_server* s, int32_t n_seg, int64_t seg_rows, const int32_t* h_counts,
                            const int32_t* h_meta, int32_t meta_stride, const int32_t* d_rows, int32_t row_words,
                            double now, int64_t* n_rejected, dgds_update_plan** out);
int dgds_update_launch(dgds_server* s, dgds_update_plan* plan, void* stream);

/* Asynchronous dgds_update_plan_routed on a server-owned planner thread: the job waits for
 * `ready_event` (a cudaEvent_t recorded after the metadata rows reached h_meta / h_counts, or
 * NULL), then plans exactly like dgds_update_plan_routed. Jobs run in submission order, so
 * plans come out in the order dgds_update_launch needs. The host buffers must stay unchanged
 * until dgds_update_plan_take returns for the job; take blocks until the job is planned and
 * hands over its plan (and the number of rejected records). */
int dgds_update_plan_routed_async(dgds_server* s, void* ready_event, int32_t n_seg, int64_t seg_rows,
                                  const int32_t* h_counts, const int32_t* h_meta, int32_t meta_stride,
                                  const int32_t* d_rows, int32_t row_words, double now, uint64_t* job);
int dgds_update_plan_take(dgds_server* s, uint64_t job, int64_t* n_rejected, dgds_update_plan** out);
/* Strided device -> host copy (cudaMemcpy2DAsync): `rows` rows of `width` bytes. */
int dgds_copy_rows_d2h(void* h_dst, int64_t dst_pitch, const void* d_src, int64_t src_pitch, int64_t width,
                       int64_t rows, void* stream);

/* Zero-copy host results: compact per-query candidate lists (CSR) in a pinned block owned
 * by the server, valid until the second-next host query batch on `s` (two result slots). Candidates of query q are
 * cands[cand_off[q] .. cand_off[q+1]) in candidate_before order (cst.cpp:29-35); the tokens
 * of candidate c are tokens[tok_off[c] .. tok_off[c+1]). Verification (engine.cpp:115-143)
 * runs when truth != NULL. Same inputs and validation as dgds_speculate_verify_batch. */
typedef struct dgds_cand_meta {
  double score;
  int64_t support;
  int32_t len;
  int32_t reserved;
} dgds_cand_meta;
typedef struct dgds_result_view {
  int64_t n_queries, n_cands, n_tokens;
  const int64_t* cand_off;      /* [n_queries + 1] */
  const dgds_cand_meta* cands;  /* [n_cands] */
  const int64_t* tok_off;       /* [n_cands + 1] */
  const int32_t* tokens;        /* [n_tokens] */
  const int32_t* drafted;       /* [n_queries] each; NULL without verification */
  const int32_t* accepted;
  const int32_t* emitted;
} dgds_result_view;
int dgds_speculate_verify_view(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                               const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                               const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                               const int32_t* limit, dgds_result_view* out);

/* Asynchronous dgds_speculate_verify_view. submit checks the arguments, starts staging the batch
 * on the server's host workers and returns a ticket without waiting; the last worker queues the
 * H2D, and the query (+ verify) kernels and the
 * copy-out are launched before any later call on `s` touches the device. So the caller's next
 * host work — typically the next tick's dgds_update_batch planning — overlaps this batch's
 * staging, and its device work overlaps the next tick's host work. The batch sees exactly the
 * updates made before the submit (stream order). wait blocks for the batch and fills `out`.
 * The host input arrays are read asynchronously: keep them valid and unchanged until wait
 * returns for this ticket. Two batches can be in flight: submitting a batch reuses the result
 * slot of the batch submitted two before it, after which waiting on that ticket fails with
 * DGDS_EINVAL. A bad group handle or decreasing pattern offsets fail the whole batch (nothing
 * of it is launched): reported by submit for batches staged in the call (< 8192 queries),
 * else by wait. */
int dgds_speculate_submit(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* pat_offs,
                          const int32_t* patterns, const dgds_spec_args* args, int64_t args_stride,
                          const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                          const int32_t* limit, uint64_t* ticket);
int dgds_speculate_wait(dgds_server* s, uint64_t ticket, dgds_result_view* out);

/* Compact n reply records (dgds_query_record_layout; e.g. the routed replies a sender
 * gathers in peer memory) into the same CSR result view, in the server's next result slot:
 * compaction on `stream` after the records are complete, then a PCIe copy-out into mapped
 * pinned memory. Returns a ticket for dgds_speculate_wait; max_spec is the reply's token row
 * stride. The records may be overwritten once the work queued on `stream` here has run. */
int dgds_replies_submit(dgds_server* s, int64_t n, const int32_t* d_replies, const dgds_query_record_layout* lay,
                        int32_t max_top_k, int32_t max_spec, void* stream, uint64_t* ticket);

/* Segmented form for owner routing: rows arrive as n_seg sender segments of seg_rows rows
 * (row j of segment s valid while j < d_seg_count[s]); the reply of row j of segment s is
 * written to seg_out[s] + r * reply_words with r = j, or with origin_field >= 0 r = the
 * record's word origin_field (the query's index at its sender, stamped by dgds_px_send) —
 * so replies land in the sender's final order, typically straight into its region in NVLink
 * peer memory (dgds_px_region). seg_out is a host array of n_seg device pointers. */
int dgds_speculate_records_seg(dgds_server* s, int32_t n_seg, int64_t seg_rows, const int32_t* d_records,
                               const int32_t* d_seg_count, const dgds_query_record_layout* layout,
                               const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k,
                               int32_t max_spec, int32_t* const* seg_out, int32_t origin_field,
                               dgds_query_stats* d_stats, void* stream);

/* The paper's zero-copy batch_speculate (Table 4; the reference SPEC does not
 * keep it): an engine passes its own device buffers. Request i's pattern is the
 * last d_pat_len[i] tokens ending (exclusive) at d_pattern_buffer[d_pat_end[i]], read in
 * place; its reply record (layout reply fields: n_cands, lens[k], scores[k] f64,
 * supports[k] i64, tokens[k][max_spec]) is written at d_output_buffer + d_out_offsets[i]
 * (int32 units). No host copies; stream-ordered on `stream`. The engine verifies the drafts
 * with its target model, so the layout's verify field is ignored. */
int dgds_batch_speculate_zc(dgds_server* s, int64_t n, const int32_t* d_handles, const int64_t* d_pat_end,
                            const int32_t* d_pat_len, const int32_t* d_pattern_buffer, const int64_t* d_out_offsets,
                            int32_t* d_output_buffer, const dgds_query_record_layout* layout,
                            const dgds_spec_args* d_args, int64_t args_stride, int32_t max_top_k, int32_t max_spec,
                            dgds_query_stats* d_stats, void* stream);

/* Verification of existing candidates (engine.cpp:115-143), host buffers. */
int dgds_verify_batch(dgds_server* s, int64_t n, const dgds_candidates* cands, const int32_t* truth_next,
                      int32_t truth_stride, const int32_t* truth_left, const int32_t* limit,
                      dgds_verify_out* out);

/* Draft length policy (engine.cpp:78-85): sd disabled -> 0; adaptive -> min(cap, budget / n_running); max(.,0). */
int32_t dgds_draft_len(int32_t sd_enabled, int32_t adaptive, int32_t per_request_cap, int32_t batch_token_budget,
                       int32_t n_running);

/* ---- kernel timing (CUDA events around every append / query launch, on the launch stream) ---- */
typedef struct dgds_profile {
  uint64_t append_launches;
  uint64_t query_launches;
  double append_ms; /* summed device time of the append kernels */
  double query_ms;  /* summed device time of the query kernels */
} dgds_profile;
int dgds_profile_enable(dgds_server* s, int32_t on);
/* Debug: record per-query phase cycles of later device-API query launches into d_buf[n][8] (NULL = off). */
/* Debug (DGDS_APPEND_DBG set at create): per-warp [start, end] globaltimer ns of the last K1 launch. */
int dgds_debug_append_timing(dgds_server* s, uint64_t* out, int64_t n_warps);
/* Debug: copies device state into out (host), at most `bytes`: which 0 = slot table (32 B slots,
 * csrc/trie.cuh), 1 = stream table, 2 = active rows, 3 = ov rows, 4 = stream-history arena,
 * 5 = conversion-event queue. */
int dgds_debug_dump(dgds_server* s, int32_t which, void* out, uint64_t bytes);
int dgds_debug_query_timing(dgds_server* s, void* d_buf);
/* Device->host bytes moved by the last host-buffer query call (results are compacted on device). */
int dgds_last_transfer(dgds_server* s, uint64_t* d2h_bytes);
/* Synchronises on the recorded events; reset != 0 clears the accumulators. */
int dgds_profile_read(dgds_server* s, dgds_profile* out, int32_t reset);

/* ---- multi-GPU routing helpers (device, enqueued on `stream`) ----
 * Bucket n fixed-size records of rec_words 32-bit words by owner rank (owner[i] in [0, world)):
 * d_out receives the records grouped by owner in stable order, d_counts[world] the bucket sizes,
 * d_perm[i] the destination index of record i (for the inverse scatter of replies). */
int dgds_route_pack(int64_t n, int32_t world, const int32_t* d_owner, const uint32_t* d_records, int32_t rec_words,
                    uint32_t* d_out, int64_t* d_counts, int64_t* d_perm, void* stream);
/* Fixed-capacity variant: d_out holds world * cap records of rec_words words, bucket o at rows
 * [o*cap, (o+1)*cap) (empty rows are all -1); d_slot[i] = row of record i; *d_overflow set to 1
 * when a bucket would exceed cap. No host synchronisation: split sizes are static. */
int dgds_route_pack_padded(int64_t n, int32_t world, const int32_t* d_owner, const uint32_t* d_records,
                           int32_t rec_words, int64_t cap, uint32_t* d_out, int64_t* d_slot, int32_t* d_overflow,
                           void* stream);
/* Inverse: d_out[i] = d_in[d_perm[i]] for n records of rec_words words. */
int dgds_route_unpack(int64_t n, const uint32_t* d_in, int32_t rec_words, const int64_t* d_perm, uint32_t* d_out,
                      void* stream);

/* ---- N GPUs behind one server (DraftServer's shard routing, dgds.cpp:10-51) ----
 * One server per device; group g is owned by GPU fnv1a64(g) % n_gpus (shard_of_group). Batch
 * calls split records / queries by owner (stable: call order per group is kept), run the owners'
 * batches concurrently (one host thread per GPU) and return replies / results in call order, so
 * a cluster call equals the same call on one server holding every group. Handles are cluster
 * handles (dgds_cluster_intern). devices: n_gpus ordinals (NULL = 0..n_gpus-1; repeats allowed,
 * e.g. several shards on one GPU); params->device is ignored. */
typedef struct dgds_cluster dgds_cluster;
int dgds_cluster_create(const dgds_params* params, int32_t n_gpus, const int32_t* devices, dgds_cluster** out);
int dgds_cluster_destroy(dgds_cluster* c);
int32_t dgds_cluster_size(dgds_cluster* c);
dgds_server* dgds_cluster_server(dgds_cluster* c, int32_t gpu); /* member server (NULL if out of range) */
int dgds_cluster_intern(dgds_cluster* c, const char* group_id, size_t len, int32_t* handle);
int dgds_cluster_owner(dgds_cluster* c, int32_t handle, int32_t* gpu);
int dgds_cluster_register_group(dgds_cluster* c, int32_t handle, double ttl_seconds, double now);
int dgds_cluster_drop_group(dgds_cluster* c, int32_t handle);
int dgds_cluster_sweep_expired(dgds_cluster* c, double now);
int dgds_cluster_has_group(dgds_cluster* c, int32_t handle, int32_t* out);
int dgds_cluster_group_version(dgds_cluster* c, int32_t handle, uint64_t* out);
int dgds_cluster_stored_tokens(dgds_cluster* c, int32_t handle, int32_t request_id, uint64_t* out);
int dgds_cluster_shard_group_count(dgds_cluster* c, int32_t shard, uint64_t* out);
int dgds_cluster_node_count(dgds_cluster* c, uint64_t* out);
/* dgds_update_batch over the cluster (host buffers). */
int dgds_cluster_update_batch(dgds_cluster* c, int64_t n, const int32_t* handles, const int32_t* request_ids,
                              const uint64_t* prev_counts, const uint64_t* tok_offsets, const int32_t* tokens,
                              double now, dgds_update_reply* replies);
/* dgds_speculate_verify_batch over the cluster (host buffers; vout and the truth inputs optional). */
int dgds_cluster_speculate_verify_batch(dgds_cluster* c, int64_t n, const int32_t* handles,
                                        const uint64_t* pat_offsets, const int32_t* patterns,
                                        const dgds_spec_args* args, int64_t args_stride, const int32_t* truth_next,
                                        int32_t truth_stride, const int32_t* truth_left, const int32_t* limit,
                                        dgds_candidates* out, dgds_verify_out* vout);

/* ---- replica sync: GDX1 blobs (cst.cpp:233-329) and DraftServer::fetch_cst (dgds.cpp:53-97) ----
 * Blobs are byte-identical to the reference's: "GDX1", kind (1 delta, 2 full), u16+group id,
 * u64 from, u64 to, u32 count, then delta records {u32 rid, u64 start, u32 len, i32 tokens[len]}
 * or full-snapshot streams {u32 rid, u64 len, i32 tokens[len]} in request-id order, all
 * big-endian. The tokens come from the device history arena that the append kernel fills. */
#define DGDS_FETCH_UP_TO_DATE 0
#define DGDS_FETCH_DELTA 1
#define DGDS_FETCH_FULL 2
#define DGDS_FETCH_UNKNOWN_GROUP 3
typedef struct dgds_fetch_reply {
  int32_t kind;      /* DGDS_FETCH_* (FetchKind, dgds.hpp:31) */
  int32_t reserved;
  uint64_t version;  /* the group's current version */
  uint64_t blob_off; /* the blob is (*blobs)[blob_off .. blob_off + blob_len) */
  uint64_t blob_len;
} dgds_fetch_reply;
/* Per group: UnknownGroup if absent or expired (lazy expiry), else the expiry is refreshed and
 * UpToDate / Delta (cached version still in the log) / Full (cached 0, from the future, or
 * compacted). *blobs points into a server-owned pinned block valid until the next fetch. */
int dgds_fetch_cst(dgds_server* s, int64_t n, const int32_t* handles, const uint64_t* cached_versions, double now,
                   dgds_fetch_reply* replies, const uint8_t** blobs);
/* compact_log: drop log entries before min(before_version, version) (dgds.cpp:153-158). */
int dgds_compact_group(dgds_server* s, int32_t handle, uint64_t before_version);
/* apply_blob on this server's copy of the group (a GPU-resident replica): a delta needs the
 * replica at the blob's from-version; a full snapshot replaces the replica. Errors are
 * DGDS_EBLOB with the reference's messages. *version = the replica's new version. */
int dgds_apply_blob(dgds_server* s, int32_t handle, const uint8_t* blob, uint64_t len, double now,
                    uint64_t* version);

/* ---- memory reclamation (TTL expiry / drop) ----
 * Retired groups' trie slots are dropped by a same-capacity rebuild and their token history
 * by a compaction of the history arena. dgds_drop_group / dgds_sweep_expired run it once
 * retired groups hold > 40% of the history; dgds_compact_memory runs it now. */
typedef struct dgds_memory_stats {
  uint64_t slots, used_slots;
  uint64_t history_capacity, history_tokens, dead_history_tokens;
  uint64_t compactions;
} dgds_memory_stats;
int dgds_compact_memory(dgds_server* s);
int dgds_get_memory_stats(dgds_server* s, dgds_memory_stats* out);

/* ---- framed wire protocol (dgds_wire.hpp:12-28, dgds_wire.cpp) ----
 * Frame = u32 BE length + payload; ops 0x01 update_cst, 0x02 fetch_cst, 0x03 register_group,
 * replies op|0x80, 0x7F error + message; replies byte-identical to the reference's
 * serve_payload. The TCP service (loopback, thread per connection like TcpDraftService)
 * hands frames to one dispatcher that applies every waiting update_cst as ONE batch. */
typedef struct dgds_wire_service dgds_wire_service;
/* update_cst's steps before the append (dgds.cpp:39-48): auto-register or refresh the expiry. */
int dgds_touch_group(dgds_server* s, int32_t handle, double now);
/* One request payload -> reply payload (DGDS_EBUFFER with *out_len set if cap is too small). */
int dgds_wire_serve_payload(dgds_server* s, const uint8_t* payload, uint64_t len, double now, uint8_t* out,
                            uint64_t cap, uint64_t* out_len);
/* port 0 = ephemeral; TTLs use the service's own clock (seconds since start). */
int dgds_wire_service_start(dgds_server* s, int32_t port, dgds_wire_service** out, int32_t* bound_port);
int dgds_wire_service_stats(dgds_wire_service* w, uint64_t* requests, uint64_t* batches);
int dgds_wire_service_stop(dgds_wire_service* w);

/* ---- peer exchange over NVLink / NVSwitch (one process per GPU, CUDA IPC) ----
 * Replaces the all-to-all of the reference's shard routing (dgds.cpp:10-14 routes a
 * group's traffic to shard fnv1a64(gid) % N) with stores straight into the owner's HBM.
 * Each rank owns one zeroed region of region_bytes; every rank maps every region. A
 * channel lives at caller-chosen byte offsets, identical in every region:
 *   flags  u64[world]               sender r's sequence number at flag_off + 8r
 *   counts i32[world] (per parity)  rows sender r delivered, at count_off + 4r
 *   slab   i32[world][cap][words]   sender r's rows at slab_off + 4 * r * cap * words
 * Sequence numbers start at 1 and grow by one per exchange of a channel. */
typedef struct dgds_px dgds_px;
#define DGDS_IPC_HANDLE_BYTES 64
int dgds_px_create(int32_t device, int32_t world, int32_t rank, uint64_t region_bytes, dgds_px** out,
                   void* handle_out /* DGDS_IPC_HANDLE_BYTES, may be NULL */);
/* handles: world * DGDS_IPC_HANDLE_BYTES in rank order (this rank's entry is ignored) */
int dgds_px_connect(dgds_px* px, const void* handles);
/* All ranks in this process (tests; different devices need peer access) */
int dgds_px_connect_local(dgds_px* const* all, int32_t world);
int dgds_px_region(dgds_px* px, int32_t peer, void** base);
/* Send record i (rec_words int32) to rank d_owner[i] (owners outside [0, world) are dropped):
 * rows are written into the owner's slab, then counts and flag = seq are published.
 * d_slot (optional) [i] = owner * cap + row, or -1. origin_word >= 0 overwrites that word of
 * each delivered row with i (for replies stored in the sender's order). stable != 0 keeps
 * record order per owner (one CTA); otherwise rows are unordered.
 * Rows beyond cap set *d_overflow = 1 (sticky) and are dropped. */
int dgds_px_send(dgds_px* px, int64_t n, const int32_t* d_owner, const int32_t* d_records, int32_t rec_words,
                 int64_t cap, uint64_t slab_off, uint64_t count_off, uint64_t flag_off, uint64_t seq,
                 int32_t stable, int32_t origin_word, int64_t* d_slot, int32_t* d_overflow, void* stream);
/* Kernels enqueued after this see every sender's data of exchange `seq` (bounded spin). */
int dgds_px_wait(dgds_px* px, uint64_t flag_off, uint64_t seq, void* stream);
/* Publish flag = seq to every peer after the work already enqueued on `stream`. */
int dgds_px_signal(dgds_px* px, uint64_t flag_off, uint64_t seq, void* stream);
/* timed_out = 1 once a wait gave up (synchronous read); launches = px kernels enqueued. */
int dgds_px_status(dgds_px* px, int32_t* timed_out, uint64_t* launches);
int dgds_px_set_timeout(dgds_px* px, uint64_t timeout_ns);
int dgds_px_destroy(dgds_px* px);

/* The routed tick loop of one rank in C++ (bench_multi.py's pipeline without the interpreter):
 * per tick s, the rank's append rows go to their owners (side stream; their metadata rows come
 * back to pinned memory for the server's planner thread), its query rows go to their owners
 * once tick s-1's replies are home (second side stream), and on the main stream the owner runs
 * K2 + fused K3 on the queries it received (replies into the senders' shared reply slab, row =
 * q_origin_word), waits for its own replies, then launches K1 with tick s's routed plan.
 * Channels are described exactly as laid out in the px regions (identical on every rank). */
typedef struct dgds_px_channel_desc {
  int32_t rows, words;     /* rows per sender (shared: of the whole slab), int32 words per row */
  int32_t shared, pad;     /* shared: one slab addressed by row (replies) */
  uint64_t flag_off;
  uint64_t count_off[2];   /* by parity seq % 2 */
  uint64_t slab_off[2];
} dgds_px_channel_desc;
typedef struct dgds_px_tick {  /* one tick's device-resident rows produced by this rank */
  int64_t n_q, n_a;
  const int32_t* q_owner;  /* [n_q] owner rank */
  const int32_t* q;        /* [n_q][q.words] query records (dgds_query_record_layout) */
  const int32_t* a_owner;  /* [n_a] */
  const int32_t* a;        /* [n_a][a.words]: handle | request id | prev lo | prev hi | count | tokens */
} dgds_px_tick;
typedef struct dgds_px_driver dgds_px_driver;
int dgds_px_driver_create(dgds_server* s, dgds_px* px, int32_t world, int32_t rank, const dgds_px_channel_desc* q,
                          const dgds_px_channel_desc* rep, const dgds_px_channel_desc* a, int32_t q_origin_word,
                          const dgds_query_record_layout* layout, const dgds_spec_args* d_args, int32_t max_top_k,
                          int32_t max_spec, int32_t* d_overflow, const dgds_px_tick* ticks, int64_t n_ticks,
                          void* main_stream, dgds_px_driver** out);
/* Ticks [first, last) on the main stream (returns once enqueued); ticks < plan_to (0: last) may
 * be planned ahead — e.g. a warm-up run plans the first tick of the next run. */
int dgds_px_driver_run(dgds_px_driver* d, int64_t first, int64_t last, int64_t plan_to, dgds_query_stats* d_stats);
/* Launches any tick planned ahead but not run, waits for the driver's streams, frees it. */
int dgds_px_driver_destroy(dgds_px_driver* d);

#ifdef __cplusplus
}
#endif

#endif /* DGDS_B200_H */

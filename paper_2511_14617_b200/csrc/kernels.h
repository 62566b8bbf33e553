// kernels.h — host-side launch interface of the sm_100a kernels (K1 append,
// K2 draft query + fused K3 verify, standalone verify, arena rebuild, routing).
#pragma once

#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include <atomic>

#include "../../include/dgds_b200.h"
#include "trie.cuh"

namespace dgds {

// Kernels enqueued by the launch helpers below (process-wide; dgds_kernel_launches)
extern std::atomic<unsigned long long> g_kernel_launches;

// One warp per segment: all records of one request stream inside one batch, in
// call order: n tokens at stream positions start .. start + n, read from the
// stream's history extent (staged there by k_stage).
struct AppendSeg {
  uint32_t stream;    // stream slot (row of DevTrie::active)
  uint32_t root;      // group root id
  uint64_t start;     // tokens stored for the stream before this batch
  uint64_t sh_base;   // the stream's extent in DevTrie::shist (after any growth)
  uint32_t n;         // tokens appended in this batch
  uint32_t pad_;
};
static_assert(sizeof(AppendSeg) == 32, "AppendSeg is 32 B");

struct AppendPiece {  // one record's tokens: batch buffer -> history arena + stream extent
  uint64_t tok_off;   // into the batch token buffer
  uint64_t hist_off;  // history arena (record order, replica blobs)
  uint64_t sh_off;    // stream extent position (DevTrie::shist)
  uint32_t n;
  uint32_t pad_;
};
static_assert(sizeof(AppendPiece) == 32, "AppendPiece is 32 B");

// One piece of a GDX1 blob (cst.cpp:233-269), serialised big-endian on the device:
// an optional header right before `dst` — kind 1: delta record {u32 rid, u64 start, u32 len}
// (16 B), kind 2: full-snapshot stream {u32 rid, u64 len} (12 B) — then `len` tokens copied
// from the history arena at src as big-endian i32.
struct BlobPiece {
  uint64_t src;  // history arena offset (tokens)
  uint64_t dst;  // byte offset of the first token in the output
  uint64_t hdr_a;  // start (kind 1) or stream length (kind 2)
  uint32_t len;  // tokens
  uint32_t rid;
  uint32_t hdr_kind;
  uint32_t pad_;
};
struct CopyPiece {  // history compaction: len tokens from src to dst
  uint64_t src, dst;
  uint32_t len, pad_;
};
cudaError_t launch_copy_pieces(const CopyPiece* d_pieces, int64_t n, const int32_t* from, int32_t* to, cudaStream_t st);
cudaError_t launch_blob_fill(const BlobPiece* d_pieces, int64_t n, const int32_t* hist, uint8_t* out,
                             cudaStream_t st);

// k_stage (tokens -> history arena + stream extents, stream table rows) then K1. Extent growth
// copies (grow, ngrow: old extent -> new extent, within shist) run first.
cudaError_t launch_append(const DevTrie& T, const AppendSeg* d_segs, int64_t nseg, const AppendPiece* d_pieces,
                          int64_t npieces, const int32_t* d_tokens, const CopyPiece* d_grow, int64_t ngrow,
                          cudaStream_t st);

int set_error(int code, const std::string& msg);  // dgds_last_error() message (server.cpp)

constexpr int kMaxSegments = 8;
constexpr int kStatParts = 64;  // partitions of the query counters (spreads the REDs)  // senders of a segmented query launch (ranks of one node)

struct CplxRec {  // a query whose locus is a node (K2a -> K2b)
  int64_t q;
  uint32_t fc, cnt;
  int32_t winner, lookups;
};

struct QueryLaunch {
  DevTrie T;
  const uint32_t* root_of;
  int32_t n_handles;
  int32_t reserved0;
  int64_t n;
  const int32_t* handles;
  const int32_t* pat_len;
  const int32_t* patterns;
  int32_t pat_stride;
  int32_t k_stride;
  const dgds_spec_args* args;
  int64_t args_stride;
  int32_t s_stride;
  int32_t truth_stride;
  int32_t* n_cands;
  int32_t* lens;
  double* scores;
  int64_t* supports;
  int32_t* tokens;
  const int32_t* truth;
  const int32_t* truth_left;
  const int32_t* limit;
  int32_t* v_drafted;
  int32_t* v_accepted;
  int32_t* v_emitted;
  dgds_query_stats* stats;          // optional: counters added here (by the last block)
  unsigned long long* stat_part;    // server scratch [kStatParts][8] + a block ticket, zero between launches
  int32_t* err_flag;  // set to 1 by any query with invalid args (device API)
  long long* dbg;     // optional per-query phase timing [n][8] (debug)
  // Per-query strides (elements). SoA buffers: in_qstride 1, out_qstride = out_qstride8 = k_stride,
  // tok_qstride = k_stride * s_stride, v_qstride 1. Routed records: all = the record width.
  int64_t in_qstride;   // handles, pat_len, truth_left, limit
  int64_t nc_qstride;   // n_cands
  int64_t out_qstride;  // lens (int32 units)
  int64_t out_qstride8; // scores, supports (8-byte units)
  int64_t tok_qstride;  // tokens (int32 units; candidate c at + c * s_stride)
  int64_t v_qstride;    // drafted / accepted / emitted
  // Reply-record output (rec_words_out > 0; replaces the SoA pointers above): the reply row of
  // query q is R = rec_out + q * rec_words_out, or with seg_rows > 0 (rows arrive in per-sender
  // segments of seg_rows, valid while j < seg_count[s]) R = seg_out[s] + j * rec_words_out —
  // typically the sender's receive region in NVLink peer memory.
  int32_t rec_words_out;
  int32_t off_nc, off_len, off_sc, off_sp, off_tk, off_v;  // field offsets in the row (int32 units; -1 = absent)
  int32_t* rec_out;
  int64_t seg_rows;
  const int32_t* seg_count;
  const int32_t* seg_origin;  // optional: the reply row is seg_origin[q * in_qstride] instead of j
  // Engine zero-copy: the pattern of query q ends at patterns[pat_end[q]] (exclusive)
  // in one long token buffer, and its reply record starts at rec_out + out_off[q].
  const int64_t* pat_end;
  const int64_t* out_off;
  int32_t* seg_out[kMaxSegments];
  // K2a -> K2b queue of queries whose locus is a node (null: one whole-query kernel), and
  // [0] its length, [1] K2b's warp ticket; server scratch of n entries, zero between launches
  CplxRec* cplx;
  unsigned long long* cplx_count;
  // Engine decode step (dgds_decode_step_device): the query's args, pattern length and the
  // no-query rule are derived per request on the device from its generated-token count and
  // limit; the last warp settles the step (totals, next draft length).
  int32_t engine;
  int32_t draft_len;              // this step's d when draft_len_dev is null
  const int32_t* draft_len_dev;   // device scalar d (e.g. the previous step's next_draft_len)
  const int32_t* gen;             // generated tokens per request
  dgds_spec_policy policy;
  unsigned long long* step_acc;   // server scratch [4], zero between launches
  int32_t* next_draft_len;        // out (device scalar), optional
  long long* step_totals;         // out [4]: still running, drafted, accepted, emitted; optional
};

// SoA strides for a QueryLaunch whose outputs are [n][k_stride][s_stride] buffers.
inline void soa_strides(QueryLaunch& L) {
  L.in_qstride = 1;
  L.nc_qstride = 1;
  L.out_qstride = L.k_stride;
  L.out_qstride8 = L.k_stride;
  L.tok_qstride = static_cast<int64_t>(L.k_stride) * L.s_stride;
  L.v_qstride = 1;
}

// max_k selects the tile width (4, 8 or 32 lanes per request); max_s bounds
// min(max_spec_tokens, max_spec_len) over the batch (per-path token registers).
cudaError_t launch_query(const QueryLaunch& L, int32_t max_k, int32_t max_s, cudaStream_t st);

cudaError_t launch_verify(int64_t n, int32_t k_stride, int32_t s_stride, const int32_t* n_cands, const int32_t* lens,
                          const int32_t* tokens, const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                          const int32_t* limit, int32_t* drafted, int32_t* accepted, int32_t* emitted,
                          cudaStream_t st);

cudaError_t launch_set_u32(uint32_t* dst, uint32_t value, cudaStream_t st);

// Arena rebuild (growth + garbage collection of dropped groups): re-place every
// live slot of `from` in `to` (home slots depend on content only), then rewrite
// parents / child lists through the old->new id map. root_alive: bitmap over
// root indices.
cudaError_t launch_rebuild(const DevTrie& from, const DevTrie& to, const uint32_t* root_alive, uint32_t* remap,
                           cudaStream_t st);
// active / ov rows of the given streams through the old->new id map
cudaError_t launch_remap_active(const DevTrie& T, const uint32_t* streams, int64_t nstreams, const uint32_t* remap,
                                cudaStream_t st, uint64_t from_cap);
// Logical trie nodes of the arena (the reference's node count without roots): entries plus the
// implicit chain below every leaf. out[0] += total (one u64).
cudaError_t launch_node_count(const DevTrie& T, unsigned long long* out, cudaStream_t st);

// Dense per-candidate record of the host path's compacted results.
struct CandMeta {
  double score;
  int64_t support;
  int32_t len;
  int32_t pad;
};
constexpr int kMaxCopyRegions = 8;
struct CopyOutRegions {
  int32_t n;
  int32_t total_idx[kMaxCopyRegions];   // < 0: fixed size fixed_bytes[r]
  int32_t begin_idx[kMaxCopyRegions];   // >= 0 (sized regions): start at element totals[begin_idx[r]]
  int32_t elem_bytes[kMaxCopyRegions];
  int64_t fixed_bytes[kMaxCopyRegions];
  const char* src[kMaxCopyRegions];  // src[r] and dst[r] congruent mod 16
  char* dst[kMaxCopyRegions];        // typically mapped pinned host memory
};
// Copies bytes [b0, b1) of region r: b1 = totals[total_idx[r]] * elem_bytes[r] (b0 from begin_idx)
// or [0, fixed_bytes[r]); sizes are multiples of 4. max_bytes sizes the grid.
cudaError_t launch_copy_out(const long long* totals, const CopyOutRegions& R, int64_t max_bytes, cudaStream_t st,
                            int max_blocks = 592);

// Compaction input: per-query candidate fields at query strides (elements), e.g. the query
// kernel's SoA outputs or fixed-size reply records.
struct CmpIn {
  const int32_t* n_cands;
  int64_t qs_nc;
  const int32_t* lens;  // lens[q * qs_len + j]
  int64_t qs_len;
  const double* scores;
  int64_t qs_sc;
  const int64_t* supports;
  int64_t qs_sp;
  const int32_t* tokens;  // tokens[q * qs_tok + j * cs_tok + i]
  int64_t qs_tok;
  int32_t cs_tok;
  const int32_t* verify;  // optional: drafted, accepted, emitted at verify[q * qs_v + 0..2]
  int64_t qs_v;
};
cudaError_t launch_compact_in(int64_t n, const CmpIn& in, long long* block_sums, long long* totals, CandMeta* meta,
                              int32_t* tok_out, int64_t* cand_off, int64_t* tok_off, int32_t* v_out,
                              const long long* carry_in, cudaStream_t st);

// block_sums: 2 * ceil(n / 256) scratch; totals[0] = candidates, totals[1] = tokens, both
// counted from carry_in (optional: the totals of an earlier chunk, so chunks of one batch
// compact into one CSR). Outputs may live in mapped pinned host memory.
// cand_off[q] (optional) = first candidate of query q; tok_off[c] (optional) = first token of c.
cudaError_t launch_compact(int64_t n, int32_t K, int32_t S, const int32_t* n_cands, const int32_t* lens,
                           const double* scores, const int64_t* supports, const int32_t* tokens,
                           long long* block_sums, long long* totals, CandMeta* meta, int32_t* tok_out,
                           int64_t* cand_off, int64_t* tok_off, const long long* carry_in, cudaStream_t st);

cudaError_t launch_route_pack(int64_t n, int32_t world, const int32_t* owner, const uint32_t* records,
                              int32_t rec_words, uint32_t* out, int64_t* counts, int64_t* perm, void* scratch,
                              cudaStream_t st);
cudaError_t launch_route_pack_padded(int64_t n, int32_t world, const int32_t* owner, const uint32_t* records,
                                     int32_t rec_words, int64_t cap, uint32_t* out, int64_t* slot, int32_t* overflow,
                                     void* scratch, cudaStream_t st);
cudaError_t launch_route_unpack(int64_t n, const uint32_t* in, int32_t rec_words, const int64_t* perm, uint32_t* out,
                                cudaStream_t st);

}  // namespace dgds

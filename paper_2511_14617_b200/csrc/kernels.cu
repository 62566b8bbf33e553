// kernels.cu — sm_100a kernels of the DGDS hot path.
//
//   K1 k_append      batched incremental insertion of appended tokens into the
//                    per-group counted suffix tries (GroupDraftIndex::append /
//                    insert_token / ensure_child, proj/src/cst.cpp:90-133).
//   K2 k_query<K>    batched longest-suffix match + top-k beam expansion
//                    (GroupDraftIndex::speculate, cst.cpp:153-228), one warp per
//                    request, with
//   K3               fused verification / accept length (Instance::decode_step,
//                    proj/src/engine.cpp:115-143); k_verify is the standalone form.
//   k_rebuild_level  arena growth + GC of dropped groups (no reference analogue:
//                    the reference's EdgeMap::grow, cst.cpp:63-74, rehashes keys only).
//   k_route_*        owner bucketing for the multi-GPU all-to-all (dgds.cpp:10-14 routing).
//
// Nothing here is a dense contraction, so there is no tensor-core path: every
// kernel is bound by dependent 32-B sector accesses to HBM / L2.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace dgds {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / kWarp;

__device__ __forceinline__ int lane_id() { return threadIdx.x & (kWarp - 1); }

// ---------------------------------------------------------------------------
// K1: append
//
// One warp per stream segment. Lane i keeps active[i], the node of the last
// (i+1)-token context of the stream (Stream::active, cst.hpp:115-118). For
// each new token t the lanes i < min(depth_cap, len+1) ensure the child
// (active[i-1], t) — lane 0 uses the group root — and bump its count, exactly
// insert_token's loop (cst.cpp:105-116) with the depth levels in parallel:
// up to 24 independent claim-or-find CASes in flight per warp per token.

struct EnsureResult {
  uint32_t id;
  bool inserted;
};

__device__ __forceinline__ EnsureResult ensure_child(const DevTrie& T, uint32_t parent, int32_t token, uint32_t depth,
                                                     uint32_t root) {
  const unsigned long long key = edge_key(parent, token);
  uint64_t i = home_slot(key, T.cap);
  while (true) {
    Slot* s = T.slots + i;
    const unsigned long long old = atomicCAS(&s->key, 0ull, key);
    if (old == 0ull || old == key) {
      atomicAdd(&s->count, 1u);  // RED: result unused
      if (old == 0ull) {
        s->depth = depth;
        s->root = root;
      }
      return EnsureResult{static_cast<uint32_t>(i + 1), old == 0ull};
    }
    i = (i + 1 == T.cap) ? 0 : i + 1;
  }
}

__global__ void __launch_bounds__(kBlock) k_append(DevTrie T, const AppendSeg* __restrict__ segs, int64_t nseg,
                                                   const AppendPiece* __restrict__ pieces,
                                                   const int32_t* __restrict__ tokens) {
  const int lane = lane_id();
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * blockDim.x / kWarp;
  const int D = T.depth_cap;
  unsigned long long inserted_total = 0;

  for (int64_t sg = warp; sg < nseg; sg += nwarps) {
    const AppendSeg g = segs[sg];
    uint64_t len = g.start;
    uint32_t* act_row = T.active + static_cast<uint64_t>(g.stream) * kWarp;
    uint32_t a = (lane < D && static_cast<uint64_t>(lane) < len) ? act_row[lane] : 0u;
    // deferred sibling link of the node this lane created at the previous token
    uint32_t link_slot = 0, link_prev = 0;
    bool link_pending = false;

    for (uint32_t p = 0; p < g.npieces; ++p) {
      const AppendPiece pc = pieces[g.piece0 + p];
      for (uint32_t base = 0; base < pc.n; base += kWarp) {
        // stage 32 tokens per coalesced load, broadcast by shuffle
        const int32_t tchunk = (base + lane < pc.n) ? tokens[pc.tok_off + base + lane] : 0;
        const uint32_t cnt = min(static_cast<uint32_t>(kWarp), pc.n - base);
        for (uint32_t j = 0; j < cnt; ++j) {
          const int32_t t = __shfl_sync(kFull, tchunk, j);
          const int newsize = static_cast<int>(min(static_cast<uint64_t>(D), len + 1));
          uint32_t parent = __shfl_up_sync(kFull, a, 1);
          if (lane == 0) parent = g.root;
          if (lane < newsize) {
            const EnsureResult r = ensure_child(T, parent, t, static_cast<uint32_t>(lane + 1), g.root);
            if (link_pending) {
              T.slots[link_slot].next_sibling = link_prev;
              link_pending = false;
            }
            if (r.inserted) {
              ++inserted_total;
              if (!is_root_id(parent, T.cap)) {
                link_prev = atomicExch(&T.slots[parent - 1].first_child, r.id);
                link_slot = r.id - 1;
                link_pending = true;
              }
            }
            a = r.id;
          }
          ++len;
        }
      }
    }
    if (link_pending) T.slots[link_slot].next_sibling = link_prev;
    if (lane < D && static_cast<uint64_t>(lane) < len) act_row[lane] = a;
  }
  // one counter update per warp
  for (int o = 16; o > 0; o >>= 1) inserted_total += __shfl_xor_sync(kFull, inserted_total, o);
  if (lane == 0 && inserted_total) atomicAdd(T.used, inserted_total);
}

// ---------------------------------------------------------------------------
// K2 + K3: draft query with fused verification.
//
// One warp per request. Phase A (longest admissible suffix, cst.cpp:160-178):
// lane l walks the suffix of length start-l from the group root, so all
// candidate lengths are probed concurrently; the lowest successful lane is the
// reference's first (longest) success. Phase B (beam, cst.cpp:180-221): lane b
// owns beam path b and walks its child list, keeping its own top-k qualifying
// children; the union of the per-lane top-k lists contains the pool's top-k,
// which a warp-wide rank selection extracts with the reference's exact total
// order: FP64 score (cnt/parent_cnt products, IEEE round-to-nearest, in the
// reference's operation order) desc, support desc, token path lexicographic
// asc. Paths of equal length compare lexicographically as (parent path rank,
// token), so only ranks — not token arrays — are compared inside the beam.
// Finals keep the reference's rule: a path is final only when it has no
// qualifying child (cst.cpp:213-214), and the kept set is the top-k under
// candidate_before (cst.cpp:29-33,225-227).

struct QSmemLayout {
  int beam_tok, fin_tok, fin_score, fin_sup, fin_len, cl_score, cl_cnt, cl_tok, cl_id, cl_fc, cl_n, nb_node, nb_fc,
      nb_score, nb_sup, nb_lex, nb_tok_src, nb_tok, total;
};

__host__ __device__ inline QSmemLayout qsmem_layout(int K, int S) {
  QSmemLayout L{};
  int off = 0;
  auto take = [&](int bytes, int align) {
    off = (off + align - 1) / align * align;
    const int r = off;
    off += bytes;
    return r;
  };
  L.fin_score = take(8 * K, 8);
  L.fin_sup = take(8 * K, 8);
  L.cl_score = take(8 * K * K, 8);
  L.nb_score = take(8 * K, 8);
  L.nb_sup = take(8 * K, 8);
  L.beam_tok = take(4 * 2 * K * S, 4);
  L.fin_tok = take(4 * K * S, 4);
  L.fin_len = take(4 * K, 4);
  L.cl_cnt = take(4 * K * K, 4);
  L.cl_tok = take(4 * K * K, 4);
  L.cl_id = take(4 * K * K, 4);
  L.cl_fc = take(4 * K * K, 4);
  L.cl_n = take(4 * K, 4);
  L.nb_node = take(4 * K, 4);
  L.nb_fc = take(4 * K, 4);
  L.nb_lex = take(4 * K, 4);
  L.nb_tok_src = take(4 * K, 4);
  L.nb_tok = take(4 * K, 4);
  L.total = (off + 15) / 16 * 16;
  return L;
}

// lexicographic compare of token arrays (std::vector<int>::operator<)
__device__ __forceinline__ bool tokens_less(const int32_t* a, int la, const int32_t* b, int lb) {
  const int m = la < lb ? la : lb;
  for (int i = 0; i < m; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return la < lb;
}

// candidate_before (cst.cpp:29-33)
__device__ __forceinline__ bool cand_before(double sa, int64_t pa, const int32_t* ta, int la, double sb, int64_t pb,
                                            const int32_t* tb, int lb) {
  if (sa != sb) return sa > sb;
  if (pa != pb) return pa > pb;
  return tokens_less(ta, la, tb, lb);
}

__device__ __forceinline__ int warp_sum_i(int v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_query(QueryLaunch P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = lane_id();
  const int wib = threadIdx.x / kWarp;
  const int64_t q = static_cast<int64_t>(blockIdx.x) * (blockDim.x / kWarp) + wib;
  if (q >= P.n) return;  // warp-uniform

  const int S = P.S;
  const QSmemLayout Ly = qsmem_layout(K, S);
  unsigned char* base = smem_raw + static_cast<size_t>(wib) * Ly.total;
  int32_t* beam_tok = reinterpret_cast<int32_t*>(base + Ly.beam_tok);  // [2][K][S]
  int32_t* fin_tok = reinterpret_cast<int32_t*>(base + Ly.fin_tok);    // [K][S]
  double* fin_score = reinterpret_cast<double*>(base + Ly.fin_score);
  int64_t* fin_sup = reinterpret_cast<int64_t*>(base + Ly.fin_sup);
  int32_t* fin_len = reinterpret_cast<int32_t*>(base + Ly.fin_len);
  double* cl_score = reinterpret_cast<double*>(base + Ly.cl_score);  // [K][K] per-lane sibling lists
  uint32_t* cl_cnt = reinterpret_cast<uint32_t*>(base + Ly.cl_cnt);
  int32_t* cl_tok = reinterpret_cast<int32_t*>(base + Ly.cl_tok);
  uint32_t* cl_id = reinterpret_cast<uint32_t*>(base + Ly.cl_id);
  uint32_t* cl_fc = reinterpret_cast<uint32_t*>(base + Ly.cl_fc);
  int32_t* cl_n = reinterpret_cast<int32_t*>(base + Ly.cl_n);
  uint32_t* nb_node = reinterpret_cast<uint32_t*>(base + Ly.nb_node);
  uint32_t* nb_fc = reinterpret_cast<uint32_t*>(base + Ly.nb_fc);
  double* nb_score = reinterpret_cast<double*>(base + Ly.nb_score);
  int64_t* nb_sup = reinterpret_cast<int64_t*>(base + Ly.nb_sup);
  int32_t* nb_lex = reinterpret_cast<int32_t*>(base + Ly.nb_lex);
  int32_t* nb_tok_src = reinterpret_cast<int32_t*>(base + Ly.nb_tok_src);
  int32_t* nb_tok = reinterpret_cast<int32_t*>(base + Ly.nb_tok);

  const DevTrie& T = P.T;
  const dgds_spec_args a = P.args[q * P.args_stride];
  const int32_t h = P.handles[q];
  const uint32_t root = (h >= 0 && h < P.n_handles) ? P.root_of[h] : 0u;
  const int plen = P.pat_len[q];
  const int eff_pmax = min(a.pattern_lookup_max, T.lim_pattern);  // cst.cpp:156-158
  const int eff_smax = min(a.max_spec_tokens, T.lim_spec);
  const int kq = a.top_k;
  const bool bad_args = a.pattern_lookup_min < 1 || a.pattern_lookup_min > a.pattern_lookup_max ||
                        a.max_spec_tokens < 0 || a.top_k < 1 || a.top_k > K || !(a.min_step_freq >= 0.0) ||
                        a.min_support < 0;
  if (bad_args && lane == 0 && P.err_flag) atomicExch(P.err_flag, 1);

  int nf = 0;  // finals kept (warp-uniform)
  int st_lookups = 0, st_exp = 0, st_csec = 0;

  // Insert one finished path (tokens in shared memory) into the top-kq finals.
  auto finals_offer = [&](const int32_t* toks, int len, double sc, int64_t sup) {
    if (lane == 0) {
      if (nf < kq) {
        for (int i = 0; i < len; ++i) fin_tok[nf * S + i] = toks[i];
        fin_len[nf] = len;
        fin_score[nf] = sc;
        fin_sup[nf] = sup;
        ++nf;
      } else {
        int w = 0;  // worst kept final
        for (int c = 1; c < nf; ++c)
          if (cand_before(fin_score[w], fin_sup[w], fin_tok + w * S, fin_len[w], fin_score[c], fin_sup[c],
                          fin_tok + c * S, fin_len[c]))
            w = c;
        if (cand_before(sc, sup, toks, len, fin_score[w], fin_sup[w], fin_tok + w * S, fin_len[w])) {
          for (int i = 0; i < len; ++i) fin_tok[w * S + i] = toks[i];
          fin_len[w] = len;
          fin_score[w] = sc;
          fin_sup[w] = sup;
        }
      }
    }
    nf = __shfl_sync(kFull, nf, 0);
  };

  if (!bad_args && root != 0u && plen > 0 && a.pattern_lookup_min <= eff_pmax) {
    // ---- phase A: all admissible suffix lengths in parallel ----
    // nlen <= lim_pattern < DGDS_MAX_DEPTH = 32 lanes (checked at server creation).
    const int start = min(eff_pmax, plen);
    const int nlen = start - a.pattern_lookup_min + 1;
    const int row_len = min(plen, P.pat_stride);  // the row holds the last row_len tokens
    const int32_t* pat = P.patterns + q * static_cast<int64_t>(P.pat_stride);
    bool ok = false;
    uint32_t node = 0;
    SlotView rec{};
    int looks = 0;
    if (lane < nlen) {
      const int len = start - lane;
      const int32_t* pt = pat + (row_len - len);
      uint32_t nd = root;
      ok = true;
      for (int i = 0; i < len; ++i) {
        ++looks;
        nd = find_child(T, nd, pt[i], rec);
        if (nd == 0u) {
          ok = false;
          break;
        }
      }
      node = nd;
    }
    const unsigned okm = __ballot_sync(kFull, ok);
    const int win = okm ? __ffs(okm) - 1 : kWarp;
    st_lookups = warp_sum_i(lane <= win ? looks : 0);
    if (okm) {
      {
        // ---- phase B: beam ----
        const uint32_t locus_cnt = __shfl_sync(kFull, rec.count, win);
        const uint32_t locus_fc = __shfl_sync(kFull, rec.first_child, win);
        const uint32_t locus = __shfl_sync(kFull, node, win);
        int nb = 1;
        if (lane == 0) nb_lex[0] = 0;
        __syncwarp();
        uint32_t b_node = locus, b_fc = locus_fc;
        double b_score = 1.0;
        int64_t b_sup = static_cast<int64_t>(locus_cnt);
        int b_lex = 0;
        int cur = 0;
        int d = 0;
        for (; d < eff_smax && nb > 0; ++d) {
          // expansion: lane b walks the child list of beam path b
          bool grew = false;
          int nchild = 0;
          if (lane < nb) {
            int my_n = 0;
            double* ls = cl_score + lane * K;
            uint32_t* lc = cl_cnt + lane * K;
            int32_t* lt = cl_tok + lane * K;
            uint32_t* li = cl_id + lane * K;
            uint32_t* lf = cl_fc + lane * K;
            uint32_t c = b_fc;
            while (c != 0u) {
              const SlotView r = load_slot_nc(T.slots + (c - 1));
              ++nchild;
              const int64_t cnt = static_cast<int64_t>(r.count);
              const double step = __ddiv_rn(static_cast<double>(cnt), static_cast<double>(b_sup));
              if (!(step < a.min_step_freq) && !(cnt < a.min_support)) {
                grew = true;
                const double sc = __dmul_rn(b_score, step);
                const int32_t tok = static_cast<int32_t>(static_cast<uint32_t>(r.key));
                // sorted insert (siblings: same parent path, so the token decides ties)
                int pos = my_n;
                while (pos > 0) {
                  const int pp = pos - 1;
                  const bool better = (sc != ls[pp]) ? (sc > ls[pp])
                                      : (cnt != static_cast<int64_t>(lc[pp])) ? (cnt > static_cast<int64_t>(lc[pp]))
                                                                               : (tok < lt[pp]);
                  if (!better) break;
                  --pos;
                }
                if (pos < kq) {
                  const int last = my_n < kq ? my_n : kq - 1;
                  for (int m = last; m > pos; --m) {
                    ls[m] = ls[m - 1];
                    lc[m] = lc[m - 1];
                    lt[m] = lt[m - 1];
                    li[m] = li[m - 1];
                    lf[m] = lf[m - 1];
                  }
                  ls[pos] = sc;
                  lc[pos] = r.count;
                  lt[pos] = tok;
                  li[pos] = c;
                  lf[pos] = r.first_child;
                  if (my_n < kq) ++my_n;
                }
              }
              c = r.next_sibling;
            }
            cl_n[lane] = my_n;
          }
          st_exp += nb;
          st_csec += warp_sum_i(lane < nb ? (8 * nchild + 31) / 32 : 0);
          __syncwarp();
          // paths with no qualifying child become finals (non-empty ones: d > 0)
          unsigned finm = __ballot_sync(kFull, lane < nb && !grew && d > 0);
          while (finm) {
            const int b = __ffs(finm) - 1;
            finm &= finm - 1;
            const double sc = __shfl_sync(kFull, b_score, b);
            const int64_t sp = __shfl_sync(kFull, b_sup, b);
            finals_offer(beam_tok + (cur * K + b) * S, d, sc, sp);
          }
          // select the next beam: rank every listed child under path_before
          const int slots = nb * kq;
          int nb_next = 0;
          for (int m0 = 0; m0 < slots; m0 += kWarp) {
            const int m = m0 + lane;
            bool valid = false;
            int rank = 0, b = 0, j = 0;
            double sc = 0;
            int64_t sp = 0;
            int plex = 0;
            int32_t tok = 0;
            if (m < slots) {
              b = m / kq;
              j = m - b * kq;
              valid = j < cl_n[b];
            }
            if (valid) {
              sc = cl_score[b * K + j];
              sp = static_cast<int64_t>(cl_cnt[b * K + j]);
              tok = cl_tok[b * K + j];
              plex = nb_lex[b];
              for (int b2 = 0; b2 < nb; ++b2) {
                const int n2 = cl_n[b2];
                const int plex2 = nb_lex[b2];
                for (int j2 = 0; j2 < n2; ++j2) {
                  const double sc2 = cl_score[b2 * K + j2];
                  const int64_t sp2 = static_cast<int64_t>(cl_cnt[b2 * K + j2]);
                  const int32_t tok2 = cl_tok[b2 * K + j2];
                  const bool before = (sc2 != sc)   ? (sc2 > sc)
                                      : (sp2 != sp) ? (sp2 > sp)
                                      : (plex2 != plex) ? (plex2 < plex)
                                                        : (tok2 < tok);
                  rank += before ? 1 : 0;
                }
              }
            }
            nb_next += warp_sum_i(valid ? 1 : 0);
            if (valid && rank < kq) {
              nb_node[rank] = cl_id[b * K + j];
              nb_fc[rank] = cl_fc[b * K + j];
              nb_score[rank] = sc;
              nb_sup[rank] = sp;
              nb_tok_src[rank] = b;
              nb_tok[rank] = tok;
            }
          }
          if (nb_next > kq) nb_next = kq;
          // beam slot b currently holds the parent lexrank in nb_lex[b]; compute the
          // children's lexrank among the selected set before overwriting it
          __syncwarp();
          int new_lex = 0;
          if (lane < nb_next) {
            const int src = nb_tok_src[lane];
            const int pl = nb_lex[src];
            const int32_t tk = nb_tok[lane];
            for (int o = 0; o < nb_next; ++o) {
              const int pl2 = nb_lex[nb_tok_src[o]];
              const int32_t tk2 = nb_tok[o];
              new_lex += (pl2 < pl || (pl2 == pl && tk2 < tk)) ? 1 : 0;
            }
            // tokens: parent path + new token
            const int32_t* src_tok = beam_tok + (cur * K + src) * S;
            int32_t* dst_tok = beam_tok + ((cur ^ 1) * K + lane) * S;
            for (int i = 0; i < d; ++i) dst_tok[i] = src_tok[i];
            dst_tok[d] = tk;
          }
          __syncwarp();
          if (lane < nb_next) {
            nb_lex[lane] = new_lex;
            b_node = nb_node[lane];
            b_fc = nb_fc[lane];
            b_score = nb_score[lane];
            b_sup = nb_sup[lane];
            b_lex = new_lex;
          }
          __syncwarp();
          nb = nb_next;
          cur ^= 1;
        }
        (void)b_node;
        (void)b_lex;
        // leftover beam paths (d tokens each) are finals when non-empty
        if (d > 0) {
          for (int b = 0; b < nb; ++b) {
            const double sc = __shfl_sync(kFull, b_score, b);
            const int64_t sp = __shfl_sync(kFull, b_sup, b);
            finals_offer(beam_tok + (cur * K + b) * S, d, sc, sp);
          }
        }
      }
    }  // no match at any admissible length: empty (no shorter fallback once matched)
  }

  // ---- output in candidate_before order ----
  __syncwarp();
  int my_rank = 0;
  if (lane < nf) {
    for (int c = 0; c < nf; ++c)
      my_rank += cand_before(fin_score[c], fin_sup[c], fin_tok + c * S, fin_len[c], fin_score[lane], fin_sup[lane],
                             fin_tok + lane * S, fin_len[lane])
                     ? 1
                     : 0;
  }
  if (P.n_cands) {
    if (lane == 0) P.n_cands[q] = nf;
    if (lane < nf) {
      const int64_t o = q * P.k_stride + my_rank;
      P.lens[o] = fin_len[lane];
      P.scores[o] = fin_score[lane];
      P.supports[o] = fin_sup[lane];
      int32_t* dst = P.tokens + o * P.s_stride;
      for (int i = 0; i < fin_len[lane]; ++i) dst[i] = fin_tok[lane * S + i];
    }
  }

  // ---- K3: verification (engine.cpp:115-143) ----
  if (P.v_emitted) {
    int drafted = 0, match = 0;
    if (lane < nf) {
      drafted = fin_len[lane];
      const int32_t* tr = P.truth + q * static_cast<int64_t>(P.truth_stride);
      const int cap = min(fin_len[lane], P.truth_left[q]);
      while (match < cap && fin_tok[lane * S + match] == tr[match]) ++match;
    }
    drafted = warp_sum_i(drafted);
    for (int o = 16; o > 0; o >>= 1) match = max(match, __shfl_xor_sync(kFull, match, o));
    if (lane == 0) {
      const int emitted = min(match + 1, P.limit[q]);
      P.v_drafted[q] = drafted;
      P.v_accepted[q] = emitted - 1;
      P.v_emitted[q] = emitted;
    }
  }

  if (P.stats) {
    int ctoks = lane < nf ? fin_len[lane] : 0;
    ctoks = warp_sum_i(ctoks);
    if (lane == 0) {
      const uint64_t B = 4ull * plen + 32ull + 32ull * st_lookups + 32ull * st_exp + 32ull * st_csec +
                         4ull * ctoks + 16ull * nf;
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->queries), 1ull);
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->pattern_tokens), static_cast<unsigned long long>(plen));
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->suffix_lookups),
                static_cast<unsigned long long>(st_lookups));
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->expansions), static_cast<unsigned long long>(st_exp));
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->child_sectors),
                static_cast<unsigned long long>(st_csec));
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->cands), static_cast<unsigned long long>(nf));
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->cand_tokens), static_cast<unsigned long long>(ctoks));
      atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats->algorithmic_bytes), static_cast<unsigned long long>(B));
    }
  }
}

// ---------------------------------------------------------------------------
// standalone verify (engine.cpp:115-143), one thread per request

__global__ void k_verify(int64_t n, int32_t k_stride, int32_t s_stride, const int32_t* __restrict__ n_cands,
                         const int32_t* __restrict__ lens, const int32_t* __restrict__ tokens,
                         const int32_t* __restrict__ truth, int32_t truth_stride,
                         const int32_t* __restrict__ truth_left, const int32_t* __restrict__ limit,
                         int32_t* drafted, int32_t* accepted, int32_t* emitted) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  int dr = 0, acc = 0;
  const int32_t* tr = truth + q * truth_stride;
  for (int c = 0; c < n_cands[q]; ++c) {
    const int len = lens[q * k_stride + c];
    dr += len;
    const int cap = min(len, truth_left[q]);
    const int32_t* tk = tokens + (q * k_stride + c) * s_stride;
    int m = 0;
    while (m < cap && tk[m] == tr[m]) ++m;
    acc = max(acc, m);
  }
  const int em = min(acc + 1, limit[q]);
  drafted[q] = dr;
  accepted[q] = em - 1;
  emitted[q] = em;
}

__global__ void k_set_u32(uint32_t* dst, uint32_t v) { *dst = v; }

// ---------------------------------------------------------------------------
// rebuild: re-insert live nodes of depth `depth` from `from` into `to`

__global__ void k_rebuild_level(DevTrie from, DevTrie to, uint32_t depth, const uint32_t* __restrict__ root_alive,
                                uint32_t* remap) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < from.cap; i += stride) {
    const Slot s = from.slots[i];
    if (s.key == 0ull || s.depth != depth) continue;
    const uint32_t ridx = kRootTop - s.root;
    if (!((root_alive[ridx >> 5] >> (ridx & 31)) & 1u)) {
      remap[i] = 0;
      continue;
    }
    const uint32_t parent = static_cast<uint32_t>(s.key >> 32);
    uint32_t np = parent;
    if (!is_root_id(parent, from.cap)) {
      np = remap[parent - 1];
      if (np == 0u) {
        remap[i] = 0;
        continue;
      }
    }
    const unsigned long long key = edge_key(np, static_cast<int32_t>(static_cast<uint32_t>(s.key)));
    uint64_t j = home_slot(key, to.cap);
    while (atomicCAS(&to.slots[j].key, 0ull, key) != 0ull) j = (j + 1 == to.cap) ? 0 : j + 1;
    Slot* d = to.slots + j;
    d->count = s.count;
    d->depth = s.depth;
    d->root = s.root;
    const uint32_t nid = static_cast<uint32_t>(j + 1);
    if (!is_root_id(np, to.cap)) d->next_sibling = atomicExch(&to.slots[np - 1].first_child, nid);
    remap[i] = nid;
    atomicAdd(to.used, 1ull);
  }
}

__global__ void k_remap_active(uint32_t* active, const uint32_t* __restrict__ streams,
                               const uint32_t* __restrict__ sizes, int64_t ns, const uint32_t* __restrict__ remap) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t s = t / kWarp;
  const int l = static_cast<int>(t % kWarp);
  if (s >= ns) return;
  if (static_cast<uint32_t>(l) >= sizes[s]) return;
  uint32_t* row = active + static_cast<uint64_t>(streams[s]) * kWarp;
  const uint32_t v = row[l];
  row[l] = v ? remap[v - 1] : 0u;
}

// ---------------------------------------------------------------------------
// routing: stable bucketing of fixed-size records by owner rank

constexpr int kRouteTile = 1024;

__global__ void k_route_count(int64_t n, int32_t world, const int32_t* __restrict__ owner, int64_t* tile_counts) {
  // tile_counts[o * ntiles + tile]
  extern __shared__ int sh_cnt[];
  for (int o = threadIdx.x; o < world; o += blockDim.x) sh_cnt[o] = 0;
  __syncthreads();
  const int64_t ntiles = gridDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRouteTile + threadIdx.x;
       i < min(n, static_cast<int64_t>(blockIdx.x + 1) * kRouteTile); i += blockDim.x)
    atomicAdd(&sh_cnt[owner[i]], 1);
  __syncthreads();
  for (int o = threadIdx.x; o < world; o += blockDim.x) tile_counts[o * ntiles + blockIdx.x] = sh_cnt[o];
}

__global__ void k_route_scan(int64_t total_entries, int32_t world, int64_t ntiles, int64_t* tile_counts,
                             int64_t* counts) {
  // single thread: exclusive scan in (owner, tile) order; tiny (world * ntiles entries)
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t run = 0;
  for (int o = 0; o < world; ++o) {
    int64_t c = 0;
    for (int64_t t = 0; t < ntiles; ++t) {
      const int64_t v = tile_counts[o * ntiles + t];
      tile_counts[o * ntiles + t] = run;
      run += v;
      c += v;
    }
    counts[o] = c;
  }
  (void)total_entries;
}

__global__ void k_route_scatter(int64_t n, int32_t world, const int32_t* __restrict__ owner,
                                const uint32_t* __restrict__ rec, int32_t rw, const int64_t* __restrict__ tile_off,
                                uint32_t* out, int64_t* perm) {
  // one block per tile; stable ranks within the tile, warp by warp
  __shared__ int warp_cnt[kRouteTile / kWarp][8];
  const int64_t ntiles = gridDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kRouteTile;
  const int warp = threadIdx.x / kWarp, lane = lane_id();
  // this kernel is launched with kRouteTile threads and world <= 8 in the fast path
  const int64_t i = t0 + threadIdx.x;
  const int o = (i < n) ? owner[i] : -1;
  int my_rank_in_warp = 0;
  for (int w = 0; w < world; ++w) {
    const unsigned m = __ballot_sync(kFull, o == w);
    if (o == w) my_rank_in_warp = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) warp_cnt[warp][w] = __popc(m);
  }
  __syncthreads();
  if (o >= 0) {
    int64_t pos = tile_off[o * ntiles + blockIdx.x];
    for (int w2 = 0; w2 < warp; ++w2) pos += warp_cnt[w2][o];
    pos += my_rank_in_warp;
    for (int k = 0; k < rw; ++k) out[pos * rw + k] = rec[i * rw + k];
    perm[i] = pos;
  }
}

__global__ void k_route_gather(int64_t n, const uint32_t* __restrict__ in, int32_t rw, const int64_t* __restrict__ perm,
                               uint32_t* out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * rw) return;
  const int64_t i = t / rw;
  const int k = static_cast<int>(t % rw);
  out[t] = in[perm[i] * rw + k];
}

template <int K>
cudaError_t launch_query_k(const QueryLaunch& L, cudaStream_t st) {
  const QSmemLayout Ly = qsmem_layout(K, L.S);
  constexpr int kSmemBudget = 200 * 1024;
  int wpb = kWarpsPerBlock;
  while (wpb > 1 && Ly.total * wpb > kSmemBudget) --wpb;
  const size_t smem = static_cast<size_t>(Ly.total) * wpb;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_query<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = (L.n + wpb - 1) / wpb;
  k_query<K><<<static_cast<unsigned>(blocks), wpb * kWarp, smem, st>>>(L);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_append(const DevTrie& T, const AppendSeg* d_segs, int64_t nseg, const AppendPiece* d_pieces,
                          const int32_t* d_tokens, cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  const int64_t blocks = (nseg + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_append<<<static_cast<unsigned>(blocks), kBlock, 0, st>>>(T, d_segs, nseg, d_pieces, d_tokens);
  return cudaGetLastError();
}

cudaError_t launch_query(const QueryLaunch& L, int32_t max_k, cudaStream_t st) {
  if (L.n <= 0) return cudaSuccess;
  if (max_k <= 1) return launch_query_k<1>(L, st);
  if (max_k <= 2) return launch_query_k<2>(L, st);
  if (max_k <= 4) return launch_query_k<4>(L, st);
  if (max_k <= 8) return launch_query_k<8>(L, st);
  if (max_k <= 16) return launch_query_k<16>(L, st);
  return launch_query_k<32>(L, st);
}

cudaError_t launch_verify(int64_t n, int32_t k_stride, int32_t s_stride, const int32_t* n_cands, const int32_t* lens,
                          const int32_t* tokens, const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                          const int32_t* limit, int32_t* drafted, int32_t* accepted, int32_t* emitted,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_verify<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, k_stride, s_stride, n_cands, lens, tokens,
                                                                      truth, truth_stride, truth_left, limit, drafted,
                                                                      accepted, emitted);
  return cudaGetLastError();
}

cudaError_t launch_set_u32(uint32_t* dst, uint32_t value, cudaStream_t st) {
  k_set_u32<<<1, 1, 0, st>>>(dst, value);
  return cudaGetLastError();
}

cudaError_t launch_rebuild_level(const DevTrie& from, const DevTrie& to, uint32_t depth, const uint32_t* root_alive,
                                 uint32_t* remap, cudaStream_t st) {
  k_rebuild_level<<<148 * 8, 256, 0, st>>>(from, to, depth, root_alive, remap);
  return cudaGetLastError();
}

cudaError_t launch_remap_active(uint32_t* active, const uint32_t* streams, const uint32_t* sizes, int64_t nstreams,
                                const uint32_t* remap, uint64_t old_cap, cudaStream_t st) {
  (void)old_cap;
  if (nstreams <= 0) return cudaSuccess;
  const int64_t threads = nstreams * kWarp;
  k_remap_active<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(active, streams, sizes, nstreams,
                                                                                 remap);
  return cudaGetLastError();
}

cudaError_t launch_route_pack(int64_t n, int32_t world, const int32_t* owner, const uint32_t* records,
                              int32_t rec_words, uint32_t* out, int64_t* counts, int64_t* perm, void* scratch,
                              cudaStream_t st) {
  if (world > 8) return cudaErrorInvalidValue;
  const int64_t ntiles = (n + kRouteTile - 1) / kRouteTile;
  int64_t* tile_counts = static_cast<int64_t*>(scratch);  // world * ntiles
  if (n > 0) {
    k_route_count<<<static_cast<unsigned>(ntiles), 256, world * sizeof(int), st>>>(n, world, owner, tile_counts);
  }
  k_route_scan<<<1, 1, 0, st>>>(world * ntiles, world, ntiles, tile_counts, counts);
  if (n > 0) {
    k_route_scatter<<<static_cast<unsigned>(ntiles), kRouteTile, 0, st>>>(n, world, owner, records, rec_words,
                                                                            tile_counts, out, perm);
  }
  return cudaGetLastError();
}

cudaError_t launch_route_unpack(int64_t n, const uint32_t* in, int32_t rec_words, const int64_t* perm, uint32_t* out,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t t = n * rec_words;
  k_route_gather<<<static_cast<unsigned>((t + 255) / 256), 256, 0, st>>>(n, in, rec_words, perm, out);
  return cudaGetLastError();
}

}  // namespace dgds

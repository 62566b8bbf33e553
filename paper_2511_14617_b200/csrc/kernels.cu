#include <algorithm>
// kernels.cu — sm_100a kernels of the DGDS hot path.
//
//   K1 k_append        batched incremental insertion of appended tokens into the
//                      per-group counted suffix tries (GroupDraftIndex::append /
//                      insert_token / ensure_child, proj/src/cst.cpp:90-133).
//   K2 k_query<G,S>    batched longest-suffix match + top-k beam expansion
//                      (GroupDraftIndex::speculate, cst.cpp:153-228): one G-lane
//                      tile (sub-warp) per request, with
//   K3                 fused verification / accept length (Instance::decode_step,
//                      proj/src/engine.cpp:115-143); k_verify is the standalone form.
//   k_rebuild_*        arena growth + GC of dropped groups (cst.cpp:63-74 grows the
//                      reference's EdgeMap; here the whole slot table is re-placed).
//   k_route_*          owner bucketing for the multi-GPU all-to-all (dgds.cpp:10-14 routing).
//
// Nothing here is a dense contraction, so there is no tensor-core path: every
// kernel is bound by dependent 32-B sector accesses to HBM / L2.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>

#include "kernels.h"

namespace dgds {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kBlock = 256;
#ifndef DGDS_APPEND_OCC
#define DGDS_APPEND_OCC 4  // resident blocks per SM the register budget is sized for
#endif
#ifndef DGDS_K1_PDL_TRIGGER
#define DGDS_K1_PDL_TRIGGER 0  // measured flat on C2 (profiles/r1_pdl_trigger.txt)
#endif
#ifndef DGDS_K2B_OCC
// K2b (M = 2): resident blocks per SM (x kBlock / B). 2 gives K2b 128 registers and no stack;
// 3 (80 registers + 112 B of stack) and 4 spilled and were 5-13% slower, 1 starved it (25%)
#define DGDS_K2B_OCC 2
#endif
#ifndef DGDS_QUERY_OCC
#define DGDS_QUERY_OCC 4
#endif
constexpr int kQueryBlockDefault = 64;  // measured: 256 -> 64 took K2 0.106 -> 0.102 ms (C2)
constexpr int kAppendBlockDefault = 64;  // measured: 256 -> 64 took K1 0.194 -> 0.188 ms (C2)

__device__ __forceinline__ int lane_id() { return threadIdx.x & (kWarp - 1); }

// ---------------------------------------------------------------------------
// k_stage: every record's tokens from the batch buffer into the history arena
// (record order; replica blobs) and into its stream's extent, and the stream
// table row {extent, stored length after the batch, root}. It runs before K1,
// so K1's conversion walks (below) read every stream of the batch at its final
// length. A negative token (possible only on the device paths; the host path
// rejects it before planning) sets err bit 1, and K1 then inserts nothing.

__global__ void k_stage(DevTrie T, const AppendSeg* __restrict__ segs, int64_t nseg,
                        const AppendPiece* __restrict__ pieces, int64_t npieces, const int32_t* __restrict__ tokens,
                        const CopyPiece* __restrict__ grow, int64_t ngrow) {
  const int lane = lane_id();
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t s = gt; s < nseg; s += nth) {
    const AppendSeg g = segs[s];
    DGDS_CHECK(T, g.stream < T.stream_cap && g.sh_base + g.start + g.n <= T.shist_cap);
    T.sinfo[g.stream] = StreamInfo{g.sh_base, static_cast<uint32_t>(g.start + g.n), g.root};
  }
  int32_t any = 0;
  for (int64_t w = gt / kWarp; w < npieces; w += nth / kWarp) {
    const AppendPiece pc = pieces[w];
    DGDS_CHECK(T, pc.hist_off + pc.n <= T.hist_cap && pc.sh_off + pc.n <= T.shist_cap);
    for (uint32_t k = lane; k < pc.n; k += kWarp) {
      const int32_t v = tokens[pc.tok_off + k];
      any |= v;
      T.hist[pc.hist_off + k] = v;
      T.shist[pc.sh_off + k] = v;
    }
  }
  // moved stream extents: the stored tokens into the new extent (disjoint from the pieces above)
  for (int64_t w = gt / kWarp; w < ngrow; w += nth / kWarp) {
    const CopyPiece pc = grow[w];
    DGDS_CHECK(T, pc.src + pc.len <= T.shist_cap && pc.dst + pc.len <= T.shist_cap);
    int32_t v[4];  // <= 128 tokens: all loads in flight before the stores
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t k = lane + u * kWarp;
      v[u] = k < pc.len ? T.shist[pc.src + k] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t k = lane + u * kWarp;
      if (k < pc.len) T.shist[pc.dst + k] = v[u];
    }
    for (uint32_t k = lane + 4 * kWarp; k < pc.len; k += kWarp) T.shist[pc.dst + k] = T.shist[pc.src + k];
  }
  if (__any_sync(kFull, any < 0) && lane == 0) atomicOr(T.err, 2);
}

// ---------------------------------------------------------------------------
// K1: append (GroupDraftIndex::append / insert_token / ensure_child, cst.cpp:90-133)
//
// One warp per stream segment. Lane i owns the window of length i+1 ending at
// the current token (Stream::active[i], cst.hpp:115-118); its parent is lane
// i-1's window at the previous token. Per token, a lane ADDS one occurrence of
// its window only when the parent is a node (count >= 2) or the group root:
//   - absent  -> a new LEAF holding this occurrence; the window's continuation
//                (all longer windows on this diagonal) is implicit from here on;
//   - a leaf  -> it becomes a node (count 2); the leaf's own occurrence (the
//                DISPLACED occurrence) must now continue explicitly;
//   - a node  -> count + 1.
// A lane whose parent is implicit does nothing: its window has count 1 and is
// the stream's own continuation below a leaf. Counts are order-free sums and a
// leaf converts exactly once (the atomic that takes its counter from 0), so
// concurrent streams of one group reach exactly the reference's trie.
//
// Riders. A displaced occurrence usually continues with the same tokens as the
// occurrence that displaced it (responses of a group share long runs). The lane
// that converted the leaf therefore carries the displaced occurrence down its
// own diagonal as a RIDER: at each next token it compares the rider's next
// token (from the rider stream's extent, staged by k_stage) with its own; equal
// tokens mean the same window, counted twice in one atomic. The first mismatch,
// the rider stream's end, or the end of the segment hands the rider to K1b as an
// event. A second displaced occurrence while a rider is aboard is queued too.
//
// Node marks. A converted leaf gets occ_pos = kNodeMark, and a window created
// with two occurrences (a lane and its rider) is born marked, so a claim that
// returns a marked entry knows it is a node: its count is a fire-and-forget RED
// instead of a returning atomic on the token's critical path.
//
// Conversion walk (K1b, one thread per event): the event's occurrence (stream
// s, window ending at e) continues with the windows ending at e+1, e+2, ... on
// the same diagonal, which nobody counted (s's owner treated them as implicit).
// The walk adds them one by one from s's extent (final for this batch: k_stage
// ran first) until it creates a leaf, reaches the depth cap or the end of s,
// with the same rider scheme; other displaced occurrences go on a DFS stack. A
// walk that reaches the end of s leaves the node it holds in ov[s][depth-1];
// s's next segment takes it as that lane's state. K1b runs after K1 has
// finished, so no segment of this batch reads ov while a walk writes it.

constexpr uint32_t kNodeMark = 0xFFFFFFFFu;  // occ_pos of an entry known to be a node
constexpr int kEvChunk = 32;                 // K1 event-queue slots a warp takes per counter atomic

__device__ __forceinline__ void cas128(Slot* s, unsigned long long n0, unsigned long long n1, unsigned long long& o0,
                                       unsigned long long& o1) {
  // {key, occ}: empty (all zero) -> ours, else returns the occupant
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(o0), "=l"(o1)
      : "l"(0ull), "l"(0ull), "l"(n0), "l"(n1), "l"(s)
      : "memory");
}

// {h32, next_sibling} of a new entry in one 64-bit store
__device__ __forceinline__ void store_link(Slot* s, uint32_t h32, uint32_t next_sibling) {
  *reinterpret_cast<unsigned long long*>(&s->h32) =
      static_cast<unsigned long long>(h32) | (static_cast<unsigned long long>(next_sibling) << 32);
}

struct AddResult {
  uint32_t id;
  bool created;
  bool converted;     // a leaf became a node: its occurrence (d_stream, d_pos) is displaced
  uint32_t d_stream;
  uint32_t d_pos;
};

// Add inc (1 or 2) occurrences of window (parent, token) at depth `depth`, one of them ending at
// `pos` of `stream`. CAS-first over the probe sequence: slots fill in probe order and are never
// freed between rebuilds, so the CAS's old value settles the case: 0 = created (a leaf holding
// this occurrence, or a marked node when inc = 2); our key = present; another key = probe on.
__device__ __forceinline__ AddResult add_window(const DevTrie& T, uint32_t h32, uint32_t parent, int32_t token,
                                                uint32_t stream, uint32_t depth, uint32_t pos, uint32_t inc) {
  const unsigned long long key = pack_key(parent, token);
  const unsigned long long occ = pack_occ(stream, depth, inc == 2u ? kNodeMark : pos);
  const uint64_t cap = T.cap;
  uint64_t i = home_bucket(h32, cap / kBucket) * kBucket;
  AddResult r{0, false, false, 0, 0};
  for (uint64_t probes = 0;; ++probes) {
    if (probes > 65536) {  // defensive: probe runs are short below the rebuild load
      atomicOr(T.err, 8);
      return r;
    }
    unsigned long long o0, o1;
    DGDS_CHECK(T, i < cap && (parent <= cap || parent >= kMinRootId));
    cas128(T.slots + i, key, occ, o0, o1);
    if (o0 == 0ull) {
      r.id = static_cast<uint32_t>(i + 1);
      r.created = true;
      if (inc == 2u) atomicAdd(&T.slots[i].count, 1u);  // born a node: the second occurrence
      return r;
    }
    if (o0 == key) {
      r.id = static_cast<uint32_t>(i + 1);
      if (static_cast<uint32_t>(o1 >> 32) == kNodeMark) {
        atomicAdd(&T.slots[i].count, inc);  // a node: no conversion possible (RED)
      } else if (atomicAdd(&T.slots[i].count, inc) == 0u) {
        r.converted = true;
        r.d_stream = occ_stream(static_cast<uint32_t>(o1));
        r.d_pos = static_cast<uint32_t>(o1 >> 32);
        T.slots[i].occ_pos = kNodeMark;
      }
      return r;
    }
    if (++i == cap) i = 0;
  }
}

// A rider: a displaced occurrence travelling down a diagonal with the occurrence that holds it.
struct Rider {
  uint32_t stream, pos;  // its window ends at `pos` of `stream`
  uint32_t abs, end;     // shist offsets of that token and of the stream's end
};

__device__ __forceinline__ Rider make_rider(const DevTrie& T, uint32_t stream, uint32_t pos) {
  const StreamInfo si = T.sinfo[stream];
  return Rider{stream, pos, static_cast<uint32_t>(si.base + pos), static_cast<uint32_t>(si.base + si.len)};
}

__device__ void conversion_walk(const DevTrie& T, WalkEvent e, unsigned long long& inserted) {
  struct Frame {
    unsigned long long h;
    uint32_t id, depth, stream, pos;
  };
  // Pushes happen at the current depth (a rider leaving) or one deeper (a conversion with a
  // rider aboard), and a popped frame carries no rider, so the stack is non-decreasing in depth
  // with at most two frames per depth.
  Frame stk[2 * DGDS_MAX_DEPTH];
  int sp = 0;
  auto push = [&](const Frame& f) {
    if (sp < 2 * DGDS_MAX_DEPTH) stk[sp++] = f;
    else atomicOr(T.err, 4);  // cannot happen (see above)
  };
  Frame cur{e.h, e.id, e.depth, e.stream, e.pos};
  bool ron = false;
  Rider rd{};
  const uint32_t D = static_cast<uint32_t>(T.depth_cap);
  int guard = 0;
  for (;; ++guard) {
    if (guard > (1 << 16)) {  // defensive: a walk is bounded by its conversions
      atomicOr(T.err, 16);
      return;
    }
    DGDS_CHECK(T, cur.stream < T.stream_cap && cur.id >= 1 && cur.id <= T.cap && cur.depth >= 1 &&
                      cur.depth <= static_cast<uint32_t>(T.depth_cap));
    const StreamInfo si = T.sinfo[cur.stream];
    const uint32_t p = cur.pos + 1;
    DGDS_CHECK(T, si.base + si.len <= T.shist_cap && (!ron || (rd.stream < T.stream_cap && rd.end <= T.shist_cap)));
    if (p == si.len) T.ov[static_cast<uint64_t>(cur.stream) * kWarp + cur.depth - 1] = cur.id;
    if (ron && rd.abs + 1u >= rd.end) {  // the rider's stream ends at this window
      T.ov[static_cast<uint64_t>(rd.stream) * kWarp + cur.depth - 1] = cur.id;
      ron = false;
    }
    if (cur.depth < D && p < si.len) {
      const int32_t x = T.shist[si.base + p];
      uint32_t inc = 1;
      if (ron) {
        if (T.shist[rd.abs + 1u] == x) {
          inc = 2;
        } else {
          push(Frame{cur.h, cur.id, cur.depth, rd.stream, rd.pos});
          ron = false;
        }
      }
      const unsigned long long h2 = hash_step(cur.h, x);
      const uint32_t hh = hash32(h2);
      const AddResult r = add_window(T, hh, cur.id, x, cur.stream, cur.depth + 1, p, inc);
      if (r.created) {
        ++inserted;
        store_link(T.slots + (r.id - 1), hh, atomicExch(&T.slots[cur.id - 1].first_child, r.id));
      }
      if (!r.created || inc == 2u) {  // a node now: this occurrence (and its rider) continue
        if (inc == 2u) rd = Rider{rd.stream, rd.pos + 1, rd.abs + 1, rd.end};
        if (r.converted) {
          if (!ron) {
            rd = make_rider(T, r.d_stream, r.d_pos);
            ron = true;
          } else {
            push(Frame{h2, r.id, cur.depth + 1, r.d_stream, r.d_pos});
          }
        }
        cur = Frame{h2, r.id, cur.depth + 1, cur.stream, p};
        continue;
      }
    } else if (ron && cur.depth < D) {  // this stream ends here; the rider's continues
      push(Frame{cur.h, cur.id, cur.depth, rd.stream, rd.pos});
    }
    ron = false;
    if (sp == 0) break;
    cur = stk[--sp];
  }
  if (T.k1_stats) {
    atomicAdd(T.k1_stats + 5, static_cast<unsigned long long>(guard + 1));
    atomicMax(T.k1_stats + 6, static_cast<unsigned long long>(guard + 1));
    atomicAdd(T.k1_stats + 7, 1ull);
  }
}

__global__ void k_walks(DevTrie T) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL launch: K1 is complete
  const unsigned long long n = __ldcg(T.ev_count);
  unsigned long long inserted = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const WalkEvent e = T.ev[i];
    if (e.id) conversion_walk(T, e, inserted);  // id 0: an unused slot of a warp's chunk
  }
  const unsigned long long w = __reduce_add_sync(kFull, static_cast<unsigned>(inserted));
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
  if (lane_id() == 0 && w) atomicAdd(T.used + ((warp & (kUsedParts - 1)) * 8), w);
  // the last block to finish resets the event queue for the next batch
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(T.ev_count + 1, 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    T.ev_count[0] = 0;
    T.ev_count[1] = 0;
  }
}

template <int B>  // threads per block (one warp per segment; B only sets the block granularity)
__global__ void __launch_bounds__(B, DGDS_APPEND_OCC * (kBlock / B))
    k_append(DevTrie T, const AppendSeg* __restrict__ segs, int64_t nseg) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL launch: k_stage is complete
  if (__ldcg(T.err) & 2) return;  // k_stage found a negative token: the batch inserts nothing
  const int lane = lane_id();
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * blockDim.x / kWarp;
  const int D = T.depth_cap;
  unsigned long long inserted_total = 0;
  // Warp-collective event queueing for K1b. A warp takes queue slots in chunks of kEvChunk (one
  // atomic on the shared counter per chunk instead of one per event batch: that counter is a
  // single L2 address every warp of the launch hits); unused slots of a chunk are marked empty
  // (id 0). Slots used <= 2 x events + kEvChunk x warps (the host sizes the queue for it).
  unsigned long long ev_base = 0;
  int ev_fill = kEvChunk;  // warp-uniform; no chunk yet
  auto close_chunk = [&]() {
    if (ev_fill < kEvChunk && ev_fill + lane < kEvChunk) T.ev[ev_base + ev_fill + lane].id = 0u;
    ev_fill = kEvChunk;
  };
  auto queue = [&](bool ev, unsigned long long eh, uint32_t eid, uint32_t edepth, uint32_t es, uint32_t ep) {
    const unsigned m = __ballot_sync(kFull, ev);
    if (m) {
      const int c = __popc(m);
      if (ev_fill + c > kEvChunk) {
        close_chunk();
        unsigned long long at = 0;
        if (lane == 0) at = atomicAdd(T.ev_count, static_cast<unsigned long long>(kEvChunk));
        ev_base = __shfl_sync(kFull, at, 0);
        ev_fill = 0;
        DGDS_CHECK(T, ev_base + kEvChunk <= T.ev_cap);
      }
      if (lane == 0 && T.k1_stats) atomicAdd(T.k1_stats + 4, static_cast<unsigned long long>(c));
      if (ev) T.ev[ev_base + ev_fill + __popc(m & ((1u << lane) - 1u))] = WalkEvent{eh, eid, edepth, es, ep};
      ev_fill += c;
    }
  };

  unsigned long long t_start = 0;
  if (T.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  for (int64_t sg = warp; sg < nseg; sg += nwarps) {
    const AppendSeg g = segs[sg];
    const uint64_t len0 = g.start;
    const uint32_t stream = g.stream;
    DGDS_CHECK(T, stream < T.stream_cap && g.sh_base + g.start + g.n <= T.shist_cap);
    uint32_t* act_row = T.active + static_cast<uint64_t>(stream) * kWarp;
    uint32_t* ov_row = T.ov + static_cast<uint64_t>(stream) * kWarp;
    const int32_t* ext = T.shist + g.sh_base;
    const unsigned long long hr = root_hash(g.root);

    // hashes of the windows ending at the last stored token, from the stream's extent
    unsigned long long h = 0;
    {
      const int have = static_cast<int>(min(static_cast<uint64_t>(D), len0));
      const int32_t mine = lane < have ? ext[len0 - have + lane] : 0;
      for (int k = 0; k < have; ++k) {
        const int32_t t = __shfl_sync(kFull, mine, k);
        const unsigned long long up = __shfl_up_sync(kFull, h, 1);
        h = hash_step(lane == 0 ? hr : up, t);
      }
    }
    const bool stored_lane = lane < D && static_cast<uint64_t>(lane) < len0;
    uint32_t a = stored_lane ? act_row[lane] : 0u;
    {
      const uint32_t o = ov_row[lane];  // a conversion walk made this lane's window a node
      if (o) {
        ov_row[lane] = 0u;
        if (stored_lane) a = o;
      }
    }
    bool ron = false;  // this lane's window carries a rider
    Rider rd{};
    uint64_t len = len0;
    uint32_t link_slot = 0, link_prev = 0, link_h = 0;
    bool link_pending = false;
    for (uint32_t j0 = 0; j0 < g.n; j0 += kWarp) {
      const int chunk = static_cast<int>(min(static_cast<uint32_t>(kWarp), g.n - j0));
      const int32_t tv = lane < chunk ? ext[len0 + j0 + lane] : 0;  // coalesced
      for (int jj = 0; jj < chunk; ++jj) {
        const int32_t t = __shfl_sync(kFull, tv, jj);
        const int newsize = static_cast<int>(min(static_cast<uint64_t>(D), len + 1));
        const unsigned long long hup = __shfl_up_sync(kFull, h, 1);
        h = hash_step(lane == 0 ? hr : hup, t);
        const uint32_t pm = __shfl_up_sync(kFull, a, 1);
        bool pron = __shfl_up_sync(kFull, ron, 1);
        Rider prd;
        prd.stream = __shfl_up_sync(kFull, rd.stream, 1);
        prd.pos = __shfl_up_sync(kFull, rd.pos, 1);
        prd.abs = __shfl_up_sync(kFull, rd.abs, 1);
        prd.end = __shfl_up_sync(kFull, rd.end, 1);
        const uint32_t parent = lane == 0 ? g.root : pm;
        DGDS_CHECK(T, lane == 0 || pm <= T.cap);
        const bool act = lane < newsize && parent != 0u;
        pron = pron && act && lane > 0;
        // the parent's rider: same next token = same window (counted twice); otherwise, or at
        // the rider stream's end, it continues in K1b from the parent window
        uint32_t inc = 1;
        bool ev1 = false;
        if (pron) {
          if (prd.abs + 1u < prd.end && T.shist[prd.abs + 1u] == t) inc = 2;
          else ev1 = true;
        }
        queue(ev1, hup, pm, static_cast<uint32_t>(lane), prd.stream, prd.pos);
        uint32_t na = 0;
        bool nron = false, ev2 = false;
        AddResult r{0, false, false, 0, 0};
        if (act) {
          const uint32_t hh = hash32(h);
          r = add_window(T, hh, parent, t, stream, static_cast<uint32_t>(lane) + 1u, static_cast<uint32_t>(len), inc);
          if (T.k1_stats) {
            atomicAdd(T.k1_stats + 0, 1ull);
            if (r.created) atomicAdd(T.k1_stats + 1, 1ull);
            if (r.converted) atomicAdd(T.k1_stats + 2, 1ull);
            if (inc == 2u) atomicAdd(T.k1_stats + 3, 1ull);
          }
          if (link_pending) {  // {h32, next_sibling} of the entry created at the previous token
            store_link(T.slots + link_slot, link_h, link_prev);
            link_pending = false;
          }
          if (r.created) {
            ++inserted_total;
            if (!is_root_id(parent, T.cap)) {  // root child lists are never enumerated
              link_prev = atomicExch(&T.slots[parent - 1].first_child, r.id);
              link_slot = r.id - 1;
              link_h = hh;
              link_pending = true;
            } else {
              store_link(T.slots + (r.id - 1), hh, 0u);
            }
          }
          if (!r.created || inc == 2u) {
            na = r.id;  // a node
            if (inc == 2u) {
              nron = true;
              rd = Rider{prd.stream, prd.pos + 1, prd.abs + 1, prd.end};
            }
            if (r.converted) {
              if (!nron) {
                nron = true;
                rd = make_rider(T, r.d_stream, r.d_pos);
              } else {
                ev2 = true;
              }
            }
          }
        }
        queue(ev2, h, r.id, static_cast<uint32_t>(lane) + 1u, r.d_stream, r.d_pos);
        a = na;
        ron = nron && lane + 1 < D;  // at the depth cap a rider has no continuation
        ++len;
      }
    }
    queue(ron, h, a, static_cast<uint32_t>(lane) + 1u, rd.stream, rd.pos);  // riders left at the segment end
    if (link_pending) store_link(T.slots + link_slot, link_h, link_prev);
    if (lane < D && static_cast<uint64_t>(lane) < len) act_row[lane] = a;
  }
  close_chunk();
  if (T.dbg && lane == 0 && warp < 65536) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    T.dbg[2 * warp] = t_start;
    T.dbg[2 * warp + 1] = t_end;
  }
  // one RED per warp into a partition of the occupancy counter (no block barrier)
  const unsigned long long ins_warp = __reduce_add_sync(kFull, static_cast<unsigned>(inserted_total));
  if (lane == 0 && ins_warp) atomicAdd(T.used + ((warp & (kUsedParts - 1)) * 8), ins_warp);
}

// ---------------------------------------------------------------------------
// K2 + K3: draft query with fused verification.
//
// A warp serves 32/G requests, one G-lane tile each, and runs them in LOCK
// STEP: every loop bound is warp-uniform (the max over the warp's tiles) and
// per-tile work is predicated, so the dependent memory chains of all tiles
// issue together instead of serialising behind divergent branches.
//
// Phase A (longest admissible suffix, cst.cpp:160-178). The longest suffix is
// tried first: its (<= 8) prefixes are probed by content hash in one round
// (two probes in flight per lane), then the parent chain root -> ... -> suffix
// is checked from the probe records; a parent mismatch (hash collision) falls
// back to an exact (parent, token) probe. Only when it is absent are the
// shorter suffixes probed, in order; the first present one is the locus and
// there is no fallback after it.
//
// Phase B (beam, cst.cpp:180-221). Lane b owns beam path b (tokens in
// registers) and walks its child list; qualifying children are merged one at a
// time into a tile-distributed sorted pool of size top_k — lane r holds rank r
// under path_before: FP64 score desc (cnt / parent_cnt products, IEEE
// round-to-nearest, reference operation order), support desc, token path
// lexicographic asc. Equal-length paths compare as (parent path rank, token),
// so only ranks travel. Finals follow cst.cpp:213-214 (final only with no
// qualifying child) and are kept top-k under candidate_before (cst.cpp:29-33,
// 225-227) by the tile's lane 0 in shared memory.

template <int G, int S>
struct __align__(16) GroupScratch {
  union {
    struct {
      uint32_t wid[36];
      uint32_t wpar[36];
      uint32_t scnt[8];
      uint32_t sfc[8];
      int32_t pat[8];  // the last `start` pattern tokens (tok_at)
    } a;
    struct {
      double score[G];
      long long sup[G];
      int32_t len[G];
      int32_t tok[G][S];
    } f;
  };
};

// lexicographic compare of token arrays (std::vector<int>::operator<)
__device__ __forceinline__ bool tokens_less(const int32_t* a, int la, const int32_t* b, int lb) {
  const int m = la < lb ? la : lb;
  for (int i = 0; i < m; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return la < lb;
}

__device__ __forceinline__ bool cand_before(double sa, long long pa, const int32_t* ta, int la, double sb,
                                            long long pb, const int32_t* tb, int lb) {
  if (sa != sb) return sa > sb;
  if (pa != pb) return pa > pb;
  return tokens_less(ta, la, tb, lb);
}

template <int S>
__device__ __forceinline__ void set_tok(int32_t (&tok)[S], int d, int32_t v) {
#pragma unroll
  for (int i = 0; i < S; ++i)
    if (i == d) tok[i] = v;
}

// tile-width collectives over a full, convergent warp
template <int G>
struct Tile {
  int tbase;
  __device__ __forceinline__ unsigned ballot(bool p) const {
    const unsigned m = __ballot_sync(kFull, p);
    return G == 32 ? m : (m >> tbase) & ((1u << G) - 1u);
  }
  template <class T>
  __device__ __forceinline__ T shfl(T v, int src) const {
    return __shfl_sync(kFull, v, src, G);
  }
  template <class T>
  __device__ __forceinline__ T shfl_up(T v, int d) const {
    return __shfl_up_sync(kFull, v, d, G);
  }
  __device__ __forceinline__ int sum(int v) const {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o, G);
    return v;
  }
  __device__ __forceinline__ int max(int v) const {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = ::max(v, __shfl_xor_sync(kFull, v, o, G));
    return v;
  }
};

// Resolve a content probe (h32, token) whose first probe window (hb[]: the slots' h32) is
// already loaded. A match on (h32, token) is a candidate; the caller checks its parent.
__device__ __forceinline__ uint32_t resolve_content(const DevTrie& T, uint32_t h, int32_t token, uint64_t b,
                                                    const uint32_t (&hb)[kWindow], SlotView& rec) {
  const uint64_t cap = T.cap;
  const uint64_t nb = cap / kBucket;
  bool first = true;
  while (true) {
#pragma unroll
    for (int s = 0; s < kWindow; ++s) {
      const uint64_t i = window_slot(b, s, cap);
      const uint32_t hs = first ? hb[s] : hash_word(T.slots + i);
      if (hs == h) {
        rec = load_slot_nc(T.slots + i);  // same sector as the hash: an L1 hit
        if (rec.token == token) return static_cast<uint32_t>(i + 1);
      }
      if (hs == 0u) return 0;
    }
    first = false;
    b += kWindow / kBucket;
    if (b >= nb) b -= nb;
  }
}

// Implicit path state (a count-1 window below a leaf): bit 63 set, bits 32-62 = continuation
// tokens still available below it (depth cap, stream end), bits 0-31 = the shist offset of
// the window's last token. 0 = an entry path (children in the entry's child list).
__device__ __forceinline__ unsigned long long make_imp(uint64_t abs, uint32_t rem) {
  return (1ull << 63) | (static_cast<unsigned long long>(rem) << 32) | static_cast<uint32_t>(abs);
}
__device__ __forceinline__ uint32_t imp_rem(unsigned long long v) { return static_cast<uint32_t>(v >> 32) & 0x7FFFFFFFu; }
__device__ __forceinline__ uint32_t imp_abs(unsigned long long v) { return static_cast<uint32_t>(v); }
// the implicit continuation below leaf r (a window of `depth` tokens)
__device__ __forceinline__ StreamInfo load_sinfo(const DevTrie& T, uint32_t stream) {
  DGDS_CHECK(T, stream < T.stream_cap);
  unsigned long long a, b;
  asm("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(T.sinfo + stream));
  return StreamInfo{a, static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32)};
}
// A leaf child in the beam pool keeps its raw occurrence (bit 62) until it becomes a beam path:
// most leaf children do not qualify, and resolving one costs a stream-table load.
constexpr unsigned long long kImpRaw = 1ull << 62;
__device__ __forceinline__ unsigned long long raw_imp(const SlotView& r) {
  return (1ull << 63) | kImpRaw | (static_cast<unsigned long long>(occ_stream(r.occ_stream)) << 32) | r.occ_pos;
}
__device__ __forceinline__ unsigned long long resolve_imp(const DevTrie& T, unsigned long long v, int depth) {
  const uint32_t pos = static_cast<uint32_t>(v);
  const StreamInfo si = load_sinfo(T, static_cast<uint32_t>(v >> 32) & kStreamMask);
  const uint32_t rem = min(static_cast<uint32_t>(T.depth_cap - depth), si.len - 1u - pos);
  return make_imp(si.base + pos, rem);
}
__device__ __forceinline__ unsigned long long leaf_imp(const DevTrie& T, const SlotView& r, int depth) {
  const StreamInfo si = load_sinfo(T, occ_stream(r.occ_stream));
  const uint32_t rem = min(static_cast<uint32_t>(T.depth_cap - depth), si.len - 1u - r.occ_pos);
  return make_imp(si.base + r.occ_pos, rem);
}

// B = threads per block. A block retires only when its slowest warp does, so smaller blocks
// free a finished warp's SM slot sooner; the register budget per SM is the same for every B.
// K2 runs in one of three modes (template parameter M):
//   0  whole query per tile (phase A + phase B) — the fallback without a complex-query queue;
//   1  K2a: phase A for every query. A query whose locus is a count-1 window (a leaf or the
//      chain below one) has a determined answer — the single path of its stream's
//      continuation, score 1.0 (every step 1/1), support 1 — written here with its
//      verification; a query whose locus is a node is queued for K2b;
//   2  K2b: phase B for the queued queries only, so its warps hold only branching queries.
// Results, counters and verification are identical in every mode.

template <int G, int S, int B, int M>
__device__ __forceinline__ void query_tile(const QueryLaunch& P, GroupScratch<G, S>& sm, const int64_t q, bool valid,
                                           const CplxRec& cr, uint32_t (&sv)[12]) {
  const int lane = lane_id();
  const int gl = lane % G;
  const Tile<G> tile{lane - gl};
  if (P.seg_rows > 0 && valid) {  // routed segments: rows past the sender's count are padding
    const int64_t sg = q / P.seg_rows;
    valid = q - sg * P.seg_rows < P.seg_count[sg];
  }
  const int64_t qi = valid ? q : 0;
  const DevTrie& T = P.T;

  dgds_spec_args a = P.args[qi * P.args_stride];
  const int64_t qin = qi * P.in_qstride;  // per-query scalars: SoA (stride 1) or routed records
  const int32_t hdl = P.handles[qin];
  int plen = P.pat_len ? P.pat_len[qin] : 0;
  int row_valid = min(plen, P.pat_stride);  // pattern tokens present in the row (left-aligned)
  if (P.engine) {
    // Instance::decode_step's query rules (engine.cpp:88-99): spec_len = min(d, limit - 1),
    // pat_len = min(pattern_lookup_max, generated); no query when spec_len <= 0 or pat_len <
    // pattern_lookup_min (or drafting is off); top_k = max(1, multi_path_k). The row holds the
    // last min(generated, pat_stride) context tokens.
    const int g = P.gen[qin];
    const int d = P.draft_len_dev ? __ldcg(P.draft_len_dev) : P.draft_len;
    const int spec_len = min(d, P.limit[qin] - 1);
    const int pat_len = min(a.pattern_lookup_max, g);
    const bool skip = !(P.policy.sd_enabled && d > 0) || spec_len <= 0 || pat_len < a.pattern_lookup_min;
    a.max_spec_tokens = max(spec_len, 0);
    a.top_k = max(1, P.policy.multi_path_k);
    plen = skip ? 0 : pat_len;
    row_valid = min(g, P.pat_stride);
  }
  int32_t tleft = 0, lim = 0;
  const bool verify = P.v_emitted != nullptr || (P.rec_words_out > 0 && P.off_v >= 0);
  if (verify) {
    tleft = P.truth_left[qin];
    lim = P.limit[qin];
  }
  const uint32_t root = (valid && hdl >= 0 && hdl < P.n_handles) ? P.root_of[hdl] : 0u;
  const int eff_pmax = min(a.pattern_lookup_max, T.lim_pattern);  // cst.cpp:156-158
  const int eff_smax = min(a.max_spec_tokens, T.lim_spec);
  const int kq = a.top_k;
  const bool bad_args = a.pattern_lookup_min < 1 || a.pattern_lookup_min > a.pattern_lookup_max ||
                        a.max_spec_tokens < 0 || a.top_k < 1 || a.top_k > G || !(a.min_step_freq >= 0.0) ||
                        a.min_support < 0 || eff_smax > S;
  if (valid && bad_args && gl == 0 && P.err_flag) atomicOr(P.err_flag, 1);

  const int start = max(0, min(eff_pmax, plen));
  const int nlen = start - a.pattern_lookup_min + 1;
  const bool act = valid && !bad_args && root != 0u && plen > 0 && a.pattern_lookup_min <= eff_pmax && nlen > 0;
  const bool fast = start <= 8;
  const int row_len = row_valid;
  // row[0..start) = the last `start` pattern tokens; suffix j (length start-j) starts at row + j
  const int32_t* row = P.pat_end ? P.patterns + (P.pat_end[qi] - start)
                                 : P.patterns + qi * static_cast<int64_t>(P.pat_stride) + (row_len - start);
  int32_t pr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) pr[i] = (act && fast && i < start) ? row[i] : 0;
  if constexpr (M != 2) {
    for (int i = gl; i < 8; i += G) sm.a.pat[i] = (act && fast && i < start) ? row[i] : 0;
    __syncwarp();
  }
  auto tok_at = [&](int x) -> int32_t { return (act && !fast) ? row[x] : sm.a.pat[x]; };
  const unsigned long long h0 = root_hash(root);
  auto hash_prefix = [&](int j, int i) {  // content hash of row[j .. j+i)
    unsigned long long h = h0;
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (t < i) h = hash_step(h, tok_at(j + t));
    return hash32(h);
  };
  auto b0 = [&](int j) { return j * start - j * (j - 1) / 2; };  // first window of suffix j

  int st_lookups = 0, st_exp = 0, st_csec = 0;
  long long tA = P.dbg ? clock64() : 0;  // phase timing (debug only)
  int it_child = 0, it_merge = 0, it_depth = 0;
  int winner = -1;
  uint32_t locus_cnt = 0, locus_fc = 0;
  unsigned long long locus_imp = 0;  // nonzero: the locus is a count-1 window (implicit path)
  const uint64_t nbk = T.cap / kBucket;

  if constexpr (M == 2) {  // the locus was found by K2a
    winner = valid ? cr.winner : -1;
    locus_cnt = cr.cnt;
    locus_fc = cr.fc;
    st_lookups = valid ? cr.lookups : 0;
  } else {
  // ---------------- phase A ----------------
  // (1) the longest suffix: windows i = gl+1 and gl+1+G, both probes in flight.
  // Its windows are prefixes of row[0..start): hash them once with static indexing.
  unsigned long long hpre[9];
  hpre[0] = h0;
#pragma unroll
  for (int i = 1; i <= 8; ++i) hpre[i] = hash_step(hpre[i - 1], pr[i - 1]);
  {
    const int i1 = gl + 1, i2 = gl + 1 + G;
    const bool d1 = act && fast && i1 <= start;
    const bool d2 = act && fast && G < 8 && i2 <= start;
    unsigned long long h1 = 0, h2 = 0;
    int32_t t1 = 0, t2 = 0;
#pragma unroll
    for (int i = 1; i <= 8; ++i) {
      if (i == i1) {
        h1 = hpre[i];
        t1 = pr[i - 1];
      }
      if (i == i2) {
        h2 = hpre[i];
        t2 = pr[i - 1];
      }
    }
    const uint32_t k1 = hash32(h1), k2 = hash32(h2);
    const uint64_t bk1 = home_bucket(k1, nbk), bk2 = home_bucket(k2, nbk);
    uint32_t x[kWindow], y[kWindow];
#pragma unroll
    for (int s = 0; s < kWindow; ++s) {
      x[s] = d1 ? hash_word(T.slots + window_slot(bk1, s, T.cap)) : 0u;
      y[s] = d2 ? hash_word(T.slots + window_slot(bk2, s, T.cap)) : 0u;
    }
    if (d1) {
      SlotView r;
      const uint32_t id = resolve_content(T, k1, t1, bk1, x, r);
      sm.a.wid[i1 - 1] = id;
      sm.a.wpar[i1 - 1] = id ? r.parent : 0u;
      if (i1 == start) {
        sm.a.scnt[0] = id ? occurrences(r.count) : 0u;
        sm.a.sfc[0] = id ? r.first_child : 0u;
      }
    }
    if (d2) {
      SlotView r;
      const uint32_t id = resolve_content(T, k2, t2, bk2, y, r);
      sm.a.wid[i2 - 1] = id;
      sm.a.wpar[i2 - 1] = id ? r.parent : 0u;
      if (i2 == start) {
        sm.a.scnt[0] = id ? occurrences(r.count) : 0u;
        sm.a.sfc[0] = id ? r.first_child : 0u;
      }
    }
    __syncwarp();
  }
  // The window of L tokens ending in entry `last` (its own record r) is the locus: a node
  // keeps its child list; a leaf (one occurrence) continues implicitly in its stream.
  auto locus_of = [&](const SlotView& r, int L, uint32_t& cnt, uint32_t& fc, unsigned long long& imp) {
    cnt = occurrences(r.count);
    fc = r.first_child;
    imp = r.count == 0u ? leaf_imp(T, r, L) : 0ull;
  };
  // Suffix j from the probe records (exact fallback on a parent mismatch). Windows past the
  // deepest entry of the suffix are count-1 windows below a leaf: they exist iff the leaf's
  // occurrence continues with the suffix's remaining tokens (one lookup per window, as the
  // reference's walk counts them).
  auto check_suffix = [&](int j, int& looks, uint32_t& cnt, uint32_t& fc, unsigned long long& imp) -> bool {
    const int L = start - j;
    const int bj = b0(j);
    uint32_t prev = root;
    unsigned long long h = h0;
    for (int i = 1; i <= L; ++i) {
      ++looks;
      const int32_t tk = tok_at(j + i - 1);
      h = hash_step(h, tk);
      uint32_t id;
      SlotView r;
      if (fast && sm.a.wid[bj + i - 1] != 0u && sm.a.wpar[bj + i - 1] == prev) {
        id = sm.a.wid[bj + i - 1];
      } else if (fast && sm.a.wid[bj + i - 1] == 0u) {
        id = 0;  // no entry with this content at all
      } else {   // hash collision or long pattern: exact (parent, token) probe
        id = find_exact(T, hash32(h), prev, tk, r);
      }
      if (id == 0u) {
        if (i == 1) return false;
        const SlotView lr = load_slot_nc(T.slots + (prev - 1));
        if (lr.count != 0u) return false;  // a node: every child of a node is an entry
        const StreamInfo si = load_sinfo(T, occ_stream(lr.occ_stream));
        uint32_t e = lr.occ_pos;
        for (int m = i; m <= L; ++m) {
          if (m > i) ++looks;
          ++e;
          if (e >= si.len || __ldg(T.shist + si.base + e) != tok_at(j + m - 1)) return false;
        }
        cnt = 1;
        fc = 0;
        imp = make_imp(si.base + e, min(static_cast<uint32_t>(T.depth_cap - L), si.len - 1u - e));
        return true;
      }
      prev = id;
    }
    locus_of(load_slot_nc(T.slots + (prev - 1)), L, cnt, fc, imp);
    return true;
  };
  {
    int looks = 0;
    uint32_t cnt = 0, fc = 0;
    unsigned long long imp = 0;
    bool ok = false;
    if (act && gl == 0) {
      // fast check of the longest suffix from the probe records
      bool dead = false, slow = false;
      uint32_t prev = root;
#pragma unroll
      for (int i = 1; i <= 8; ++i) {
        if (fast && i <= start && !dead && !slow) {
          ++looks;
          const uint32_t id = sm.a.wid[i - 1];
          if (id == 0u) {
            if (i == 1) dead = true;
            else slow = true;  // maybe the implicit continuation of a leaf: checked below
          } else if (sm.a.wpar[i - 1] != prev) {
            slow = true;  // hash collision: exact walk below
          } else {
            prev = id;
          }
        }
      }
      if (fast && !slow) {
        ok = !dead;
        cnt = sm.a.scnt[0];
        fc = sm.a.sfc[0];
        if (ok && cnt == 1u) locus_of(load_slot_nc(T.slots + (prev - 1)), start, cnt, fc, imp);
      } else {
        looks = 0;
        ok = check_suffix(0, looks, cnt, fc, imp);
      }
    }
    st_lookups = tile.shfl(looks, 0);
    const bool ok0 = tile.shfl(static_cast<int>(ok), 0) != 0;
    const uint32_t c0 = tile.shfl(cnt, 0), f0 = tile.shfl(fc, 0);
    const unsigned long long i0 = tile.shfl(imp, 0);
    if (ok0) {
      winner = 0;
      locus_cnt = c0;
      locus_fc = f0;
      locus_imp = i0;
    }
  }
  // (2) only when the longest suffix is absent: the shorter ones, in order
  const bool need2 = act && winner < 0 && nlen > 1;
  if (__any_sync(kFull, need2)) {
    if (__any_sync(kFull, need2 && fast)) {
      const int W = need2 && fast ? b0(nlen) - b0(1) : 0;
      const int Wmax = tile.max(W);
      const int iters = __reduce_max_sync(kFull, (Wmax + G - 1) / G);
      for (int it = 0; it < iters; ++it) {
        const int w = b0(1) + gl + it * G;
        const bool dw = w < b0(1) + W;
        int j = 1, rem = w - b0(1);
        while (dw && rem >= start - j) {
          rem -= start - j;
          ++j;
        }
        const int i = rem + 1;
        uint32_t id = 0;
        SlotView r;
        if (dw) {
          const uint32_t h = hash_prefix(j, i);
          uint32_t hb[kWindow];
          const uint64_t bk = home_bucket(h, nbk);
#pragma unroll
          for (int s = 0; s < kWindow; ++s) hb[s] = hash_word(T.slots + window_slot(bk, s, T.cap));
          id = resolve_content(T, h, tok_at(j + i - 1), bk, hb, r);
          sm.a.wid[w] = id;
          sm.a.wpar[w] = id ? r.parent : 0u;
          if (i == start - j) {
            sm.a.scnt[j] = id ? occurrences(r.count) : 0u;
            sm.a.sfc[j] = id ? r.first_child : 0u;
          }
        }
      }
      __syncwarp();
    }
    // lanes check suffixes 1.., G at a time, in order
    const int rounds = __reduce_max_sync(kFull, need2 ? (nlen - 1 + G - 1) / G : 0);
    bool done = !need2;
    for (int u = 0; u < rounds; ++u) {
      const int j = 1 + u * G + gl;
      int looks = 0;
      uint32_t cnt = 0, fc = 0;
      unsigned long long imp = 0;
      const bool ok = !done && j < nlen && check_suffix(j, looks, cnt, fc, imp);
      const unsigned m = tile.ballot(ok);
      const int w = m ? __ffs(m) - 1 : G - 1;
      // collectives at one call site for every lane (tiles that are done add 0)
      const int add = tile.sum((!done && gl <= w) ? looks : 0);
      const uint32_t wc = tile.shfl(cnt, w);
      const uint32_t wf = tile.shfl(fc, w);
      const unsigned long long wi = tile.shfl(imp, w);
      if (!done) {
        st_lookups += add;
        if (m) {
          winner = 1 + u * G + w;
          locus_cnt = wc;
          locus_fc = wf;
          locus_imp = wi;
          done = true;
        }
      }
    }
  }
  }  // M != 2
  __syncwarp();  // phase-A scratch is dead from here (reused for finals)

  long long tB = P.dbg ? clock64() : 0;
  // ---------------- phase B ----------------
  int nf = 0;  // finals kept (tile-uniform)
  int32_t tok[S];
#pragma unroll
  for (int i = 0; i < S; ++i) tok[i] = 0;
  int nb = winner >= 0 ? 1 : 0;
  if constexpr (M == 1) {
    const bool cplx = valid && act && winner >= 0 && locus_imp == 0ull;  // the locus is a node: K2b
    const unsigned cm = __ballot_sync(kFull, cplx && gl == 0);
    if (cm) {
      unsigned long long at = 0;
      if (lane == __ffs(cm) - 1) at = atomicAdd(P.cplx_count, static_cast<unsigned long long>(__popc(cm)));
      at = __shfl_sync(kFull, at, __ffs(cm) - 1);
      if (cplx && gl == 0)
        P.cplx[at + __popc(cm & ((1u << lane) - 1u))] = CplxRec{q, locus_fc, locus_cnt, winner, st_lookups};
    }
    if (cplx) valid = false;  // answered (and counted) by K2b
    // a count-1 locus: one path along its occurrence's continuation (cst.cpp:196-215 with one
    // child per step, step = 1/1), expanded min(rem + 1, eff_smax) times; it qualifies unless the
    // query's min_step_freq > 1 or min_support > 1
    const bool imp = valid && winner >= 0 && locus_imp != 0ull;
    const int rem = imp ? static_cast<int>(imp_rem(locus_imp)) : 0;
    const bool qual = !(1.0 < a.min_step_freq) && !(1ll < a.min_support);
    const int k = (imp && qual && eff_smax > 0) ? min(rem, eff_smax) : 0;
    if (imp && eff_smax > 0) {
      st_exp = qual ? min(rem + 1, eff_smax) : 1;
      st_csec = qual ? k : (rem > 0 ? 1 : 0);
    }
    if (gl < k) sm.f.tok[0][gl] = __ldg(T.shist + imp_abs(locus_imp) + 1u + gl);
    for (int i = gl + G; i < k; i += G) sm.f.tok[0][i] = __ldg(T.shist + imp_abs(locus_imp) + 1u + i);
    if (k > 0 && gl == 0) {
      sm.f.len[0] = k;
      sm.f.score[0] = 1.0;
      sm.f.sup[0] = 1;
    }
    nf = k > 0 ? 1 : 0;  // written directly (a count-1 locus)
    nb = 0;
  }
  uint32_t b_fc = locus_fc;
  unsigned long long b_imp = locus_imp;  // nonzero: an implicit path (one continuation token in shist)
  const int locus_len = start - winner;  // depth of the locus (tile-uniform when nb > 0)
  double b_score = 1.0;
  long long b_sup = static_cast<long long>(locus_cnt);
  int b_lex = 0;
  int dl = 0;  // depth reached (tokens per beam path)
  const double msf = a.min_step_freq;
  const long long msup = a.min_support;

  // offer beam path b (dl tokens) of each tile with want=true to its finals
  auto finals_offer = [&](bool want, int b) {
    int32_t ct[S];
#pragma unroll
    for (int i = 0; i < S; ++i) ct[i] = tile.shfl(tok[i], b);
    const double cs = tile.shfl(b_score, b);
    const long long cp = tile.shfl(b_sup, b);
    if (want && gl == 0) {
      const int len = dl;
      int dst = -1;
      if (nf < kq) {
        dst = nf++;
      } else {
        int w = 0;  // worst kept final
        for (int c = 1; c < nf; ++c)
          if (cand_before(sm.f.score[w], sm.f.sup[w], sm.f.tok[w], sm.f.len[w], sm.f.score[c], sm.f.sup[c],
                          sm.f.tok[c], sm.f.len[c]))
            w = c;
        bool better;
        if (cs != sm.f.score[w]) {
          better = cs > sm.f.score[w];
        } else if (cp != sm.f.sup[w]) {
          better = cp > sm.f.sup[w];
        } else {
          int r = 0;  // lexicographic compare of ct[0..len) with the kept final
          const int m = len < sm.f.len[w] ? len : sm.f.len[w];
#pragma unroll
          for (int i = 0; i < S; ++i)
            if (r == 0 && i < m && ct[i] != sm.f.tok[w][i]) r = ct[i] < sm.f.tok[w][i] ? -1 : 1;
          better = r < 0 || (r == 0 && len < sm.f.len[w]);
        }
        if (better) dst = w;
      }
      if (dst >= 0) {
#pragma unroll
        for (int i = 0; i < S; ++i)
          if (i < len) sm.f.tok[dst][i] = ct[i];
        sm.f.len[dst] = len;
        sm.f.score[dst] = cs;
        sm.f.sup[dst] = cp;
      }
    }
    nf = tile.shfl(nf, 0);
  };

  for (int d = 0; __any_sync(kFull, nb > 0 && d < eff_smax); ++d) {
    const bool live = nb > 0 && d < eff_smax;  // tile-uniform
    // pool entry held by lane r (rank r), r < np
    double p_score = 0.0;
    long long p_sup = 0;
    int p_lex = 0, p_src = 0;
    int32_t p_tok = 0;
    uint32_t p_fc = 0;
    unsigned long long p_imp = 0;
    int np = 0;
    // an entry path enumerates its child list; an implicit path has at most one child, the
    // next token of its occurrence (count 1)
    uint32_t c = (live && gl < nb && b_imp == 0ull) ? b_fc : 0u;
    bool impc = live && gl < nb && b_imp != 0ull && imp_rem(b_imp) > 0u;
    const int child_depth = locus_len + d + 1;
    bool grew = false;
    int nchild = 0;
    ++it_depth;
    while (__any_sync(kFull, c != 0u || impc)) {
      ++it_child;
      SlotView r{};
      const bool have = c != 0u || impc;
      unsigned long long cimp = 0;
      if (c != 0u) {
        DGDS_CHECK(T, c <= T.cap);
        r = load_slot_nc(T.slots + (c - 1));
        if (r.count == 0u) cimp = raw_imp(r);  // a leaf: implicit below it (resolved if it is kept)
      } else if (impc) {
        const uint32_t at = imp_abs(b_imp) + 1u;
        DGDS_CHECK(T, at < T.shist_cap);
        r.token = __ldg(T.shist + at);
        r.count = 0u;
        r.first_child = 0u;
        r.next_sibling = 0u;
        cimp = make_imp(at, imp_rem(b_imp) - 1u);
      }
      bool qual = false;
      double sc = 0.0;
      const long long cnt = have ? static_cast<long long>(occurrences(r.count)) : 0ll;
      if (have) {
        ++nchild;
        const double step = __ddiv_rn(static_cast<double>(cnt), static_cast<double>(b_sup));
        qual = !(step < msf) && !(cnt < msup);
        if (qual) {
          grew = true;
          sc = __dmul_rn(b_score, step);
          if (r.first_child) prefetch_l1(T.slots + (r.first_child - 1));  // the next level's first load
        }
      }
      unsigned m = tile.ballot(qual);
      while (__any_sync(kFull, m != 0u)) {  // merge one candidate per tile into its sorted pool
        ++it_merge;
        const bool has = m != 0u;
        const int b = has ? __ffs(m) - 1 : 0;
        if (has) m &= m - 1;
        const double cs = tile.shfl(sc, b);
        const long long cp = tile.shfl(cnt, b);
        const int cl = tile.shfl(b_lex, b);
        const int32_t ct = tile.shfl(r.token, b);
        const uint32_t cfc = tile.shfl(r.first_child, b);
        const unsigned long long cim = tile.shfl(cimp, b);
        const bool before = has && gl < np &&
                            (p_score != cs ? p_score > cs
                             : p_sup != cp ? p_sup > cp
                             : p_lex != cl ? p_lex < cl
                                           : p_tok < ct);
        const int pos = __popc(tile.ballot(before));
        const bool ins = has && pos < kq;
        const double us = tile.shfl_up(p_score, 1);
        const long long up = tile.shfl_up(p_sup, 1);
        const int ul = tile.shfl_up(p_lex, 1);
        const int usrc = tile.shfl_up(p_src, 1);
        const int32_t ut = tile.shfl_up(p_tok, 1);
        const uint32_t ufc = tile.shfl_up(p_fc, 1);
        const unsigned long long uim = tile.shfl_up(p_imp, 1);
        if (ins && gl > pos && gl <= np) {
          p_score = us;
          p_sup = up;
          p_lex = ul;
          p_src = usrc;
          p_tok = ut;
          p_fc = ufc;
          p_imp = uim;
        }
        if (ins && gl == pos) {
          p_score = cs;
          p_sup = cp;
          p_lex = cl;
          p_src = b;
          p_tok = ct;
          p_fc = cfc;
          p_imp = cim;
        }
        if (ins) np = min(np + 1, kq);
      }
      c = c != 0u ? r.next_sibling : 0u;
      impc = false;
    }
    if (live) {
      st_exp += nb;
    }
    st_csec += tile.sum((live && gl < nb) ? (8 * nchild + 31) / 32 : 0);
    // paths without a qualifying child are final (when non-empty, i.e. d > 0)
    unsigned fm = tile.ballot(live && gl < nb && !grew && d > 0);
    while (__any_sync(kFull, fm != 0u)) {
      const bool has = fm != 0u;
      const int b = has ? __ffs(fm) - 1 : 0;
      if (has) fm &= fm - 1;
      finals_offer(has, b);
    }
    // the pool becomes the next beam: lane r takes pool rank r
    int32_t nt[S];
#pragma unroll
    for (int i = 0; i < S; ++i) nt[i] = tile.shfl(tok[i], p_src);
    int lex = 0;
    const int npmax = __reduce_max_sync(kFull, live ? np : 0);  // warp-uniform bound
    for (int o = 0; o < npmax; ++o) {
      const int ol = tile.shfl(p_lex, o);
      const int32_t ot = tile.shfl(p_tok, o);
      lex += (o < np && (ol < p_lex || (ol == p_lex && ot < p_tok))) ? 1 : 0;
    }
    if (live) {
#pragma unroll
      for (int i = 0; i < S; ++i) tok[i] = nt[i];
      set_tok<S>(tok, d, p_tok);
      b_fc = p_fc;
      b_imp = (p_imp & kImpRaw) && gl < np ? resolve_imp(T, p_imp, child_depth) : p_imp;
      b_score = p_score;
      b_sup = p_sup;
      b_lex = lex;
      nb = np;
      if (np > 0) dl = d + 1;
    }
  }
  // leftover beam paths (dl tokens each) are finals when non-empty (cst.cpp:222-223)
  {
    const int rounds = __reduce_max_sync(kFull, dl > 0 ? nb : 0);
    for (int b = 0; b < rounds; ++b) finals_offer(dl > 0 && b < nb, b);
  }

  long long tC = P.dbg ? clock64() : 0;
  // ---- output in candidate_before order ----
  __syncwarp();
  int my_rank = 0;
  if (gl < nf) {
    for (int c = 0; c < nf; ++c)
      my_rank += cand_before(sm.f.score[c], sm.f.sup[c], sm.f.tok[c], sm.f.len[c], sm.f.score[gl], sm.f.sup[gl],
                             sm.f.tok[gl], sm.f.len[gl])
                     ? 1
                     : 0;
  }
  // per-query output pointers: SoA buffers or one reply record (local or in peer memory)
  int32_t *o_nc = nullptr, *o_len = nullptr, *o_tk = nullptr, *o_v = nullptr;
  double* o_sc = nullptr;
  int64_t* o_sp = nullptr;
  if (P.rec_words_out > 0) {
    int32_t* R;
    if (P.seg_rows > 0) {
      const int64_t sg = q / P.seg_rows;
      const int64_t row = P.seg_origin ? static_cast<int64_t>(P.seg_origin[q * P.in_qstride]) : q - sg * P.seg_rows;
      R = P.seg_out[sg] + row * P.rec_words_out;
    } else {
      R = P.rec_out + (P.out_off ? P.out_off[q] : q * P.rec_words_out);
    }
    if (P.off_nc >= 0) {
      o_nc = R + P.off_nc;
      o_len = R + P.off_len;
      o_sc = reinterpret_cast<double*>(R + P.off_sc);
      o_sp = reinterpret_cast<int64_t*>(R + P.off_sp);
      o_tk = R + P.off_tk;
    }
    if (P.off_v >= 0) o_v = R + P.off_v;
  } else {
    if (P.n_cands) {
      o_nc = P.n_cands + q * P.nc_qstride;
      o_len = P.lens + q * P.out_qstride;
      o_sc = P.scores + q * P.out_qstride8;
      o_sp = P.supports + q * P.out_qstride8;
      o_tk = P.tokens + q * P.tok_qstride;
    }
  }
  if (o_nc && valid) {
    if (gl == 0) *o_nc = nf;
    if (gl < nf) {
      o_len[my_rank] = sm.f.len[gl];
      o_sc[my_rank] = sm.f.score[gl];
      o_sp[my_rank] = sm.f.sup[gl];
      int32_t* dst = o_tk + static_cast<int64_t>(my_rank) * P.s_stride;
      for (int i = 0; i < sm.f.len[gl]; ++i) dst[i] = sm.f.tok[gl][i];
    }
  }

  // ---- K3: verification (engine.cpp:115-143) ----
  if (verify) {
    int drafted = 0, match = 0;
    if (gl < nf) {
      drafted = sm.f.len[gl];
      const int32_t* tr = P.truth + qi * static_cast<int64_t>(P.truth_stride);
      const int cap = min(sm.f.len[gl], tleft);
      int32_t trv[S];
#pragma unroll
      for (int i = 0; i < S; ++i) trv[i] = i < cap ? tr[i] : 0;  // independent loads
      bool run = true;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        run = run && i < cap && sm.f.tok[gl][i] == trv[i];
        match += run ? 1 : 0;
      }
    }
    drafted = tile.sum(drafted);
    match = tile.max(match);
    if (valid && gl == 0) {
      const int emitted = min(match + 1, lim);
      if (P.engine) {  // the step's totals and the requests still running after it
        sv[8] += lim - emitted > 0 ? 1u : 0u;
        sv[9] += static_cast<uint32_t>(drafted);
        sv[10] += static_cast<uint32_t>(emitted - 1);
        sv[11] += static_cast<uint32_t>(emitted);
      }
      if (P.rec_words_out > 0) {
        o_v[0] = drafted;
        o_v[1] = emitted - 1;
        o_v[2] = emitted;
      } else {
        P.v_drafted[q * P.v_qstride] = drafted;
        P.v_accepted[q * P.v_qstride] = emitted - 1;
        P.v_emitted[q * P.v_qstride] = emitted;
      }
    }
  }

  if (P.dbg && valid && gl == 0) {
    long long* o = P.dbg + q * 8;
    o[0] = tB - tA;
    o[1] = tC - tB;
    o[2] = clock64() - tC;
    o[3] = it_depth;
    o[4] = it_child;
    o[5] = it_merge;
    o[6] = winner;
    o[7] = nf;
  }
  if (P.stats) {
    const int ctoks = tile.sum(gl < nf ? sm.f.len[gl] : 0);
    const bool lead = valid && gl == 0;
    if (lead) {
      sv[0] += 1u;
      sv[1] += static_cast<uint32_t>(plen);
      sv[2] += static_cast<uint32_t>(st_lookups);
      sv[3] += static_cast<uint32_t>(st_exp);
      sv[4] += static_cast<uint32_t>(st_csec);
      sv[5] += static_cast<uint32_t>(nf);
      sv[6] += static_cast<uint32_t>(ctoks);
      sv[7] += static_cast<uint32_t>(4ull * plen + 32ull + 32ull * st_lookups + 32ull * st_exp + 32ull * st_csec +
                                     4ull * ctoks + 16ull * nf);
    }
  }
}

// K2b holds only branching queries and loops over them: 3 blocks of 256 per SM (85 registers)
// instead of 4 (64), which removes its spills.
template <int G, int S, int B, int M>
__global__ void __launch_bounds__(B, (M == 2 ? DGDS_K2B_OCC : DGDS_QUERY_OCC) * (kBlock / B)) k_query(QueryLaunch P) {
  // Programmatic dependent launch: the blocks may be resident before the previous kernel in
  // the stream (K1, or K2a for K2b) has finished; nothing is read until it has.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int kTiles = B / G;
  __shared__ GroupScratch<G, S> scratch[kTiles];
  const int lane = lane_id();
  const int gib = threadIdx.x / G;
  uint32_t sv[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  if constexpr (M != 2) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * kTiles + gib;
    query_tile<G, S, B, M>(P, scratch[gib], q, q < P.n, CplxRec{}, sv);  // invalid tiles stay, idle
  } else {
    const unsigned long long cnt = __ldcg(P.cplx_count);
    const int64_t tiles = static_cast<int64_t>(gridDim.x) * kTiles;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * kTiles + gib;
         __any_sync(kFull, r < static_cast<int64_t>(cnt)); r += tiles) {
      const bool has = r < static_cast<int64_t>(cnt);
      const CplxRec cr = has ? P.cplx[r] : CplxRec{0, 0, 0, -1, 0};
      query_tile<G, S, B, M>(P, scratch[gib], has ? cr.q : 0, has, cr, sv);
      __syncwarp();
    }
  }
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (B / kWarp);
  if (P.stats || P.engine) {
    // tile leaders' counters -> warp sums (redux) -> one RED per counter per warp into one of
    // kStatParts partitions: no same-address storm
#pragma unroll
    for (int k = 0; k < 12; ++k) sv[k] = __reduce_add_sync(kFull, sv[k]);
    if (lane == 0) {
      const uint32_t part = (blockIdx.x * (B / kWarp) + threadIdx.x / kWarp) & (kStatParts - 1);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (P.stats && sv[k]) atomicAdd(P.stat_part + part * 8 + k, static_cast<unsigned long long>(sv[k]));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (P.engine && sv[8 + k]) atomicAdd(P.step_acc + k, static_cast<unsigned long long>(sv[8 + k]));
    }
    // The last warp to finish folds the partitions into P.stats and settles the engine step (no
    // separate launch, and no block barrier holding finished warps' SM slots): the fence orders
    // this warp's atomics before its ticket. K2a leaves its counters for K2b's fold.
    bool last = false;
    if (M != 1 && lane == 0) {
      __threadfence();
      unsigned long long* ticket = P.stat_part + kStatParts * 8;
      last = atomicAdd(ticket, 1ull) == static_cast<unsigned long long>(nwarps) - 1;
    }
    if (__shfl_sync(kFull, last, 0)) {
      __threadfence();
      if (P.stats && lane < 8) {
        unsigned long long t = 0;
        for (int p = 0; p < kStatParts; ++p) t += atomicExch(P.stat_part + p * 8 + lane, 0ull);
        reinterpret_cast<unsigned long long*>(P.stats)[lane] += t;
      }
      if (P.engine && lane == 0) {
        unsigned long long tot[4];
        for (int k = 0; k < 4; ++k) tot[k] = atomicExch(P.step_acc + k, 0ull);
        // next step's draft length (engine.cpp:78-85) over the requests still running
        const long long n_next = static_cast<long long>(tot[0]);
        int d = 0;
        if (P.policy.sd_enabled && n_next > 0)
          d = P.policy.adaptive ? static_cast<int>(min(static_cast<long long>(P.policy.per_request_cap),
                                                       P.policy.batch_token_budget / n_next))
                                : P.policy.per_request_cap;
        d = max(d, 0);
        if (P.policy.feedback == 1 && P.n > 0) {  // extension: acceptance-scaled (not in the reference)
          const long long mean_acc = (static_cast<long long>(tot[2]) + P.n - 1) / P.n;
          d = static_cast<int>(min(static_cast<long long>(d), mean_acc + 1));
        }
        if (P.next_draft_len) *P.next_draft_len = d;
        if (P.step_totals)
          for (int k = 0; k < 4; ++k) P.step_totals[k] = static_cast<long long>(tot[k]);
      }
      if (lane == 0) P.stat_part[kStatParts * 8] = 0ull;
    }
  }
  if constexpr (M == 2) {  // the last warp resets the queue for the next batch
    if (lane == 0 && atomicAdd(P.cplx_count + 1, 1ull) == static_cast<unsigned long long>(nwarps) - 1) {
      P.cplx_count[0] = 0;
      P.cplx_count[1] = 0;
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

// GDX1 blob serialisation: warp per piece; byte stores (blob fields are not 4-B aligned).
__device__ __forceinline__ void put_be(uint8_t* p, uint64_t v, int bytes) {
  for (int b = 0; b < bytes; ++b) p[b] = static_cast<uint8_t>(v >> (8 * (bytes - 1 - b)));
}

__global__ void k_blob_fill(const BlobPiece* __restrict__ pieces, int64_t n, const int32_t* __restrict__ hist,
                            uint8_t* out) {
  const int lane = lane_id();
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x / kWarp);
  for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp; w < n; w += nw) {
    const BlobPiece pc = pieces[w];
    uint8_t* dst = out + pc.dst;
    if (lane == 0 && pc.hdr_kind == 1) {  // delta record: u32 rid, u64 start, u32 len
      put_be(dst - 16, pc.rid, 4);
      put_be(dst - 12, pc.hdr_a, 8);
      put_be(dst - 4, pc.len, 4);
    } else if (lane == 0 && pc.hdr_kind == 2) {  // full-snapshot stream: u32 rid, u64 len
      put_be(dst - 12, pc.rid, 4);
      put_be(dst - 8, pc.hdr_a, 8);
    }
    for (uint32_t i = lane; i < pc.len; i += kWarp) {
      const uint32_t v = static_cast<uint32_t>(hist[pc.src + i]);
      uint8_t* q = dst + 4ull * i;
      q[0] = static_cast<uint8_t>(v >> 24);
      q[1] = static_cast<uint8_t>(v >> 16);
      q[2] = static_cast<uint8_t>(v >> 8);
      q[3] = static_cast<uint8_t>(v);
    }
  }
}

__global__ void k_set_u32(uint32_t* dst, uint32_t v) { *dst = v; }

// ---------------------------------------------------------------------------
// rebuild. Pass 1 re-places every live slot of `from` at its home in `to`
// (keys are unique, so claiming an empty slot suffices) and records
// old id -> new id. Pass 2 rewrites parents through the map and relinks the
// child lists. Slots of dropped groups (root not alive) are not carried over.

__global__ void k_rebuild_place(DevTrie from, DevTrie to, const uint32_t* __restrict__ root_alive, uint32_t* remap) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < from.cap; i += stride) {
    const Slot s = from.slots[i];
    remap[i] = 0;
    if (s.parent == 0u) continue;
    const uint32_t ridx = kRootTop - from.sinfo[occ_stream(s.occ_stream)].root;  // the entry's group
    if (!((root_alive[ridx >> 5] >> (ridx & 31)) & 1u)) continue;
    const uint64_t nbk = to.cap / kBucket;
    const unsigned long long key = pack_key(s.parent, s.token);  // keys are unique: any empty slot will do
    uint64_t j = home_bucket(s.h32, nbk) * kBucket;
    while (atomicCAS(reinterpret_cast<unsigned long long*>(to.slots + j), 0ull, key) != 0ull)
      if (++j == to.cap) j = 0;
    Slot* d = to.slots + j;
    d->occ_stream = s.occ_stream;  // parent: old id until pass 2
    d->occ_pos = s.occ_pos;
    d->count = s.count;
    d->h32 = s.h32;
    remap[i] = static_cast<uint32_t>(j + 1);
    atomicAdd(to.used + ((i & (kUsedParts - 1)) * 8), 1ull);
  }
}

__global__ void k_rebuild_link(DevTrie to, const uint32_t* __restrict__ remap) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < to.cap; j += stride) {
    Slot* d = to.slots + j;
    const uint32_t op = d->parent;
    if (op == 0u || op >= kMinRootId) continue;  // empty, or depth 1 (parent = group root)
    const uint32_t np = remap[op - 1];
    d->parent = np;
    d->next_sibling = atomicExch(&to.slots[np - 1].first_child, static_cast<uint32_t>(j + 1));
  }
}

// active / ov rows through the old -> new id map (ids of dropped groups map to 0)
__global__ void k_remap_active(uint32_t* active, uint32_t* ov, const uint32_t* __restrict__ streams, int64_t ns,
                               const uint32_t* __restrict__ remap, uint64_t from_cap) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t s = t / kWarp;
  const int l = static_cast<int>(t % kWarp);
  if (s >= ns) return;
  const uint64_t at = static_cast<uint64_t>(streams[s]) * kWarp + l;
  const uint32_t v = active[at], o = ov[at];
  active[at] = (v && v <= from_cap) ? remap[v - 1] : 0u;
  ov[at] = (o && o <= from_cap) ? remap[o - 1] : 0u;
}

// logical trie nodes: every entry, plus the count-1 chain below each leaf
__global__ void k_node_count(DevTrie T, unsigned long long* out) {
  unsigned long long n = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < T.cap; i += stride) {
    const Slot s = T.slots[i];
    if (s.parent == 0u) continue;
    n += 1;
    if (s.count == 0u) {
      const StreamInfo si = T.sinfo[occ_stream(s.occ_stream)];
      n += min(static_cast<uint32_t>(T.depth_cap) - occ_depth(s.occ_stream), si.len - 1u - s.occ_pos);
    }
  }
  n = __reduce_add_sync(kFull, static_cast<unsigned>(n));  // < 2^32 per warp
  if (lane_id() == 0 && n) atomicAdd(out, n);
}

// ---------------------------------------------------------------------------
// routing: stable bucketing of fixed-size records by owner rank

constexpr int kRouteTile = 1024;

__global__ void k_route_count(int64_t n, int32_t world, const int32_t* __restrict__ owner, int64_t* tile_counts) {
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

__global__ void k_route_scan(int32_t world, int64_t ntiles, int64_t* tile_counts, int64_t* counts) {
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
}

__global__ void k_route_scatter(int64_t n, int32_t world, const int32_t* __restrict__ owner,
                                const uint32_t* __restrict__ rec, int32_t rw, const int64_t* __restrict__ tile_off,
                                uint32_t* out, int64_t* perm) {
  __shared__ int warp_cnt[kRouteTile / kWarp][8];
  const int64_t ntiles = gridDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kRouteTile;
  const int warp = threadIdx.x / kWarp, lane = lane_id();
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

// padded mode: exclusive scan of tile counts restarted for every owner (position inside its bucket)
__global__ void k_route_scan_local(int32_t world, int64_t ntiles, int64_t* tile_counts) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int o = 0; o < world; ++o) {
    int64_t run = 0;
    for (int64_t t = 0; t < ntiles; ++t) {
      const int64_t v = tile_counts[o * ntiles + t];
      tile_counts[o * ntiles + t] = run;
      run += v;
    }
  }
}

__global__ void k_route_scatter_padded(int64_t n, int32_t world, const int32_t* __restrict__ owner,
                                       const uint32_t* __restrict__ rec, int32_t rw, int64_t cap,
                                       const int64_t* __restrict__ tile_off, uint32_t* out, int64_t* slot,
                                       int32_t* overflow) {
  __shared__ int warp_cnt[kRouteTile / kWarp][8];
  const int64_t ntiles = gridDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kRouteTile;
  const int warp = threadIdx.x / kWarp, lane = lane_id();
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
    if (pos >= cap) {
      atomicExch(overflow, 1);
      pos = cap - 1;  // results are invalid; the flag says so
    }
    const int64_t row = o * cap + pos;
    for (int k = 0; k < rw; ++k) out[row * rw + k] = rec[i * rw + k];
    slot[i] = row;
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

template <int G, int S, int B, int M>
cudaError_t launch_query_gsbm(const QueryLaunch& L, cudaStream_t st, int64_t blocks) {
  // launched with programmatic stream serialization: the launch overlaps the previous
  // kernel's tail (k_query waits for its completion in griddepcontrol.wait)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(B);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaLaunchKernelEx(&cfg, k_query<G, S, B, M>, L);
}

// K2b's grid: the blocks that fit the GPU at once (it loops over its queue)
template <int G, int S, int B>
int64_t resident_blocks() {
  static const int64_t n = [] {
    int per_sm = 0, sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query<G, S, B, 2>, B, 0);
    return static_cast<int64_t>(std::max(1, per_sm)) * sms;
  }();
  return n;
}

template <int G, int S, int B>
cudaError_t launch_query_gsb(const QueryLaunch& L, cudaStream_t st) {
  const int per_block = B / G;
  const int64_t blocks = (L.n + per_block - 1) / per_block;
  if (!L.cplx || !L.cplx_count) return launch_query_gsbm<G, S, B, 0>(L, st, blocks);
  cudaError_t e = launch_query_gsbm<G, S, B, 1>(L, st, blocks);
  if (e != cudaSuccess) return e;
  // K2b: a grid-stride pass over the queued queries (their number is known only on the device)
  return launch_query_gsbm<G, S, B, 2>(L, st, std::min<int64_t>(blocks, resident_blocks<G, S, B>()));
}

// K1 / K2 block sizes: DGDS_APPEND_BLOCK = 32 | 64 | 256, DGDS_QUERY_BLOCK = 32 | 64 | 128 | 256
// (read once per process)
int block_env(const char* name, int dflt) {
  const char* e = std::getenv(name);
  const int v = e ? std::atoi(e) : dflt;
  return (v == 32 || v == 64 || v == 128) ? v : kBlock;
}
int query_block() {
  static const int b = block_env("DGDS_QUERY_BLOCK", kQueryBlockDefault);
  return b;
}
int append_block() {
  static const int b = block_env("DGDS_APPEND_BLOCK", kAppendBlockDefault);
  return b == 128 ? kBlock : b;
}

// DGDS_DEBUG_SYNC=1: wait for each append kernel with a deadline and name the one that does not
// finish (debug builds of a new kernel; off by default).
void debug_sync(cudaStream_t st, const char* what) {
  static const bool on = std::getenv("DGDS_DEBUG_SYNC") != nullptr;
  if (!on) return;
  for (int i = 0; i < 5000; ++i) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) {
      std::fprintf(stderr, "[dgds debug] %s failed: %s\n", what, cudaGetErrorString(e));
      std::abort();
    }
    usleep(1000);
  }
  std::fprintf(stderr, "[dgds debug] %s did not finish within 5 s\n", what);
  std::abort();
}

template <int G, int S>
cudaError_t launch_query_gs(const QueryLaunch& L, cudaStream_t st) {
  const int blk = query_block();
  if (blk == 32) return launch_query_gsb<G, S, 32>(L, st);
  if (blk == 64) return launch_query_gsb<G, S, 64>(L, st);
  if (blk == 128) return launch_query_gsb<G, S, 128>(L, st);
  return launch_query_gsb<G, S, 256>(L, st);
}

template <int G>
cudaError_t launch_query_g(const QueryLaunch& L, int32_t max_s, cudaStream_t st) {
  if (max_s <= 8) return launch_query_gs<G, 8>(L, st);
  if (max_s <= 16) return launch_query_gs<G, 16>(L, st);
  return launch_query_gs<G, 32>(L, st);
}

}  // namespace

std::atomic<unsigned long long> g_kernel_launches{0};

namespace {
// Launch with programmatic stream serialization: the launch overlaps the previous kernel's
// tail; the kernel's first instruction (griddepcontrol.wait) waits for that kernel's completion.
template <class... P, class... A>
cudaError_t launch_pdl(void (*kernel)(P...), int64_t blocks, int threads, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(threads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}
}  // namespace

cudaError_t launch_append(const DevTrie& T, const AppendSeg* d_segs, int64_t nseg, const AppendPiece* d_pieces,
                          int64_t npieces, const int32_t* d_tokens, const CopyPiece* d_grow, int64_t ngrow,
                          cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  {
    const int64_t work = std::max<int64_t>(nseg, (npieces + ngrow) * kWarp);
    const int64_t blocks = std::min<int64_t>((work + 255) / 256, 148 * 8);
    k_stage<<<static_cast<unsigned>(blocks), 256, 0, st>>>(T, d_segs, nseg, d_pieces, npieces, d_tokens, d_grow,
                                                             ngrow);
  }
  debug_sync(st, "k_stage");
  const int blk = append_block();
  const int64_t wpb = blk / kWarp;
  const int64_t blocks = (nseg + wpb - 1) / wpb;
  cudaError_t e;
  if (blk == 32) e = launch_pdl(k_append<32>, blocks, 32, st, T, d_segs, nseg);
  else if (blk == 64) e = launch_pdl(k_append<64>, blocks, 64, st, T, d_segs, nseg);
  else e = launch_pdl(k_append<kBlock>, blocks, kBlock, st, T, d_segs, nseg);
  if (e != cudaSuccess) return e;
  debug_sync(st, "k_append");
  if ((e = launch_pdl(k_walks, 148 * 16, 128, st, T)) != cudaSuccess) return e;  // ~1 thread per event
  debug_sync(st, "k_walks");
  g_kernel_launches.fetch_add(3, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_query(const QueryLaunch& L, int32_t max_k, int32_t max_s, cudaStream_t st) {
  if (L.n <= 0) return cudaSuccess;
  if (L.stats && !L.stat_part) return cudaErrorInvalidValue;
  cudaError_t e;
  if (max_k <= 4) e = launch_query_g<4>(L, max_s, st);
  else if (max_k <= 8) e = launch_query_g<8>(L, max_s, st);
  else e = launch_query_g<32>(L, max_s, st);
  return e;  // the counters are folded by k_query's last block
}

cudaError_t launch_verify(int64_t n, int32_t k_stride, int32_t s_stride, const int32_t* n_cands, const int32_t* lens,
                          const int32_t* tokens, const int32_t* truth, int32_t truth_stride, const int32_t* truth_left,
                          const int32_t* limit, int32_t* drafted, int32_t* accepted, int32_t* emitted,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  k_verify<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, k_stride, s_stride, n_cands, lens, tokens,
                                                                      truth, truth_stride, truth_left, limit, drafted,
                                                                      accepted, emitted);
  return cudaGetLastError();
}

__global__ void k_copy_pieces(const CopyPiece* __restrict__ pieces, int64_t n, const int32_t* __restrict__ from,
                              int32_t* to) {
  const int lane = lane_id();
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x / kWarp);
  for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp; w < n; w += nw) {
    const CopyPiece pc = pieces[w];
    for (uint32_t i = lane; i < pc.len; i += kWarp) to[pc.dst + i] = from[pc.src + i];
  }
}

cudaError_t launch_copy_pieces(const CopyPiece* d_pieces, int64_t n, const int32_t* from, int32_t* to, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 8);
  k_copy_pieces<<<static_cast<unsigned>(blocks), 256, 0, st>>>(d_pieces, n, from, to);
  return cudaGetLastError();
}

cudaError_t launch_blob_fill(const BlobPiece* d_pieces, int64_t n, const int32_t* hist, uint8_t* out,
                             cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 8);
  k_blob_fill<<<static_cast<unsigned>(blocks), 256, 0, st>>>(d_pieces, n, hist, out);
  return cudaGetLastError();
}

cudaError_t launch_set_u32(uint32_t* dst, uint32_t value, cudaStream_t st) {
  k_set_u32<<<1, 1, 0, st>>>(dst, value);
  return cudaGetLastError();
}

cudaError_t launch_rebuild(const DevTrie& from, const DevTrie& to, const uint32_t* root_alive, uint32_t* remap,
                           cudaStream_t st) {
  k_rebuild_place<<<148 * 8, 256, 0, st>>>(from, to, root_alive, remap);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_rebuild_link<<<148 * 8, 256, 0, st>>>(to, remap);
  return cudaGetLastError();
}

cudaError_t launch_remap_active(const DevTrie& T, const uint32_t* streams, int64_t nstreams, const uint32_t* remap,
                                cudaStream_t st, uint64_t from_cap) {
  if (nstreams <= 0) return cudaSuccess;
  const int64_t threads = nstreams * kWarp;
  k_remap_active<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(T.active, T.ov, streams, nstreams,
                                                                                 remap, from_cap);
  return cudaGetLastError();
}

cudaError_t launch_node_count(const DevTrie& T, unsigned long long* out, cudaStream_t st) {
  k_node_count<<<148 * 8, 256, 0, st>>>(T, out);
  return cudaGetLastError();
}

cudaError_t launch_route_pack(int64_t n, int32_t world, const int32_t* owner, const uint32_t* records,
                              int32_t rec_words, uint32_t* out, int64_t* counts, int64_t* perm, void* scratch,
                              cudaStream_t st) {
  if (world > 8) return cudaErrorInvalidValue;
  const int64_t ntiles = (n + kRouteTile - 1) / kRouteTile;
  int64_t* tile_counts = static_cast<int64_t*>(scratch);
  if (n > 0)
    k_route_count<<<static_cast<unsigned>(ntiles), 256, world * sizeof(int), st>>>(n, world, owner, tile_counts);
  k_route_scan<<<1, 1, 0, st>>>(world, ntiles, tile_counts, counts);
  if (n > 0)
    k_route_scatter<<<static_cast<unsigned>(ntiles), kRouteTile, 0, st>>>(n, world, owner, records, rec_words,
                                                                            tile_counts, out, perm);
  return cudaGetLastError();
}

cudaError_t launch_route_pack_padded(int64_t n, int32_t world, const int32_t* owner, const uint32_t* records,
                                     int32_t rec_words, int64_t cap, uint32_t* out, int64_t* slot, int32_t* overflow,
                                     void* scratch, cudaStream_t st) {
  if (world > 8) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(out, 0xFF, static_cast<size_t>(world) * cap * rec_words * 4, st);
  if (e != cudaSuccess || n <= 0) return e;
  const int64_t ntiles = (n + kRouteTile - 1) / kRouteTile;
  int64_t* tile_counts = static_cast<int64_t*>(scratch);
  k_route_count<<<static_cast<unsigned>(ntiles), 256, world * sizeof(int), st>>>(n, world, owner, tile_counts);
  k_route_scan_local<<<1, 1, 0, st>>>(world, ntiles, tile_counts);
  k_route_scatter_padded<<<static_cast<unsigned>(ntiles), kRouteTile, 0, st>>>(n, world, owner, records, rec_words,
                                                                                 cap, tile_counts, out, slot,
                                                                                 overflow);
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

// ---------------------------------------------------------------------------
// Compaction of query results for the host path: strided [n][K][S] candidate
// buffers -> dense per-candidate records + dense tokens, so the device->host
// copy carries only real candidates.
#include <cub/block/block_scan.cuh>

namespace dgds {
namespace {

constexpr int kCmpBlock = 256;

__global__ void k_cmp_count(int64_t n, CmpIn in, long long* block_sums) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * kCmpBlock + threadIdx.x;
  int c = 0, t = 0;
  if (q < n) {
    c = in.n_cands[q * in.qs_nc];
    for (int j = 0; j < c; ++j) t += in.lens[q * in.qs_len + j];
  }
  using BS = cub::BlockScan<int, kCmpBlock>;
  __shared__ typename BS::TempStorage tmp;
  int cs, ts;
  BS(tmp).InclusiveSum(c, cs);
  __syncthreads();
  BS(tmp).InclusiveSum(t, ts);
  if (threadIdx.x == kCmpBlock - 1) {
    block_sums[2 * blockIdx.x] = cs;
    block_sums[2 * blockIdx.x + 1] = ts;
  }
}

__global__ void __launch_bounds__(kCmpBlock) k_cmp_scan(int64_t nblocks, long long* block_sums, long long* totals,
                                                        const long long* __restrict__ carry_in) {
  // exclusive scan of the per-block (candidates, tokens) sums, one block, kCmpBlock at a time
  using BS = cub::BlockScan<long long, kCmpBlock>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ long long carry[2];
  if (threadIdx.x == 0) {
    carry[0] = carry_in ? carry_in[0] : 0;
    carry[1] = carry_in ? carry_in[1] : 0;
  }
  __syncthreads();
  for (int64_t b0 = 0; b0 < nblocks; b0 += kCmpBlock) {
    const int64_t b = b0 + threadIdx.x;
    long long c = b < nblocks ? block_sums[2 * b] : 0, t = b < nblocks ? block_sums[2 * b + 1] : 0;
    long long cx, tx, ct, tt;
    BS(tmp).ExclusiveSum(c, cx, ct);
    __syncthreads();
    BS(tmp).ExclusiveSum(t, tx, tt);
    if (b < nblocks) {
      block_sums[2 * b] = carry[0] + cx;
      block_sums[2 * b + 1] = carry[1] + tx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry[0] += ct;
      carry[1] += tt;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    totals[0] = carry[0];
    totals[1] = carry[1];
  }
}

__global__ void k_cmp_scatter(int64_t n, CmpIn in, const long long* __restrict__ block_sums, CandMeta* meta,
                              int32_t* tok_out, int64_t* cand_off, int64_t* tok_off, int32_t* v_out) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * kCmpBlock + threadIdx.x;
  int c = 0, t = 0;
  if (q < n) {
    c = in.n_cands[q * in.qs_nc];
    for (int j = 0; j < c; ++j) t += in.lens[q * in.qs_len + j];
  }
  using BS = cub::BlockScan<int, kCmpBlock>;
  __shared__ typename BS::TempStorage tmp;
  int co, to;
  BS(tmp).ExclusiveSum(c, co);
  __syncthreads();
  BS(tmp).ExclusiveSum(t, to);
  if (q >= n) return;
  long long cb = block_sums[2 * blockIdx.x] + co, tb = block_sums[2 * blockIdx.x + 1] + to;
  if (cand_off) cand_off[q] = cb;
  for (int j = 0; j < c; ++j) {
    const int L = in.lens[q * in.qs_len + j];
    meta[cb + j] = CandMeta{in.scores[q * in.qs_sc + j], in.supports[q * in.qs_sp + j], L, 0};
    if (tok_off) tok_off[cb + j] = tb;
    const int32_t* src = in.tokens + q * in.qs_tok + static_cast<int64_t>(j) * in.cs_tok;
    for (int i = 0; i < L; ++i) tok_out[tb + i] = src[i];
    tb += L;
  }
  if (in.verify && v_out)  // drafted | accepted | emitted -> [3][n]
    for (int k = 0; k < 3; ++k) v_out[k * n + q] = in.verify[q * in.qs_v + k];
}

// Device -> (mapped) host copy of regions whose sizes are only known on the device:
// 4-B head up to 16-B alignment, coalesced 16-B body (PCIe-friendly), 4-B tail.
__global__ void k_copy_out(const long long* __restrict__ totals, CopyOutRegions R) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int r = 0; r < R.n; ++r) {
    int64_t b0 = 0, b1 = R.fixed_bytes[r];
    if (R.total_idx[r] >= 0) {
      b1 = totals[R.total_idx[r]] * R.elem_bytes[r];
      if (R.begin_idx[r] >= 0) b0 = totals[R.begin_idx[r]] * R.elem_bytes[r];
    }
    if (b1 <= b0) continue;
    const char* src = R.src[r];
    char* dst = R.dst[r];
    const int64_t mis = static_cast<int64_t>((reinterpret_cast<uintptr_t>(src) + b0) & 15);
    const int64_t a0 = b0 + ((16 - mis) & 15) < b1 ? b0 + ((16 - mis) & 15) : b1;
    const int64_t body = (b1 - a0) & ~int64_t{15};
    const int64_t a1 = a0 + body;
    if (tid < (a0 - b0) / 4)
      reinterpret_cast<uint32_t*>(dst + b0)[tid] = reinterpret_cast<const uint32_t*>(src + b0)[tid];
    const uint4* s16 = reinterpret_cast<const uint4*>(src + a0);
    uint4* d16 = reinterpret_cast<uint4*>(dst + a0);
    for (int64_t i = tid; i < body / 16; i += nth) d16[i] = s16[i];
    if (tid < (b1 - a1) / 4)
      reinterpret_cast<uint32_t*>(dst + a1)[tid] = reinterpret_cast<const uint32_t*>(src + a1)[tid];
  }
}

}  // namespace

cudaError_t launch_compact_in(int64_t n, const CmpIn& in, long long* block_sums, long long* totals, CandMeta* meta,
                              int32_t* tok_out, int64_t* cand_off, int64_t* tok_off, int32_t* v_out,
                              const long long* carry_in, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t nb = (n + kCmpBlock - 1) / kCmpBlock;
  g_kernel_launches.fetch_add(3, std::memory_order_relaxed);
  k_cmp_count<<<static_cast<unsigned>(nb), kCmpBlock, 0, st>>>(n, in, block_sums);
  k_cmp_scan<<<1, kCmpBlock, 0, st>>>(nb, block_sums, totals, carry_in);
  k_cmp_scatter<<<static_cast<unsigned>(nb), kCmpBlock, 0, st>>>(n, in, block_sums, meta, tok_out, cand_off, tok_off,
                                                                  v_out);
  return cudaGetLastError();
}

cudaError_t launch_compact(int64_t n, int32_t K, int32_t S, const int32_t* n_cands, const int32_t* lens,
                           const double* scores, const int64_t* supports, const int32_t* tokens,
                           long long* block_sums, long long* totals, CandMeta* meta, int32_t* tok_out,
                           int64_t* cand_off, int64_t* tok_off, const long long* carry_in, cudaStream_t st) {
  CmpIn in{};  // the query kernel's internal SoA outputs
  in.n_cands = n_cands;
  in.qs_nc = 1;
  in.lens = lens;
  in.qs_len = K;
  in.scores = scores;
  in.qs_sc = K;
  in.supports = supports;
  in.qs_sp = K;
  in.tokens = tokens;
  in.qs_tok = static_cast<int64_t>(K) * S;
  in.cs_tok = S;
  return launch_compact_in(n, in, block_sums, totals, meta, tok_out, cand_off, tok_off, nullptr, carry_in, st);
}

cudaError_t launch_copy_out(const long long* totals, const CopyOutRegions& R, int64_t max_bytes, cudaStream_t st,
                            int max_blocks) {
  if (R.n == 0 || max_bytes <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>(max_blocks, (max_bytes / 16 + 255) / 256 + 1);
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  k_copy_out<<<static_cast<unsigned>(blocks), 256, 0, st>>>(totals, R);
  return cudaGetLastError();
}

}  // namespace dgds

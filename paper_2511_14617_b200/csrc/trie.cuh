// trie.cuh — HBM layout of the per-GPU draft-index arena and its device helpers.
//
// One arena per GPU holds the counted suffix tries of every prompt group the
// GPU owns (reference: one GroupDraftIndex per group, proj/src/cst.cpp:79-116).
// B200-first layout: one open-addressing table of 32-byte SLOTS — one DRAM
// sector each — where a slot IS a trie node:
//
//   h            u64  rolling content hash of (group root, window tokens); 0 = empty
//   parent       u32  node id of the window without its last token (root id at depth 1)
//   token        i32  last token of the window
//   count        u32  occurrences of the window MINUS ONE (Node::count - 1, cst.hpp:93):
//                     the inserting occurrence is implicit, so an insert never
//                     touches the counter and only repeat occurrences add to it
//   first_child  u32  most recently created child, 0 = none (Node::first_child)
//   next_sibling u32  prepend-linked sibling list (Node::next_sibling)
//   root         u32  group root id (lets a rebuild drop dead groups)
//
// Node id = slot index + 1. The 16-byte key {h, parent, token} is matched
// EXACTLY — (parent, token) is the reference's edge key (cst.cpp:86-88) — so
// hash collisions can cost a probe but never change a result. The hash only
// chooses the HOME slot, and because it depends on window content rather than
// on node ids, (a) append can compute and prefetch the home slot of every
// window of a record before the dependent claim chain runs, and (b) a draft
// query can probe all prefixes of all candidate suffixes in one parallel round
// trip instead of walking parent -> child (cst.cpp:160-178).
//
// Group roots are not slots: root ids are 0xFFFFFFFF - r for root index r.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dgds {

constexpr int kWarp = 32;
constexpr int kUsedParts = 64;  // partitions of the occupancy counter (index p * 8)
constexpr uint32_t kRootTop = 0xFFFFFFFFu;
constexpr unsigned long long kHashMul = 0x9E3779B97F4A7C15ull;  // odd multiplier of the rolling hash

struct __align__(32) Slot {
  unsigned long long h;
  uint32_t parent;
  int32_t token;
  uint32_t count;
  uint32_t first_child;
  uint32_t next_sibling;
  uint32_t root;
};
static_assert(sizeof(Slot) == 32, "slot must be one 32-B sector");

struct SlotView {  // one 256-bit load
  unsigned long long h;
  uint32_t parent;
  int32_t token;
  uint32_t count;
  uint32_t first_child;
  uint32_t next_sibling;
  uint32_t root;
};

struct DevTrie {
  Slot* slots;
  uint64_t cap;              // slots (ids 1..cap); arbitrary size (fast-range reduction)
  uint32_t* active;          // [stream][32]: node of the last (i+1)-token context (Stream::active, cst.hpp:117)
  int32_t* tail;             // [stream][32]: ring of the last 32 tokens (position & 31)
  unsigned long long* used;  // occupied slots: kUsedParts counters, 64 B apart (sum = occupancy)
  int32_t depth_cap;         // max_pattern_len + max_spec_len (cst.cpp:106-107)
  int32_t lim_pattern;       // Limits::max_pattern_len
  int32_t lim_spec;          // Limits::max_spec_len
  int32_t ahead;             // append look-ahead (tokens) of the L2 prefetch; 0 = off
  int32_t claim_cas;         // append claim: 1 = CAS-first, 0 = read the window first
  int32_t* hist;             // append-only token history (replica sync blobs); K1 copies every token
  unsigned long long* dbg;   // optional (debug): per-warp [start, end] globaltimer of K1
};

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ bool is_root_id(uint32_t id, uint64_t cap) { return id > cap; }

// Hash of the empty window of a group, and one rolling step.
__device__ __forceinline__ unsigned long long root_hash(uint32_t root) { return splitmix64(root); }
__device__ __forceinline__ unsigned long long hash_step(unsigned long long h, int32_t t) {
  return h * kHashMul + static_cast<uint32_t>(t) + 1ull;
}
__device__ __forceinline__ unsigned long long key_hash(unsigned long long h) { return h ? h : 1ull; }

__device__ __forceinline__ unsigned long long pack_pt(uint32_t parent, int32_t token) {
  return static_cast<unsigned long long>(parent) |
         (static_cast<unsigned long long>(static_cast<uint32_t>(token)) << 32);
}

// Slots are grouped in BUCKETS of 2 (64 B = one DRAM access at the L2's 64-B
// fetch granularity). Probing is linear at bucket granularity: a lookup reads a
// whole bucket per step; at load 0.42 that is 1.12 bucket reads per access
// (4-slot 128-B buckets: 1.03 reads but two DRAM accesses each).
constexpr int kBucket = 2;
// A probe step reads kWindow consecutive slots (one bucket) per round trip;
// probing is plain linear probing over slots. (Reading the next bucket too —
// kWindow 4 — removes the 12% overflow round trips but doubles the DRAM
// accesses, and measured slower: both kernels are random-access bound.)
constexpr int kWindow = 2;

// slot index k of the probe window that starts at bucket b (wraps at the end)
__device__ __forceinline__ uint64_t window_slot(uint64_t b, int k, uint64_t cap) {
  const uint64_t i = b * kBucket + static_cast<uint64_t>(k);
  return i < cap ? i : i - cap;
}

// Home bucket: Lemire fast-range over a remixed hash (uniform for any size).
__device__ __forceinline__ uint64_t home_bucket(unsigned long long h, uint64_t nbuckets) {
  return __umul64hi(splitmix64(h), nbuckets);
}

// occurrences of a node from its stored counter (see Slot::count)
__device__ __forceinline__ uint32_t occurrences(uint32_t stored) { return stored + 1u; }

__device__ __forceinline__ SlotView load_slot_nc(const Slot* p) {
  unsigned long long a, b, c, d;
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  SlotView v;
  v.h = a;
  v.parent = static_cast<uint32_t>(b);
  v.token = static_cast<int32_t>(static_cast<uint32_t>(b >> 32));
  v.count = static_cast<uint32_t>(c);
  v.first_child = static_cast<uint32_t>(c >> 32);
  v.next_sibling = static_cast<uint32_t>(d);
  v.root = static_cast<uint32_t>(d >> 32);
  return v;
}

// 16-byte key {h, parent|token} of a slot, read-only path.
__device__ __forceinline__ void load_key_nc(const Slot* p, unsigned long long& k0, unsigned long long& k1) {
  asm("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(k0), "=l"(k1) : "l"(p));
}

__device__ __forceinline__ void prefetch_l2_window(const void* p) {  // one probe window
#ifdef DGDS_BULK_PREFETCH
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "n"(kWindow * 32) : "memory");
#else
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));  // per-thread: no TMA-unit queue
#endif
}
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// Bucket probe on the read-only path. exact: match {h, parent|token};
// otherwise match {h, token} (content probe — the caller checks the parent).
// Returns the node id (slot + 1), 0 if absent; rec = the matched slot.
template <bool kExact>
__device__ __forceinline__ uint32_t probe(const DevTrie& T, unsigned long long h, uint32_t parent, int32_t token,
                                          SlotView& rec) {
  const uint64_t cap = T.cap;
  const uint64_t nb = cap / kBucket;
  const unsigned long long pt = pack_pt(parent, token);
  uint64_t b = home_bucket(h, nb);
  while (true) {
    unsigned long long k0[kWindow], k1[kWindow];
#pragma unroll
    for (int s = 0; s < kWindow; ++s) load_key_nc(T.slots + window_slot(b, s, cap), k0[s], k1[s]);
#pragma unroll
    for (int s = 0; s < kWindow; ++s) {
      const bool hit = k0[s] == h && (kExact ? k1[s] == pt : static_cast<int32_t>(k1[s] >> 32) == token);
      if (hit) {
        const uint64_t i = window_slot(b, s, cap);
        rec = load_slot_nc(T.slots + i);  // same sector as the key: an L1 hit
        return static_cast<uint32_t>(i + 1);
      }
      if (k0[s] == 0ull) return 0;
    }
    b += kWindow / kBucket;
    if (b >= nb) b -= nb;
  }
}

__device__ __forceinline__ uint32_t find_exact(const DevTrie& T, unsigned long long h, uint32_t parent, int32_t token,
                                               SlotView& rec) {
  return probe<true>(T, h, parent, token, rec);
}
__device__ __forceinline__ uint32_t find_by_content(const DevTrie& T, unsigned long long h, int32_t token,
                                                    SlotView& rec) {
  return probe<false>(T, h, 0u, token, rec);
}

}  // namespace dgds

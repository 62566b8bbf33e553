// trie.cuh — HBM layout of the per-GPU draft-index arena and its device helpers.
//
// One arena per GPU holds the counted suffix tries of every prompt group the
// GPU owns (reference: one GroupDraftIndex per group, proj/src/cst.cpp:79-116,
// a trie of every window of length <= max_pattern_len + max_spec_len).
//
// B200-first layout: the trie is stored COMPRESSED. Only two kinds of windows
// are materialised as ENTRIES of one open-addressing table of 32-byte slots
// (one DRAM sector each):
//   - nodes: windows that occur at least twice (count >= 2);
//   - leaves: windows that occur exactly once and whose parent is a node (or
//     the group root). A leaf records its one occurrence (stream, position).
// Every other window occurs exactly once and lies on the chain below a leaf:
// its content is the stream's own continuation after the leaf's occurrence,
// read from the per-stream token history (StreamInfo below). A count-1 window
// has at most one child, and its prefixes all have counts >= its own, so the
// whole subtree under a leaf is that single chain, capped at the depth limit
// and the stream's stored length. The reference's trie is therefore fully
// determined (nodes, counts, child sets), with ~1-2 entries per appended token
// instead of ~22 trie nodes (17-23 nodes per token).
//
// Slot (32 B):
//   [0,4)   parent       node id of the window without its last token (group root id at depth 1)
//   [4,8)   token        last token of the window            } edge key (cst.cpp:86-88): exact
//   [8,12)  occ_stream   stream slot (bits 0-23) | depth-1 (bits 24-28) } the first occurrence:
//   [12,16) occ_pos      position of the window's last token in it     } set atomically with the key
//   [16,20) count        occurrences - 1 (0 = leaf)
//   [20,24) first_child  most recently created child entry, 0 = none (Node::first_child)
//   [24,28) h32          content hash (home bucket + content probes); never 0 once written
//   [28,32) next_sibling prepend-linked sibling list (Node::next_sibling)
//
// Node id = slot index + 1. The 8-byte key {parent, token} is the reference's
// edge key and is matched exactly; the content hash only chooses the home
// slot, so (a) a draft query probes all prefixes of a suffix in one parallel
// round instead of walking parent -> child (cst.cpp:160-178), and (b) a rebuild
// re-places an entry from its own fields. Group roots are not slots: root ids
// are 0xFFFFFFFF - r for root index r.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dgds {

constexpr int kWarp = 32;
constexpr int kUsedParts = 64;  // partitions of the occupancy counter (index p * 8)
constexpr uint32_t kRootTop = 0xFFFFFFFFu;
constexpr unsigned long long kHashMul = 0x9E3779B97F4A7C15ull;  // odd multiplier of the rolling hash
constexpr uint32_t kStreamMask = 0x00FFFFFFu;                 // occ_stream: stream slot bits
constexpr uint32_t kRootSpan = 1u << 22;                      // group root ids: kRootTop - r, r < kRootSpan
constexpr uint32_t kMinRootId = kRootTop - kRootSpan + 1u;

struct __align__(32) Slot {
  uint32_t parent;
  int32_t token;
  uint32_t occ_stream;  // stream | (depth - 1) << 24
  uint32_t occ_pos;
  uint32_t count;
  uint32_t first_child;
  uint32_t h32;
  uint32_t next_sibling;
};
static_assert(sizeof(Slot) == 32, "slot must be one 32-B sector");

// Per request stream: its token history extent and stored length (Stream::tokens,
// cst.hpp:115-118). The history lives in one arena (DevTrie::shist), each stream in a
// contiguous extent that is moved (copied) to a larger one when it fills.
struct __align__(16) StreamInfo {
  unsigned long long base;  // first token of the stream in DevTrie::shist
  uint32_t len;             // tokens stored
  uint32_t root;            // group root id of the stream's group
};

// A leaf converted to a node by K1: its displaced occurrence continues in K1b (k_walks).
struct WalkEvent {
  unsigned long long h;  // rolling content hash of the window
  uint32_t id;           // the entry (now a node)
  uint32_t depth;        // its window length
  uint32_t stream;       // the displaced occurrence: the window ends at `pos` of `stream`
  uint32_t pos;
};

struct DevTrie {
  Slot* slots;
  uint64_t cap;              // slots (ids 1..cap)
  uint32_t* active;          // [stream][32]: entry id of the (i+1)-token window ending at the stream's last
                             // token when it is a node (count >= 2), else 0 (Stream::active, cst.hpp:117)
  uint32_t* ov;              // [stream][32]: the same, set by conversion walks; taken by the next append
  StreamInfo* sinfo;         // [stream]
  int32_t* shist;            // per-stream token extents (queries and walks read continuations here)
  unsigned long long* used;  // entries: kUsedParts counters, 64 B apart (sum = occupancy)
  int32_t depth_cap;         // max_pattern_len + max_spec_len (cst.cpp:106-107)
  int32_t lim_pattern;       // Limits::max_pattern_len
  int32_t lim_spec;          // Limits::max_spec_len
  int32_t pad_;
  int32_t* hist;             // append-only token history in record order (replica sync blobs)
  int32_t* err;              // device error flags (bit 1: negative token in a device-path batch)
  WalkEvent* ev;             // conversion events of the batch being appended (capacity: its window count)
  unsigned long long* ev_count;  // [0] events queued, [1] k_walks block ticket
  // capacities, for the bounds checks of the test-only "checked" build (DGDS_CHECK)
  uint64_t stream_cap, shist_cap, hist_cap, ev_cap;
  unsigned long long* dbg;   // optional (debug): per-warp [start, end] globaltimer of K1
  // optional (debug, DGDS_K1_STATS): [0] K1 claims, [1] K1 leaves created, [2] K1 conversions,
  // [3] K1 rider matches, [4] events queued, [5] walk steps, [6] longest walk (steps), [7] walks
  unsigned long long* k1_stats;
};

// Test-only bounds checks (build variant "checked", -DDGDS_CHECKED): a violated invariant sets err
// bit 5 (dgds_device_error), so a parity run under that build also proves every index in range.
#ifdef DGDS_CHECKED
#define DGDS_CHECK(T, cond)                          \
  do {                                               \
    if (!(cond)) atomicOr((T).err, 32);              \
  } while (0)
#else
#define DGDS_CHECK(T, cond) \
  do {                      \
  } while (0)
#endif

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ bool is_root_id(uint32_t id, uint64_t cap) { return id > cap; }

// Rolling hash of a window: the empty window of a group, then one step per token.
__device__ __forceinline__ unsigned long long root_hash(uint32_t root) { return splitmix64(root); }
__device__ __forceinline__ unsigned long long hash_step(unsigned long long h, int32_t t) {
  return h * kHashMul + static_cast<uint32_t>(t) + 1ull;
}
// Stored 32-bit content hash (never 0). DGDS_TEST_HASH_BITS (test builds only) truncates it so
// that content probes collide constantly and every exact-key fallback path runs.
// One xor-shift and one multiply: the rolling hash is linear in the tokens, and the finaliser only
// has to spread it over 32 bits (keys are exact; a collision costs a probe, never a result).
__device__ __forceinline__ uint32_t hash32(unsigned long long h) {
  h ^= h >> 32;
  uint32_t v = static_cast<uint32_t>((h * 0xD6E8FEB86659FD93ull) >> 32);
#ifdef DGDS_TEST_HASH_BITS
  v &= (1u << DGDS_TEST_HASH_BITS) - 1u;
#endif
  return v ? v : 1u;
}

__device__ __forceinline__ unsigned long long pack_key(uint32_t parent, int32_t token) {
  return static_cast<unsigned long long>(parent) |
         (static_cast<unsigned long long>(static_cast<uint32_t>(token)) << 32);
}
__device__ __forceinline__ unsigned long long pack_occ(uint32_t stream, uint32_t depth, uint32_t pos) {
  return static_cast<unsigned long long>(stream | ((depth - 1u) << 24)) |
         (static_cast<unsigned long long>(pos) << 32);
}
__host__ __device__ __forceinline__ uint32_t occ_stream(uint32_t s) { return s & kStreamMask; }
__host__ __device__ __forceinline__ uint32_t occ_depth(uint32_t s) { return (s >> 24) + 1u; }

// Slots are grouped in BUCKETS of 2 (64 B = one DRAM access at the L2's 64-B
// fetch granularity); probing is linear over slots from the first slot of the home bucket.
constexpr int kBucket = 2;
constexpr int kWindow = 2;  // slots read per probe round trip (one bucket)

__device__ __forceinline__ uint64_t window_slot(uint64_t b, int k, uint64_t cap) {
  const uint64_t i = b * kBucket + static_cast<uint64_t>(k);
  return i < cap ? i : i - cap;
}

// Home bucket from the stored hash alone (a rebuild re-places entries without their windows):
// fast-range of the 32-bit hash. Test builds that truncate the hash spread it again first.
__host__ __device__ __forceinline__ uint64_t home_bucket(uint32_t h32, uint64_t nbuckets) {
#ifdef DGDS_TEST_HASH_BITS
  return (static_cast<uint64_t>(splitmix64(h32) >> 32) * nbuckets) >> 32;
#else
  return (static_cast<uint64_t>(h32) * nbuckets) >> 32;
#endif
}

// occurrences of a window from its stored counter (see Slot::count)
__device__ __forceinline__ uint32_t occurrences(uint32_t stored) { return stored + 1u; }

struct SlotView {
  uint32_t parent;
  int32_t token;
  uint32_t occ_stream;
  uint32_t occ_pos;
  uint32_t count;
  uint32_t first_child;
  uint32_t h32;
  uint32_t next_sibling;
};

__device__ __forceinline__ SlotView load_slot_nc(const Slot* p) {
  unsigned long long a, b, c, d;
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  SlotView v;
  v.parent = static_cast<uint32_t>(a);
  v.token = static_cast<int32_t>(static_cast<uint32_t>(a >> 32));
  v.occ_stream = static_cast<uint32_t>(b);
  v.occ_pos = static_cast<uint32_t>(b >> 32);
  v.count = static_cast<uint32_t>(c);
  v.first_child = static_cast<uint32_t>(c >> 32);
  v.h32 = static_cast<uint32_t>(d);
  v.next_sibling = static_cast<uint32_t>(d >> 32);
  return v;
}

__device__ __forceinline__ unsigned long long ld_nc_u64(const void* p) {
  unsigned long long v;
  asm("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t hash_word(const Slot* p) {  // h32 (0 = empty slot, after K1)
  return static_cast<uint32_t>(ld_nc_u64(&p->h32));
}

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// Exact probe of edge (parent, token) on the read-only path. Returns the entry id, 0 if absent.
__device__ __forceinline__ uint32_t find_exact(const DevTrie& T, uint32_t h32, uint32_t parent, int32_t token,
                                               SlotView& rec) {
  const uint64_t cap = T.cap;
  const uint64_t nb = cap / kBucket;
  const unsigned long long key = pack_key(parent, token);
  uint64_t b = home_bucket(h32, nb);
  while (true) {
    unsigned long long k[kWindow];
#pragma unroll
    for (int s = 0; s < kWindow; ++s) k[s] = ld_nc_u64(T.slots + window_slot(b, s, cap));
#pragma unroll
    for (int s = 0; s < kWindow; ++s) {
      if (k[s] == key) {
        const uint64_t i = window_slot(b, s, cap);
        rec = load_slot_nc(T.slots + i);  // same sector as the key: an L1 hit
        return static_cast<uint32_t>(i + 1);
      }
      if (k[s] == 0ull) return 0;
    }
    b += kWindow / kBucket;
    if (b >= nb) b -= nb;
  }
}

}  // namespace dgds

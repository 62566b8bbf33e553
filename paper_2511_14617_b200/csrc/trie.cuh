// trie.cuh — HBM layout of the per-GPU draft-index arena and its device helpers.
//
// One arena per GPU holds the counted suffix tries of every prompt group the
// GPU owns (reference: one GroupDraftIndex per group, proj/src/cst.cpp:79-116).
// B200-first layout: a single open-addressing table of 32-byte SLOTS, one DRAM
// sector each, where a slot IS a trie node:
//
//   key          u64  (parent_id << 32) | uint32(token); 0 = empty slot
//   count        u32  occurrences of the window this node spells (Node::count)
//   first_child  u32  id of the most recently created child, 0 = none
//   next_sibling u32  prepend-linked sibling list (Node::next_sibling)
//   depth        u32  window length (1..depth_cap); used by the rebuild only
//   root         u32  id of the group root this node hangs under (rebuild GC)
//   pad          u32
//
// A node's id is (slot index + 1), so a key lookup returns the node record in
// the same 32-B sector — the reference needs an EdgeMap probe (keys_ + vals_)
// plus a separate nodes_[] access per edge (cst.cpp:38-47,86-103). Inserting a
// window is ONE atomicCAS on the home slot (claim-or-find) and a RED on the
// count in the same sector; no node allocator exists at all.
//
// Group roots are not slots: root ids are 0xFFFFFFFF - r for root index r, so
// (parent, token) keys stay unique across all groups in the arena. Root child
// lists are never enumerated (a draft query's locus is never the root,
// cst.cpp:179), so roots need no storage.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dgds {

constexpr int kWarp = 32;
constexpr uint32_t kRootTop = 0xFFFFFFFFu;

struct __align__(32) Slot {
  unsigned long long key;
  uint32_t count;
  uint32_t first_child;
  uint32_t next_sibling;
  uint32_t depth;
  uint32_t root;
  uint32_t pad;
};
static_assert(sizeof(Slot) == 32, "slot must be one 32-B sector");

struct SlotView {  // the fields a query needs, from one 256-bit load
  unsigned long long key;
  uint32_t count;
  uint32_t first_child;
  uint32_t next_sibling;
  unsigned long long tail;  // depth | root (unused by queries)
};

struct DevTrie {
  Slot* slots;
  uint64_t cap;            // slots (ids 1..cap); arbitrary (fast-range reduction, not a mask)
  uint32_t* active;        // [stream_cap][32]: active[i] = node of the last (i+1)-token context
  unsigned long long* used;  // occupied slots (device counter)
  int32_t depth_cap;       // max_pattern_len + max_spec_len (cst.cpp:106-107)
  int32_t lim_pattern;     // Limits::max_pattern_len
  int32_t lim_spec;        // Limits::max_spec_len
  int32_t pad_;
};

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ bool is_root_id(uint32_t id, uint64_t cap) { return id > cap; }

__device__ __forceinline__ unsigned long long edge_key(uint32_t parent, int32_t token) {
  return (static_cast<unsigned long long>(parent) << 32) | static_cast<uint32_t>(token);
}

// Home slot: Lemire fast-range over the 64-bit hash (uniform for any cap).
__device__ __forceinline__ uint64_t home_slot(unsigned long long key, uint64_t cap) {
  return __umul64hi(splitmix64(key), cap);
}

// One 32-byte sector per node visit (LDG.E.ENL2.256 on sm_100a), through the
// non-coherent path: query kernels never run concurrently with an append.
__device__ __forceinline__ SlotView load_slot_nc(const Slot* p) {
  unsigned long long a, b, c, d_unused;
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d_unused) : "l"(p));
  SlotView v;
  v.key = a;
  v.count = static_cast<uint32_t>(b);
  v.first_child = static_cast<uint32_t>(b >> 32);
  v.next_sibling = static_cast<uint32_t>(c);
  v.tail = d_unused;
  return v;
}

// Read-only lookup of child (parent, token): returns the node id (0 = absent)
// and its slot record. Mirrors GroupDraftIndex::child_of (cst.cpp:86-88).
__device__ __forceinline__ uint32_t find_child(const DevTrie& T, uint32_t parent, int32_t token, SlotView& rec) {
  const unsigned long long key = edge_key(parent, token);
  uint64_t i = home_slot(key, T.cap);
  while (true) {
    rec = load_slot_nc(T.slots + i);
    if (rec.key == key) return static_cast<uint32_t>(i + 1);
    if (rec.key == 0ull) return 0;
    i = (i + 1 == T.cap) ? 0 : i + 1;
  }
}

}  // namespace dgds

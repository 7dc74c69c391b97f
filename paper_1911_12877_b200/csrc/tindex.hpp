// tindex.hpp -- triangle index and the folded (closed-form) unit counts of the
// star-shaped plans (see tindex.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/symmine_gpu.h"

namespace smg {

// Per-slot common-neighbour lists of a device CSR.  For slot e = (u, v) (v in
// N(u)), T(e) lists the positions p in N(u) (0 <= p < deg u) with
// adj[off[u] + p] in N(v), ascending (= ascending ids).  T(e) is the row of v
// in the local graph G[N(u)] -- the ego network of u -- in local ids.
struct TIndex {
  uint64_t slots = 0;
  uint64_t entries = 0;                   // sum of tri = 6 x #triangles
  unsigned long long* rev = nullptr;      // slots: index of the reverse slot (v, u)
  uint32_t* tri = nullptr;                // slots: |N(u) & N(v)|
  unsigned long long* toff = nullptr;     // slots + 1: T-list offsets
  uint32_t* tent = nullptr;               // entries: positions in N(u)
  unsigned long long* lowpref = nullptr;  // slots: sum over earlier slots f of u of |T(f) & [0, pos f)|
  uint32_t* k4 = nullptr;                 // entries: |T(u, x) & T(u, w)| for entry w of T(u, x)
  bool has_low = false, has_k4 = false;
};

// Builds the parts that are missing (the lists always; lowpref / k4 on
// request).  Returns 0, or 1 with *err set on a CUDA error (out of memory).
int tindex_build(TIndex* t, const unsigned long long* off, const uint32_t* adj, const uint32_t* src,
                 uint64_t n, uint64_t slots, int num_sms, cudaStream_t st, bool want_low, bool want_k4,
                 std::string* err);
void tindex_free(TIndex* t);

// Plans whose deeper levels all lie in the neighbourhood of v1 and whose
// leaves fold into closed forms over the ego network of v1 (tindex.cu).
enum FastKind {
  kFastNone = 0, kFastStar4 = 1, kFastTailedDiamondA = 2, kFastHouse = 3, kFastTailedDiamondB = 4,
  kFastTailedTriangle = 5, kFastDiamond = 6, kFastPath4 = 7, kFastRectangle = 8, kFastRectangleMotif = 9,
  kFastClique4 = 10,  // never returned by fast_kind: a fully restricted 4-clique plan inside a batch (m4_weights)
  kFastClique5 = 11   // never returned by fast_kind: a fully restricted 5-clique plan (k4.cu, k = 5), counted alone
};
int fast_kind(const smg_plan& p);

struct FastArgs {
  const unsigned long long* off;
  const uint32_t* adj;
  const uint32_t* src;
  uint64_t n, slots;
  uint32_t root_lo, root_hi;           // units (v0, v1) with v0 in [root_lo, root_hi)
  uint64_t e_lo, e_hi;                 // slots the unit kernels walk ([0, slots), or off[lo]..off[hi])
  int via_rev;                         // the unit's own slot is the reverse of the walked one
  uint32_t num_shards;                 // > 1: shard map below
  uint32_t shard;                      // this shard (m4_launch: vertices dealt round-robin)
  uint32_t units_per_edge;             // m4_launch: level-1 units per undirected edge (1: v1 < v0, else 2)
  uint32_t hub_count;                  // m4_launch: centres [0, hub_count) take the grid-wide C4 path
  uint32_t group_end;                  // centres [hub_count, group_end): group tier; the rest one CTA each
  uint32_t c4_blocks;                  // CTAs (= dense tables) of c4_kernel, <= the launch's blocks
  const uint32_t* tcount;              // per-slot triangle counts from k4_count (or null: m4_edge_kernel intersects)
  uint32_t groups;                     // CTA groups of the group tier (each owns one table of gtab)
  uint32_t* gtab;                      // groups x m4_group_table_words(n): packed 16-bit counters, zero
  unsigned long long* gbar;            // groups barrier counters
  const unsigned long long* map_begin;
  const unsigned long long* map_pref;
  uint32_t map_k;
  TIndex t;
  uint32_t* scratch;                   // per warp: scratch_words words (zero between units)
  uint64_t scratch_words;
  uint64_t dmax;                       // max degree
  // two-center kinds (house, tailed diamond b): per-slot accumulators and a
  // dense per-CTA codegree table of n words (zero between centers)
  unsigned long long* acc0;            // slots
  unsigned long long* acc1;            // slots
  unsigned long long* acc2;            // slots
  uint32_t* dense;                     // blocks x n
  unsigned long long* next2;           // second queue cursor (zeroed by the caller)
  // full-count mode (whole root range; house, tailed diamond a/b): signed
  // partial sums, one 128-bit slot (lo, hi) per CTA, summed by the host
  unsigned long long* part;            // blocks x 2
  unsigned long long* next_chunk;      // queue cursor (zeroed by the caller)
  unsigned long long* count;           // checked uint64 sum
  unsigned long long* units;
  unsigned int* overflow;
};

// Scratch words per warp that a kind needs for max degree dmax; per-slot
// accumulator arrays (0..3) and whether it needs the dense per-CTA tables.
uint64_t fast_scratch_words(int kind, uint64_t dmax);
int fast_slot_arrays(int kind);
bool fast_dense(int kind);
// Blocks x 256 threads, persistent.  combine_only: the per-slot accumulators
// of this kind are still valid (a cached earlier full pass): only combine.
int fast_launch(int kind, const FastArgs& a, unsigned blocks, cudaStream_t st, bool combine_only);
// Full-count mode: the per-unit sums of kind over this shard's units land in
// a.part (signed); the host adds global terms (fast_global_terms).  Returns 0
// when launched, 2 when the kind has no full mode.
int fast_launch_full(int kind, const FastArgs& a, unsigned blocks, cudaStream_t st);
bool fast_has_full(int kind);
// 4-vertex kinds, label-free full counts (see tindex.cu): integer combinations
// of subgraph counts of the whole graph.  m4_launch stores the raw sums, per
// CTA as 128-bit pairs, in regions of a.part (kM4Regions x blocks pairs); the
// host applies the kind's weights (m4_weights; false: no such form) and adds
// k4 x the 4-clique count.  Needs a.dense (blocks x n words, zero; C4 wanted),
// a.acc0 (n words, zero; PAW wanted), a.next2 / a.next_chunk (zeroed) and
// a.off/adj/src of the (degree-ordered) CSR.
enum M4Region { kM4C4 = 0, kM4D = 1, kM4T3 = 2, kM4P4E = 3, kM4Paw = 4, kM4Star = 5, kM4Regions = 6 };
struct M4Weights {
  int w[kM4Regions] = {0, 0, 0, 0, 0, 0};
  int k4 = 0;
  unsigned need() const {
    unsigned m = 0;
    for (int r = 0; r < kM4Regions; ++r)
      if (w[r]) m |= 1u << r;
    return m;
  }
};
bool m4_weights(int kind, M4Weights* w);
// words of one group-tier table: packed 16-bit counters, padded to 16 bytes
__host__ __device__ constexpr uint64_t m4_group_table_words(uint64_t n) { return (((n + 1) / 2) + 3) & ~3ull; }
constexpr uint32_t kM4GroupDegree = 512;  // centres from this degree up to the hub degree: group tier
constexpr uint32_t kM4HubDegree = 16384;  // centres of at least this degree are scattered by the whole grid
constexpr uint32_t kM4MaxHubs = 16384;
int m4_launch(const FastArgs& a, unsigned need, unsigned blocks, cudaStream_t st, cudaEvent_t* ev);
// Sum over index entries of k4 * (k4 - 1) (every entry of the index; needs
// the k4 array).  Synchronous.
int tindex_k4_pairs(const TIndex& t, int num_sms, cudaStream_t st, unsigned long long* out, std::string* err);
// Kinds whose units sit on the reverse slot (centre v1 = src of the unit slot).
bool fast_center_v1(int kind);
constexpr int kFastThreads = 256;

}  // namespace smg

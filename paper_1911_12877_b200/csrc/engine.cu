// engine.cu -- B200 (sm_100a) plan executor for symmine count_instances.
//
// Replaces the reference hot path (proj/src/engine.cpp:28-179 and
// proj/include/symmine/set_ops.hpp:18-57):
//   * K1 persistent warp-DFS executor: units are level-1 partial embeddings
//     (directed edge slots (v0,v1) that pass level 1's bound), handed out in
//     chunks from a global atomic queue (dynamic work stealing) instead of the
//     reference's static root blocks (engine.cpp:157-158).  One warp runs the
//     nested loops of one unit depth-first; every set operation is
//     warp-parallel.
//   * K2/K3 bounded intersect / difference: sorted-set probes (branchless
//     binary search), the side to iterate chosen per pair from the two
//     lengths, bounds folded in as prefix truncation (set_ops.hpp:20-25).
//   * K4 count-only leaf: ballot + popc, never materialised
//     (engine.cpp:97-105).
//   * K5 uint64 reduction with carry detection (checked_add, engine.cpp:13-19).
// Candidate sets are hoisted per program.hpp: a prefix is built once when its
// last source vertex is fixed and reused by every deeper sibling.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/symmine_gpu.h"
#include "graph_build.hpp"
#include "k4.hpp"
#include "program.hpp"
#include "tindex.hpp"

namespace smg {

constexpr int kWarpsPerBlock = 8;
constexpr int kThreads = kWarpsPerBlock * 32;
constexpr uint32_t kChunk = 32;  // edge slots per queue grab
// Multi-GPU shard map: the level-1 unit chunks are cut into num_shards *
// kShardSplit super-chunks of equal estimated cost, dealt round-robin.
constexpr uint32_t kShardSplit = 64;
constexpr unsigned kFull = 0xffffffffu;
// Per-warp shared-memory hash.  The generic kernel (plans of depth >= 5, the
// clique-local path) keeps 2048 slots (8 KB) at 3 CTAs/SM; the depth-4 batch
// kernel trades table size for residency: 512 slots (2 KB) at 8 CTAs/SM =
// 64 warps/SM (measured: profiles/r01_tuning.md).
constexpr uint32_t kHashSlots = 2048;       // generic shape (and the static maximum)
constexpr uint32_t kBatchHashSlots = 512;   // depth-4 batch shape
constexpr uint32_t kEmptySlot = 0xffffffffu;  // never a vertex id (ids < n < 2^32)
constexpr size_t kDynSmem = sizeof(uint32_t) * kHashSlots * kWarpsPerBlock;
constexpr size_t kBatchDynSmem = sizeof(uint32_t) * kBatchHashSlots * kWarpsPerBlock;
// CTA tier (heavy_kernel): two 16-warp CTAs per SM (one can run while the
// other waits at a barrier).  Node builds probe an 8K-slot (32 KB) hash
// table; the batched leaf probes a 512K-bit (64 KB) bitmap of the probe set
// over an id slice.
#ifndef SMG_HEAVY_WARPS
#define SMG_HEAVY_WARPS 16
#endif
#ifndef SMG_BITMAP_LOG2
#define SMG_BITMAP_LOG2 14
#endif
constexpr int kHeavyWarps = SMG_HEAVY_WARPS;
constexpr int kHeavyThreads = kHeavyWarps * 32;
#ifndef SMG_HEAVY_MINB
#define SMG_HEAVY_MINB 2
#endif
constexpr int kHeavyMinBlocks = SMG_HEAVY_MINB;             // CTAs per SM
#ifndef SMG_HEAVY_SLOTS_LOG2
#define SMG_HEAVY_SLOTS_LOG2 13
#endif
constexpr uint32_t kHeavySlots = 1u << SMG_HEAVY_SLOTS_LOG2;
constexpr uint32_t kBitmapWords = 1u << SMG_BITMAP_LOG2;    // 64 KB
constexpr uint64_t kBitmapSpan = uint64_t(kBitmapWords) * 32;  // ids per slice
constexpr size_t kHeavySmem = sizeof(uint32_t) * (kHeavySlots + kBitmapWords);
constexpr uint64_t kHeavyMinStream = 32768;  // defer only batches with real streaming work
constexpr uint64_t kHeavyQueueCap = 1ull << 24;

// ---------------------------------------------------------------- device ---

struct Counters {
  unsigned long long next_chunk;
  unsigned long long count;
  unsigned long long elements;
  unsigned long long units;
  unsigned long long heavy_count;  // batches deferred to the CTA tier
  unsigned long long heavy_next;   // CTA-tier queue cursor
  unsigned int overflow;
  unsigned int heavy_done;         // CTAs of heavy_kernel finished
  // SMG_TRACE=1: per-phase cycle and event counters (see kTr* below)
  unsigned long long trace[32];  // >= kTrCount
};

enum {
  kTrUnits = 0, kTrBuildCycles, kTrBatchCycles, kTrBatches, kTrBatchesHashed, kTrStreamElems,
  kTrSearchLists, kTrProbeSetSum, kTrStreamSetSum, kTrLeafCycles, kTrLeaves, kTrBigPCycles,
  kTrDeferred, kTrHeavyItems, kTrHeavyCycles, kTrLongLists, kTrHeavyBuild, kTrHeavyStream,
  kTrWarpBusySum, kTrWarpBusyMax, kTrHeavyElems, kTrHeavyTiles, kTrCount
};

struct KernelArgs {
  const unsigned long long* off;  // n+1
  const uint32_t* adj;            // slots
  const uint32_t* src;            // slots: source vertex of each slot
  uint32_t* scratch;
  uint64_t cap;                   // scratch elements per slot
  uint64_t unit_begin, unit_end;  // edge-slot range
  uint64_t nverts;
  // SMG_TUNE bits (A/B switches kept for measurement; 0 = the tuned defaults):
  //   1 degree-only side choice, 2 no clique-local, 16 always bisect long-list
  //   windows, 64 no per-warp global work area (bisection probes for big P),
  //   512 per-warp global bitmap instead of the radix index for big P,
  //   1024 hub-hub units deferred before their loop-1 sets are built
  uint32_t tune;
  uint32_t heavy_stream;  // SMG_HEAVY_STREAM: CTA-tier threshold on a batch's streamed elements
  uint32_t heavy_min;     // SMG_HEAVY_MIN: big-probe-set batches stream at least this to be deferred
  float list_cost;        // SMG_LIST_COST
  uint32_t shard, num_shards;
  // Cost-balanced shard map (num_shards > 1): this shard's super-chunks as
  // chunk ranges [map_begin[k], map_end[k]) and the exclusive prefix of their
  // lengths map_pref[0..map_k] (the shard's queue position -> global chunk).
  const unsigned long long* map_begin;
  const unsigned long long* map_pref;
  uint32_t map_k;
  Counters* ctr;
  uint32_t* heavy_items;          // CTA-tier queue (kHeavyItemWords per item), may be null
  unsigned long long heavy_cap;
  uint32_t* heavy_scratch;        // CTA-tier node scratch (nslots * cap per CTA)
  uint32_t* local_rows;           // clique-local rows, warp tier (per warp), or null
  uint32_t* warp_bitmaps;         // per-warp id bitmaps (bitmap_words each, kept zero), or null
  uint64_t bitmap_words;
  uint32_t* heavy_rows;           // clique-local rows, CTA tier (per CTA)
  Program prog;
};

struct WarpState {
  uint32_t vals[kMaxLevels];
  const uint32_t* ptr[kMaxNodes];
  uint32_t len[kMaxNodes];
};

// lower_bound on a sorted list (branchless; all lanes may call it).
__device__ __forceinline__ uint32_t lower_bound_dev(const uint32_t* __restrict__ a, uint32_t n,
                                                    uint32_t x) {
  if (n == 0) return 0;
  const uint32_t* base = a;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (__ldg(base + half) < x) ? base + half : base;
    n -= half;
  }
  return static_cast<uint32_t>(base - a) + (__ldg(base) < x ? 1u : 0u);
}

// Membership in a sorted list: the last element <= x is the candidate.
__device__ __forceinline__ bool contains_dev(const uint32_t* __restrict__ a, uint32_t n,
                                             uint32_t x) {
  if (n == 0) return false;
  const uint32_t* base = a;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (__ldg(base + half) <= x) ? base + half : base;
    n -= half;
  }
  return __ldg(base) == x;
}

// Same, for lists written earlier in this kernel (scratch): plain loads.
__device__ __forceinline__ bool contains_rw(const uint32_t* a, uint32_t n, uint32_t x) {
  if (n == 0) return false;
  const uint32_t* base = a;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (base[half] <= x) ? base + half : base;
    n -= half;
  }
  return *base == x;
}

__device__ __forceinline__ uint32_t lower_bound_rw(const uint32_t* a, uint32_t n, uint32_t x) {
  if (n == 0) return 0;
  const uint32_t* base = a;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (base[half] < x) ? base + half : base;
    n -= half;
  }
  return static_cast<uint32_t>(base - a) + (*base < x ? 1u : 0u);
}

// Warp-cooperative lower_bound for a warp-uniform query (every lane gets the
// answer): a 32-ary search, one round of 32 independent pivot loads + ballot
// per factor of 32 (64K-element list: 3 rounds + 1) instead of a 16-step
// chain of dependent loads.  All 32 lanes must call it.  LDG: read-only
// (CSR) data through the non-coherent path.
template <bool LDG>
__device__ __forceinline__ uint32_t warp_lower_bound(const uint32_t* a, uint32_t n, uint32_t x) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t idx = min(lo + (lane + 1) * step - 1, hi - 1);
    const uint32_t v = LDG ? __ldg(a + idx) : a[idx];
    const int cnt = __popc(__ballot_sync(0xffffffffu, v < x));  // pivots below x (a prefix)
    const uint32_t nlo = cnt ? min(lo + cnt * step, hi) : lo;
    const uint32_t nhi = cnt < 32 ? min(lo + (cnt + 1) * step - 1, hi - 1) : hi;
    lo = nlo;
    hi = max(nhi, nlo);
  }
  const uint32_t idx = lo + lane;
  const bool lt = idx < hi && (LDG ? __ldg(a + idx) : a[idx]) < x;
  return lo + __popc(__ballot_sync(0xffffffffu, lt));
}

// CTA-cooperative version (all threads of the block must call it; contains
// barriers): a blockDim-ary search, e.g. 2 rounds for a 64K-element list.
template <bool LDG>
__device__ __forceinline__ uint32_t cta_lower_bound(const uint32_t* a, uint32_t n, uint32_t x) {
  const uint32_t nt = blockDim.x, t = threadIdx.x;
  uint32_t lo = 0, hi = n;
  while (hi - lo > nt) {
    const uint32_t step = (hi - lo + nt - 1) / nt;
    const uint32_t idx = min(lo + (t + 1) * step - 1, hi - 1);
    const uint32_t v = LDG ? __ldg(a + idx) : a[idx];
    const uint32_t cnt = __syncthreads_count(v < x);
    const uint32_t nlo = cnt ? min(lo + cnt * step, hi) : lo;
    const uint32_t nhi = cnt < nt ? min(lo + (cnt + 1) * step - 1, hi - 1) : hi;
    lo = nlo;
    hi = max(nhi, nlo);
  }
  const uint32_t idx = lo + t;
  const bool lt = idx < hi && (LDG ? __ldg(a + idx) : a[idx]) < x;
  return lo + __syncthreads_count(lt);
}

// Window ends of a sorted neighbour list without a bisection chain.  Ids are
// spread evenly over a list's value range (the configs permute ids), so the
// rank of a bound is predicted from the end values; one load at the
// prediction minus (plus) a margin of a few standard deviations proves a
// safe index, and only a failed check falls back to bisection.  The returned
// window may include a few elements outside [lo, hi): callers filter each
// element against the window anyway.
//   window_start: i with a[j] < lo for all j < i  (requires a[0] < lo)
//   window_end:   e with a[j] >= hi for all j >= e (requires a[n-1] >= hi)
__device__ __forceinline__ uint32_t guess_margin(uint32_t n) {
  return 8u + 2u * static_cast<uint32_t>(sqrtf(static_cast<float>(n)));
}

__device__ __forceinline__ uint32_t window_start(const uint32_t* a, uint32_t n, uint32_t first,
                                                 uint32_t last, uint32_t lo) {
  const float f = static_cast<float>(lo - first) / (static_cast<float>(last - first) + 1.f);
  const uint32_t g = static_cast<uint32_t>(f * static_cast<float>(n));
  const uint32_t m = guess_margin(n);
  if (g <= m) return 0u;
  const uint32_t i = g - m;
  if (__ldg(a + i) < lo) return i;
  return lower_bound_dev(a, i, lo);
}

__device__ __forceinline__ uint32_t window_end(const uint32_t* a, uint32_t n, uint32_t first,
                                               uint32_t last, uint32_t hi) {
  const float f = static_cast<float>(hi - first) / (static_cast<float>(last - first) + 1.f);
  const uint32_t g = static_cast<uint32_t>(f * static_cast<float>(n));
  const uint32_t e = g + guess_margin(n);
  if (e >= n - 1) return n;
  if (__ldg(a + e) >= hi) return e;
  return e + 1 + lower_bound_dev(a + e + 1, n - e - 1, hi);
}

struct Ctx {
  const unsigned long long* __restrict__ off;
  const uint32_t* __restrict__ adj;
  WarpState* s;
  uint32_t* scratch;
  uint64_t cap;
  uint32_t* hash;
  int lane;
  float nv;  // number of vertices (id range), for window-fraction estimates
  uint32_t tune;
  uint32_t heavy_stream;  // defer batches streaming at least this many elements (0: off)
  uint32_t heavy_min;     // defer big-probe-set batches only above this streamed degree sum
  uint32_t* gbm;          // this warp's global bitmap over all ids (zero between uses), or null
  uint32_t gbm_words;     // its size in words
  uint32_t hslots;        // slots of `hash` (power of two)
  float list_cost;        // per-list setup cost of a stream, in elements (side choice)
};

__device__ __forceinline__ void nbrs(const Ctx& c, uint32_t v, const uint32_t*& p, uint32_t& len) {
  const unsigned long long b = __ldg(c.off + v);
  const unsigned long long e = __ldg(c.off + v + 1);
  p = c.adj + b;
  len = static_cast<uint32_t>(e - b);
}

// ------------------------------------------------------------ set ops ---
// Every set operation streams one sorted list with coalesced, unrolled warp
// loads and tests membership in the other operand through a ProbeSet: a
// shared-memory hash table when the operand is small enough (build cost
// |operand| inserts, probe ~1-2 LDS), else a branchless binary search.  The
// side to stream and the probe structure are chosen per pair from the two
// lengths: tiny-vs-large pairs (hub lists) binary-search the few elements;
// comparable or moderately skewed pairs hash the smaller side and stream the
// larger.  Bounds arrive as prefix truncations (set_ops.hpp:20-25).

struct ProbeSet {
  const uint32_t* arr;  // sorted (scratch or CSR slice)
  uint32_t n;
  uint32_t lo, hi;      // arr[0], arr[n-1]
  uint32_t* hash;       // shared-memory table, valid when bits > 0
  int bits;
  const uint32_t* bm;   // CTA tier: bitmap of the set over ids [bm_base, bm_base + kBitmapSpan)
  uint32_t bm_base;
};

// The table is bucketised: a key hashes to a bucket of 4 consecutive slots
// (one 16-byte LDS.128), buckets fill in slot order and overflow linearly
// into the next bucket only when full, so a lookup stops at the first bucket
// whose last slot is empty.  At load <= 1/2 nearly every lookup (hit or
// miss) is one LDS.128, and the warp no longer waits for the longest of 32
// linear-probe chains.
__device__ __forceinline__ uint32_t hbucket(uint32_t x, int bbits) {
  return (x * 0x9E3779B1u) >> (32 - bbits);
}

__device__ __forceinline__ bool probe(const ProbeSet& P, uint32_t y) {
  if (P.bits < 0) {
    if (P.bits == -1)  // the warp's global (L2-resident) bitmap; L1 bypassed, it is rewritten per batch
      return (__ldcg(P.hash + (y >> 5)) >> (y & 31)) & 1u;
    // radix index over the sorted P (see leaf_batch)
    if (y < P.lo || y > P.hi) return false;
    const uint32_t b = (y - P.lo) >> P.bm_base;
    uint32_t i = __ldcg(P.hash + b);
    const uint32_t e = __ldcg(P.hash + b + 1);
    for (; i < e; ++i) {
      const uint32_t v = P.arr[i];
      if (v >= y) return v == y;
    }
    return false;
  }
  if (P.bits) {
    const int bbits = P.bits - 2;
    const uint32_t mask = (1u << bbits) - 1u;
    const uint4* tb = reinterpret_cast<const uint4*>(P.hash);
    uint32_t h = hbucket(y, bbits);
    for (;;) {
      const uint4 q = tb[h];
      if (q.x == y || q.y == y || q.z == y || q.w == y) return true;
      if (q.w == kEmptySlot) return false;
      h = (h + 1) & mask;
    }
  }
  return contains_rw(P.arr, P.n, y);
}

__device__ __forceinline__ int table_bits(uint32_t n) {
  int bits = 6;
  while ((1u << bits) < 2 * n) ++bits;
  return bits;
}

// Cooperative table fill by threads [tid, tid+nthreads); the caller syncs
// between the two phases and after.  Requires 2 * P.n <= table capacity.
__device__ __forceinline__ void fill_table(uint32_t* table, const ProbeSet& P, int tid,
                                           int nthreads) {
  const uint32_t nb = 1u << (P.bits - 2);
  uint4* tb = reinterpret_cast<uint4*>(table);
  for (uint32_t i = tid; i < nb; i += nthreads) tb[i] = make_uint4(kEmptySlot, kEmptySlot, kEmptySlot, kEmptySlot);
}

__device__ __forceinline__ void insert_table(uint32_t* table, const ProbeSet& P, int tid,
                                             int nthreads) {
  const int bbits = P.bits - 2;
  const uint32_t mask = (1u << bbits) - 1u;
  for (uint32_t i = tid; i < P.n; i += nthreads) {
    const uint32_t key = P.arr[i];
    uint32_t h = hbucket(key, bbits);
    for (;;) {
      uint32_t* bk = table + 4 * h;
      if (atomicCAS(bk, kEmptySlot, key) == kEmptySlot || atomicCAS(bk + 1, kEmptySlot, key) == kEmptySlot ||
          atomicCAS(bk + 2, kEmptySlot, key) == kEmptySlot || atomicCAS(bk + 3, kEmptySlot, key) == kEmptySlot)
        break;
      h = (h + 1) & mask;
    }
  }
}

// A ProbeSet over arr[0..n) (n > 0): hashed into the warp's table if it fits
// and `hash` is requested, else binary search.
__device__ __forceinline__ ProbeSet make_probe(const Ctx& c, const uint32_t* arr, uint32_t n,
                                               bool hash) {
  ProbeSet p;
  p.arr = arr;
  p.n = n;
  p.lo = arr[0];
  p.hi = arr[n - 1];
  p.hash = c.hash;
  p.bits = 0;
  if (hash && 2 * n <= c.hslots) {
    p.bits = table_bits(n);
    __syncwarp();
    fill_table(c.hash, p, c.lane, 32);
    __syncwarp();
    insert_table(c.hash, p, c.lane, 32);
    __syncwarp();
  }
  return p;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;  // every lane holds the sum
}

constexpr int kUnroll = 4;  // independent loads in flight per lane

__device__ __forceinline__ int ilog2p1(uint32_t x) { return 32 - __clz(x | 1u); }

// Hash the small side and stream the large one, or binary-search the small
// side into the large one?  Per-warp cycle model: a binary-search round costs
// ~log2(large) dependent loads, a stream iteration ~one load latency per
// 32*kUnroll elements.
__device__ __forceinline__ bool prefer_stream(uint32_t small, uint32_t large, uint32_t hslots) {
  if (small * 2 > hslots) return false;
  const uint64_t bs = static_cast<uint64_t>((small + 31) / 32) * ilog2p1(large);
  const uint64_t st = (large + 32 * kUnroll - 1) / (32 * kUnroll) + (small + 31) / 32;
  return st < bs;
}

// Stream X[0..nX), keep x iff (x in Pr) == keep_found and x != exclude.
// COUNT: return the number kept; else also write them, in order, to out.
template <bool COUNT, int U = kUnroll>
__device__ uint32_t filter_list(const Ctx& c, const uint32_t* X, uint32_t nX, const ProbeSet& Pr,
                                bool keep_found, uint32_t exclude, uint32_t* out) {
  const unsigned lt_mask = (1u << c.lane) - 1u;
  uint32_t written = 0;
  for (uint32_t base = 0; base < nX; base += 32 * U) {
    uint32_t x[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = base + u * 32 + c.lane;
      ok[u] = i < nX;
      x[u] = ok[u] ? X[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bool keep = ok[u] && x[u] != exclude;
      if (keep) keep = probe(Pr, x[u]) == keep_found;
      const unsigned m = __ballot_sync(kFull, keep);
      if (!COUNT && keep) out[written + __popc(m & lt_mask)] = x[u];
      written += __popc(m);
    }
  }
  return written;
}

// Apply a node's ops to the input set `in` (sorted, already bounded).
// COUNT: return |result| only; else write the sorted result to `out`.
template <bool COUNT>
__device__ uint32_t apply_ops(const Ctx& c, const Node& nd, const uint32_t* in, uint32_t inlen,
                              uint32_t* out) {
  const WarpState& s = *c.s;
  if (inlen == 0) return 0;
  if (nd.nops == 1) {
    // Choose the streamed list X and the probe structure, then one filter
    // pass (a single call site keeps the inlined probe loops small).
    const uint32_t v = s.vals[nd.ops[0].level];
    const uint32_t* L;
    uint32_t nL;
    nbrs(c, v, L, nL);
    const uint32_t* X = in;
    uint32_t nX = inlen;
    const uint32_t* Q = L;  // probe set (sorted)
    uint32_t nQ = 0;
    bool keep_found = true, use_hash = false;
    uint32_t exclude = kEmptySlot;
    if (nd.ops[0].mode == kOpIsect) {
      if (nd.bound >= 0) nL = warp_lower_bound<true>(L, nL, s.vals[nd.bound]);
      if (nL == 0) return 0;
      // result = in & L; iterate either side (both sorted -> sorted output)
      const bool in_small = inlen <= nL;
      const uint32_t* Sm = in_small ? in : L;
      const uint32_t nSm = in_small ? inlen : nL;
      const uint32_t* Lg = in_small ? L : in;
      const uint32_t nLg = in_small ? nL : inlen;
      if (prefer_stream(nSm, nLg, c.hslots)) {
        X = Lg, nX = nLg, Q = Sm, nQ = nSm, use_hash = true;
      } else {
        X = Sm, nX = nSm, Q = Lg, nQ = nLg;  // bisection into the large side
      }
    } else {
      // result = in - N[v]: stream `in`; only N(v) within [in.lo, in.hi] matters
      keep_found = false;
      exclude = v;
      const uint32_t lo = in[0], hi = in[inlen - 1];
      const uint32_t wa = warp_lower_bound<true>(L, nL, lo);
      const uint32_t wb = wa + warp_lower_bound<true>(L + wa, nL - wa, hi + 1u);
      Q = L + wa;
      nQ = wb - wa;
      use_hash = nQ && 2 * nQ <= c.hslots && nQ <= 8u * inlen;
    }
    // (A global-bitmap probe set for big node operands was measured slower
    // than bisection here: +4-7 % on cfg2; it stays on the leaf batches.)
    ProbeSet pr;
    if (nQ) {
      pr = make_probe(c, Q, nQ, use_hash);
    } else {
      pr.arr = Q;
      pr.n = 0;
      pr.bits = 0;
    }
    return filter_list<COUNT>(c, X, nX, pr, keep_found, exclude, out);
  }
  // Several ops (a start node with earlier differences): binary-search all.
  const unsigned lt_mask = (1u << c.lane) - 1u;
  const uint32_t* opp[kMaxOps];
  uint32_t opl[kMaxOps];
  uint32_t opv[kMaxOps];
  for (int o = 0; o < nd.nops; ++o) {
    opv[o] = s.vals[nd.ops[o].level];
    nbrs(c, opv[o], opp[o], opl[o]);
  }
  uint32_t written = 0;
  for (uint32_t base = 0; base < inlen; base += 32) {
    const uint32_t i = base + c.lane;
    bool keep = i < inlen;
    const uint32_t x = keep ? in[i] : 0u;
    for (int o = 0; o < nd.nops; ++o) {
      if (keep) {
        const bool f = contains_dev(opp[o], opl[o], x);
        keep = (nd.ops[o].mode == kOpIsect) ? f : (!f && x != opv[o]);
      }
    }
    const unsigned m = __ballot_sync(kFull, keep);
    if (!COUNT && keep) out[written + __popc(m & lt_mask)] = x;
    written += __popc(m);
  }
  return written;
}

// Resolve a node's input set (source node or raw list), bounded.
__device__ __forceinline__ void node_input(const Ctx& c, const Node& nd, const uint32_t*& in,
                                           uint32_t& inlen) {
  const WarpState& s = *c.s;
  if (nd.src >= 0) {
    in = s.ptr[nd.src];
    inlen = s.len[nd.src];
  } else {
    nbrs(c, s.vals[nd.list], in, inlen);
  }
  if (nd.bound >= 0) inlen = warp_lower_bound<false>(in, inlen, s.vals[nd.bound]);
}

// CTA tier: the same, with a block-cooperative search (all threads call it).
__device__ __forceinline__ void node_input_cta(const Ctx& c, const Node& nd, const uint32_t*& in,
                                               uint32_t& inlen) {
  const WarpState& s = *c.s;
  if (nd.src >= 0) {
    in = s.ptr[nd.src];
    inlen = s.len[nd.src];
  } else {
    nbrs(c, s.vals[nd.list], in, inlen);
  }
  if (nd.bound >= 0) inlen = cta_lower_bound<false>(in, inlen, s.vals[nd.bound]);
}

__device__ void build_node(const Ctx& c, const Program& P, int t) {
  const Node& nd = P.nodes[t];
  const uint32_t* in;
  uint32_t inlen;
  node_input(c, nd, in, inlen);
  uint32_t len = inlen;
  const uint32_t* ptr = in;
  if (!nd.raw) {
    uint32_t* out = c.scratch + static_cast<uint64_t>(nd.slot) * c.cap;
    len = apply_ops<false>(c, nd, in, inlen, out);
    ptr = out;
  }
  __syncwarp();
  if (c.lane == 0) {
    c.s->ptr[t] = ptr;
    c.s->len[t] = len;
  }
  __syncwarp();
}

__device__ __forceinline__ uint32_t leaf_count(const Ctx& c, const Program& P) {
  const uint32_t* in;
  uint32_t inlen;
  node_input(c, P.leaf, in, inlen);
  if (P.leaf.raw) return inlen;
  return apply_ops<true>(c, P.leaf, in, inlen, nullptr);
}

// E contribution of building level i from the current prefix v_0..v_{i-1}:
// sum over sources j < i of |{x in N(v_j) : x < beta_i}|.
__device__ __forceinline__ uint64_t meter_level(const Ctx& c, const Program& P, int i) {
  uint32_t term = 0;
  if (c.lane < i) {
    const uint32_t* p;
    uint32_t len;
    nbrs(c, c.s->vals[c.lane], p, len);
    const int par = P.parent[i];
    term = (par >= 0) ? lower_bound_dev(p, len, c.s->vals[par]) : len;
  }
  return __reduce_add_sync(kFull, term);
}

// E of all leaf builds of a batch: for every sibling x in C_{n-2}, level n-1 is
// built from v_0..v_{n-3}, x with bound beta (v_p, x itself, or none).
__device__ uint64_t meter_batch(const Ctx& c, const Program& P) {
  const WarpState& s = *c.s;
  const int n = P.depth;
  const int an = P.cand[n - 2];
  const uint32_t* A = s.ptr[an];
  const uint32_t nA = s.len[an];
  const int par = P.parent[n - 1];
  uint64_t acc = 0;
  for (uint32_t i = c.lane; i < nA; i += 32) {
    const uint32_t x = A[i];
    const bool unbounded = par < 0;
    const uint32_t beta = par < 0 ? 0u : (par == n - 2 ? x : s.vals[par]);
    for (int j = 0; j <= n - 2; ++j) {
      const uint32_t v = j == n - 2 ? x : s.vals[j];
      const uint32_t* p;
      uint32_t len;
      nbrs(c, v, p, len);
      acc += unbounded ? len : lower_bound_dev(p, len, beta);
    }
  }
  return warp_sum64(acc);
}

__device__ __forceinline__ void checked_acc(uint64_t& acc, uint64_t add, bool& ovf) {
  const uint64_t r = acc + add;
  ovf |= (r < acc);
  acc = r;
}

// ------------------------------------------------------- leaf batching ---
// With the leaf  C_{n-1}(x) = B (op) N(x)  for every sibling x in A = C_{n-2},
// the sum of the leaf counts over all siblings is an edge count between two
// vertex sets:  sum_{x in A} |B & N(x) & [0, beta_x)|  (= sum_{y in B} |A & N(y)|,
// the adjacency is symmetric).  One side is put in a shared-memory hash (the
// probe set P) and the neighbour lists of the other side S are streamed with
// coalesced, load-balanced warp loads; for skewed pairs (a hub s and a small
// P) the elements of P are binary-searched into N(s) instead.  The side is
// chosen per batch from the degree sums.  Differences use
// |B - N[x]| = |B| - |B & N(x)| - [x in B].
//
// Two tiers: a batch whose probe set fits the per-warp table (kHashSlots) runs
// in the warp that found it; a bigger one with real streaming work is queued
// (its prefix v_0..v_{n-3}) for heavy_kernel, where a whole CTA shares a
// 64 KB table and streams the lists with all its warps.

constexpr uint32_t kLongList = 64;  // lists this long are streamed by the whole warp

// sum_{s in S} |{p in P : p in N(s)}| with rel: 0 none, 1 p < s, 2 p > s, over
// the groups of 32 elements of S starting at g_first with stride g_stride.
// Each lane resolves one s and the value window [lo, hi) of P (and the rel
// bound).  Long lists are then streamed one at a time by the whole warp
// (coalesced, kUnroll loads in flight per lane, early exit at hi -- sorted
// lists need no upper-bound search, and the lower one only when the list
// starts below lo); short lists are flattened across the lanes; skewed pairs
// (|P| log |N(s)| << |N(s)|) binary-search P into N(s).  Returns this warp's
// partial (all lanes hold it).
// One long list streamed by the whole warp: KU coalesced loads in flight per
// lane, window [lo, hi), early exit once the sorted list passes hi.
template <int KU>
__device__ __forceinline__ uint32_t stream_long(const Ctx& c, const uint32_t* jp, uint32_t jl, uint32_t jlo,
                                                uint32_t jhi, const ProbeSet& P, uint64_t* tr) {
  uint32_t hits = 0;
  for (uint32_t t0 = 0; t0 < jl; t0 += 32 * KU) {
    uint32_t y[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint32_t idx = t0 + u * 32 + c.lane;
      y[u] = idx < jl ? __ldg(jp + idx) : kEmptySlot;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u)
      if (y[u] < jhi && y[u] >= jlo && probe(P, y[u])) ++hits;
    if (__any_sync(kFull, y[KU - 1] >= jhi)) break;  // sorted: the rest is >= hi
  }
  return hits;
}

template <bool TRACE>
__device__ uint64_t stream_count(const Ctx& c, const uint32_t* S, uint32_t nS, const ProbeSet& P,
                                 int rel, uint32_t g_first, uint32_t g_stride, uint64_t* tr) {
  uint64_t total = 0;
  for (uint32_t g0 = g_first; g0 < nS; g0 += g_stride) {
    const uint32_t i = g0 + c.lane;
    uint32_t start = 0, len = 0, lo_val = P.lo, hi_val = P.hi + 1u;
    const uint32_t* base = c.adj;
    bool is_long = false, search = false;
    if (i < nS) {
      const uint32_t s = S[i];
      if (rel == 1) hi_val = min(hi_val, s);
      if (rel == 2) lo_val = max(lo_val, s + 1u);
      const unsigned long long b = __ldg(c.off + s), e = __ldg(c.off + s + 1);
      base = c.adj + b;
      const uint32_t deg = static_cast<uint32_t>(e - b);
      if (lo_val < hi_val && deg) {
        const uint32_t first = __ldg(base), last = __ldg(base + deg - 1);
        if (last >= lo_val && first < hi_val) {
          len = deg;
          if (deg >= kLongList) {
            is_long = true;
            // lower window end by binary search only when the part below it
            // is a sizeable fraction of the list (else it is streamed and
            // filtered; ids spread evenly over a list's value range)
            if (first < lo_val && ((c.tune & 16u) ||
                static_cast<float>(lo_val - first) > (static_cast<float>(last - first) + 1.f) * 0.0625f))
              start = window_start(base, deg, first, last, lo_val);
            len = deg - start;
            search = static_cast<uint64_t>(P.n) * ilog2p1(len) * 2u < len;
            is_long = !search;
          }
        }
      }
    }
    uint32_t hits = 0;
    // 1) long lists: one at a time, whole warp, early exit at hi
    unsigned lm = __ballot_sync(kFull, is_long);
    if (TRACE) {
      tr[kTrSearchLists] += __popc(__ballot_sync(kFull, search));
      tr[kTrLongLists] += __popc(lm);
    }
    while (lm) {
      const int j = __ffs(lm) - 1;
      lm &= lm - 1;
      const uint32_t* jp = reinterpret_cast<const uint32_t*>(
                               __shfl_sync(kFull, reinterpret_cast<unsigned long long>(base), j)) +
                           __shfl_sync(kFull, start, j);
      const uint32_t jl = __shfl_sync(kFull, len, j);
      const uint32_t jlo = __shfl_sync(kFull, lo_val, j);
      const uint32_t jhi = __shfl_sync(kFull, hi_val, j);
      if (TRACE && c.lane == 0) tr[kTrStreamElems] += jl;  // upper bound (early exit)
      hits += stream_long<kUnroll>(c, jp, jl, jlo, jhi, P, tr);
    }
    // 2) short lists: flattened over the lanes, range-filtered per element
    const uint32_t slen = is_long || search ? 0u : len;
    const uint32_t incl = warp_incl_scan(slen, c.lane);
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - slen;
    if (TRACE) tr[kTrStreamElems] += tot;
    for (uint32_t t = 0; t < tot; t += 64) {
      uint32_t y[2], ylo[2], yhi[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t idx = t + u * 32 + c.lane;
        int j = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const uint32_t ex = __shfl_sync(kFull, excl, j + step);
          if (ex <= idx) j += step;
        }
        const uint32_t o_excl = __shfl_sync(kFull, excl, j);
        ylo[u] = __shfl_sync(kFull, lo_val, j);
        yhi[u] = __shfl_sync(kFull, hi_val, j);
        const uint32_t* o_base = reinterpret_cast<const uint32_t*>(
            __shfl_sync(kFull, reinterpret_cast<unsigned long long>(base), j));
        y[u] = idx < tot ? __ldg(o_base + (idx - o_excl)) : kEmptySlot;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (y[u] >= ylo[u] && y[u] < yhi[u] && probe(P, y[u])) ++hits;
    }
    // 3) skewed pairs: the (list, element of P's window) pairs are flattened
    //    over the lanes; every lane binary-searches one element into its list
    uint32_t pa = 0, npairs = 0;
    if (search) {
      pa = lower_bound_rw(P.arr, P.n, lo_val);
      npairs = lower_bound_rw(P.arr, P.n, hi_val) - pa;
    }
    const uint32_t pincl = warp_incl_scan(npairs, c.lane);
    const uint32_t ptot = __shfl_sync(kFull, pincl, 31);
    const uint32_t pexcl = pincl - npairs;
    for (uint32_t t = 0; t < ptot; t += 32) {
      const uint32_t idx = t + c.lane;
      int j = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t ex = __shfl_sync(kFull, pexcl, j + step);
        if (ex <= idx) j += step;
      }
      const uint32_t o_pa = __shfl_sync(kFull, pa, j);
      const uint32_t o_ex = __shfl_sync(kFull, pexcl, j);
      const uint32_t o_len = __shfl_sync(kFull, len, j);
      const uint32_t* o_list = reinterpret_cast<const uint32_t*>(
                                   __shfl_sync(kFull, reinterpret_cast<unsigned long long>(base), j)) +
                               __shfl_sync(kFull, start, j);
      if (idx < ptot) {
        const uint32_t key = P.arr[o_pa + (idx - o_ex)];
        if (contains_dev(o_list, o_len, key)) ++hits;
      }
    }
    total += hits;
  }
  return warp_sum64(total);
}

// Sum of deg over X[g_first + lane], stride (partial; all lanes hold it).
__device__ __forceinline__ uint64_t degree_sum(const Ctx& c, const uint32_t* X, uint32_t n,
                                               uint32_t first, uint32_t stride) {
  uint64_t acc = 0;
  uint32_t i = first + c.lane;
  for (; i + 3 * stride < n; i += 4 * stride) {  // four lists' offsets in flight
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = X[i + k * stride];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += __ldg(c.off + v[k] + 1) - __ldg(c.off + v[k]);
  }
  for (; i < n; i += stride) {
    const uint32_t v = X[i];
    acc += __ldg(c.off + v + 1) - __ldg(c.off + v);
  }
  return warp_sum64(acc);
}

// The batch's two sets (see above), from the warp's current state.
struct BatchSets {
  const uint32_t* A;
  uint32_t nA;
  const uint32_t* B;
  uint32_t nB;
  bool same;
};

__device__ __forceinline__ BatchSets batch_sets(const WarpState& s, const Program& P) {
  BatchSets b;
  const int an = P.cand[P.depth - 2];
  const int bn = P.leaf.src;
  b.A = s.ptr[an];
  b.nA = s.len[an];
  b.B = s.ptr[bn];
  b.nB = s.len[bn];
  if (P.batch_fixed_bound >= 0) b.nB = warp_lower_bound<false>(b.B, b.nB, s.vals[P.batch_fixed_bound]);
  b.same = an == bn;
  return b;
}

// DIFF leaves: sum_x |{y in B : y < beta_x}| - [x in B, x < beta_x]; warp partial.
__device__ uint64_t diff_terms(const Ctx& c, const Program& P, const BatchSets& b, uint32_t first,
                               uint32_t stride, bool add_product) {
  uint64_t t = 0;
  if (P.batch_yltx) {
    for (uint32_t i = first + c.lane; i < b.nA; i += stride) t += lower_bound_rw(b.B, b.nB, b.A[i]);
    return warp_sum64(t);
  }
  uint64_t hits = 0;
  for (uint32_t i = first + c.lane; i < b.nA; i += stride) hits += contains_rw(b.B, b.nB, b.A[i]) ? 1u : 0u;
  hits = warp_sum64(hits);
  return (add_product ? static_cast<uint64_t>(b.nA) * b.nB : 0ull) - hits;
}

// Which side to stream: only the part of each streamed list inside the other
// set's value window is read, so weigh each side's degree sum by the width of
// the window it is clipped to (ids are unordered w.r.t. degree, so a list
// spreads roughly uniformly over the id range).
// Each streamed list also pays a fixed setup (offsets, window search, a
// warp-serial pass for long lists), ~kListCost elements' worth.
constexpr float kListCost = 384.f;  // default of Ctx::list_cost (SMG_LIST_COST); measured 16..4096
__device__ __forceinline__ bool stream_b_cheaper(const Ctx& c, const BatchSets& b, uint64_t deg_a,
                                                 uint64_t deg_b) {
  if (c.tune & 1u) return deg_b < deg_a;
  const float wa = fminf(1.f, (static_cast<float>(b.A[b.nA - 1] - b.A[0]) + 1.f) / c.nv);
  const float wb = fminf(1.f, (static_cast<float>(b.B[b.nB - 1] - b.B[0]) + 1.f) / c.nv);
  const float cost_a = c.list_cost * b.nA + static_cast<float>(deg_a) * wb;  // stream A's lists
  const float cost_b = c.list_cost * b.nB + static_cast<float>(deg_b) * wa;
  return cost_b < cost_a;
}

// Side choice with a lazy degree sum: the smaller set's degree sum first; the
// larger set's cost is at least kListCost + 1 window element per list, and
// when that bound already loses its degree sum (a long, latency-bound loop
// for hub-sized sets) is skipped.  `dsum(X, n)` returns the full degree sum
// of X[0..n) on every participating thread.  Returns flip (= stream B) and
// the streamed side's degree sum.
template <class DegSum>
__device__ __forceinline__ bool choose_stream_b(const Ctx& c, const BatchSets& b, DegSum dsum,
                                                uint64_t& sum_s) {
  const bool a_small = b.nA <= b.nB;
  const uint32_t* X = a_small ? b.A : b.B;
  const uint32_t nX = a_small ? b.nA : b.nB;
  const uint32_t nY = a_small ? b.nB : b.nA;
  const uint64_t dx = dsum(X, nX);
  if (!(c.tune & 1u)) {
    const float wa = fminf(1.f, (static_cast<float>(b.A[b.nA - 1] - b.A[0]) + 1.f) / c.nv);
    const float wb = fminf(1.f, (static_cast<float>(b.B[b.nB - 1] - b.B[0]) + 1.f) / c.nv);
    const float wx = a_small ? wb : wa, wy = a_small ? wa : wb;  // window the other side clips to
    const float cost_x = c.list_cost * nX + static_cast<float>(dx) * wx;
    const float cost_y_min = (c.list_cost + wy) * nY;
    if (cost_y_min >= cost_x) {
      sum_s = dx;
      return !a_small;
    }
  }
  const uint64_t dy = dsum(a_small ? b.B : b.A, nY);
  const bool flip = stream_b_cheaper(c, b, a_small ? dx : dy, a_small ? dy : dx);
  sum_s = flip ? (a_small ? dy : dx) : (a_small ? dx : dy);
  return flip;
}

struct HeavyQueue {
  uint32_t* items;          // kHeavyItemWords per item
  unsigned long long cap;
  unsigned long long* count;
};
constexpr int kHeavyItemWords = 6;  // v_0 .. v_{n-3}, n <= 8
constexpr uint32_t kCliqueItem = 0xffffffffu;  // last word of a clique-local item (never an id)

// Warp tier.  Returns the batch total, or defers it to the heavy queue.
template <bool TRACE>
__device__ uint64_t leaf_batch(const Ctx& c, const Program& P, const HeavyQueue& hq, uint64_t* tr) {
  const WarpState& s = *c.s;
  const BatchSets b = batch_sets(s, P);
  if (b.nA == 0) return 0;
  const bool yltx = P.batch_yltx != 0;
  uint64_t core = 0;
  if (b.nB) {
    bool flip = false;
    uint64_t sum_s;
    if (b.same) {
      sum_s = 0;
    } else {
      flip = choose_stream_b(c, b, [&](const uint32_t* X, uint32_t n) { return degree_sum(c, X, n, 0, 32); },
                             sum_s);
    }
    ProbeSet ps;
    ps.arr = flip ? b.A : b.B;
    ps.n = flip ? b.nA : b.nB;
    ps.lo = ps.arr[0];
    ps.hi = ps.arr[ps.n - 1];
    ps.hash = c.hash;
    ps.bits = 0;
    if (b.same && (ps.n * 2 > c.hslots || c.heavy_stream)) sum_s = degree_sum(c, b.A, b.nA, 0, 32);
    if (ps.n * 2 > c.hslots || (c.heavy_stream && sum_s >= c.heavy_stream)) {
      // Too big for the warp's table (or a long stream).  Queue it for the CTA
      // tier unless the streaming side is trivially small (then binary search
      // is cheaper).
      if (sum_s > c.heavy_min && hq.items) {
        unsigned long long slot = 0;
        if (c.lane == 0) slot = atomicAdd(hq.count, 1ull);
        slot = __shfl_sync(kFull, slot, 0);
        if (slot < hq.cap) {
          if (c.lane < P.depth - 2) hq.items[slot * kHeavyItemWords + c.lane] = s.vals[c.lane];
          else if (c.lane == kHeavyItemWords - 1) hq.items[slot * kHeavyItemWords + c.lane] = 0u;
          if (TRACE) tr[kTrDeferred] += 1;
          return 0;
        }
      }
    }
    bool global_bm = false;
    uint32_t radix_nb = 0;
    if (ps.n * 2 > c.hslots && c.gbm && !(c.tune & 512u)) {
      // Radix index over the sorted P (SMG_TUNE 512: a plain bitmap instead):
      // bucket b of width 2^k holds
      // P's positions [idx[b], idx[b+1]); ~2 elements per bucket, built in
      // one pass without atomics; ~6 bytes per element of P in L2 instead of
      // a 32-byte bitmap sector per element.
      const uint32_t span = ps.hi - ps.lo;
      int k = 0;
      while ((static_cast<uint64_t>(span >> k) + 2) * 2 > ps.n && (span >> k) > 0) ++k;
      radix_nb = (span >> k) + 2;
      if (radix_nb <= c.gbm_words) {
        uint32_t* idx = c.gbm;
        for (uint32_t i = c.lane; i < ps.n; i += 32) {
          const uint32_t bi = (ps.arr[i] - ps.lo) >> k;
          const uint32_t bp = i ? ((ps.arr[i - 1] - ps.lo) >> k) + 1 : 0u;
          for (uint32_t bb = bp; bb <= bi; ++bb) idx[bb] = i;
          if (i == ps.n - 1)
            for (uint32_t bb = bi + 1; bb < radix_nb; ++bb) idx[bb] = ps.n;
        }
        __syncwarp();
        ps.hash = idx;
        ps.bm_base = static_cast<uint32_t>(k);
        ps.bits = -3;
      } else {
        radix_nb = 0;
      }
    }
    if (ps.n * 2 > c.hslots && c.gbm && !radix_nb) {
      // Too big for the warp's smem table: a bitmap over all ids in global
      // memory (L2-resident words), one dependent load per probe instead of
      // a bisection chain; cleared again below.
      for (uint32_t i = c.lane; i < ps.n; i += 32) {
        const uint32_t x = ps.arr[i];
        atomicOr(c.gbm + (x >> 5), 1u << (x & 31));
      }
      __syncwarp();
      ps.hash = c.gbm;
      ps.bits = -1;
      global_bm = true;
    }
    if (ps.n * 2 <= c.hslots) {
      ps.bits = table_bits(ps.n);
      __syncwarp();
      fill_table(c.hash, ps, c.lane, 32);
      __syncwarp();
      insert_table(c.hash, ps, c.lane, 32);
      __syncwarp();
    }
    if (TRACE) {
      tr[kTrBatches] += 1;
      tr[kTrBatchesHashed] += ps.bits ? 1 : 0;
      tr[kTrProbeSetSum] += ps.n;
      tr[kTrStreamSetSum] += flip ? b.nB : b.nA;
    }
    long long t0 = TRACE ? clock64() : 0;
    core = stream_count<TRACE>(c, flip ? b.B : b.A, flip ? b.nB : b.nA, ps, yltx ? (flip ? 2 : 1) : 0, 0,
                               32, tr);
    if (global_bm) {
      __syncwarp();
      for (uint32_t i = c.lane; i < ps.n; i += 32) c.gbm[ps.arr[i] >> 5] = 0u;
      __syncwarp();
    }
    if (radix_nb) {
      __syncwarp();
      for (uint32_t i = c.lane; i < radix_nb; i += 32) c.gbm[i] = 0u;
      __syncwarp();
    }
    if (TRACE && !ps.bits) tr[kTrBigPCycles] += clock64() - t0;
  }
  if (!P.batch_diff) return core;
  return diff_terms(c, P, b, 0, 32, true) - core;
}

// ------------------------------------------------------------ clique-local ---
// Clique plans (no difference sources): every level >= 2 is a subset of
// U = N(v0) & N(v1).  Per unit the induced subgraph on U is built once as
// bitmap rows over U's local ids (local id = rank in sorted U, so value order
// = id order and every bound becomes a bit prefix), then the nested loops of
// levels 2..n-1 run as word-wise ANDs with a popcount leaf.  The reference
// re-merges full neighbour lists at every level of every prefix
// (engine.cpp:58-80); here each neighbour list is read once per unit.
// Warp tier: |U| <= kLocalWarpMax (one row word per lane); bigger units go to
// the CTA tier (heavy_kernel) with |U| <= kLocalCtaMax; beyond that the
// generic path runs.

constexpr uint32_t kLocalWarpMax = kHashSlots / 4;  // keys, index and row buffer fit the generic warp hash area
constexpr uint32_t kLocalCtaMax = 4096;
constexpr uint32_t kLocalCtaSlots = 2 * kLocalCtaMax;            // index table slots
constexpr uint32_t kLocalRowWords = kLocalCtaMax / 32;           // CTA row stride (words)
constexpr uint32_t kLocalWarpRowWords = kLocalWarpMax / 32;      // warp row stride (words)
constexpr size_t kHeavyCliqueSmem = kLocalCtaSlots * 4 + kLocalCtaSlots * 2 +
                                    kHeavyWarps * kLocalRowWords * 4;

struct LocalIndex {
  uint32_t* keys;   // bucketised like the probe tables
  uint16_t* idx;    // local id of the key in the same slot
  int bits;
};

// Build the value -> local id table for U[0..u) with threads [tid, tid+nth).
__device__ void local_index_build(LocalIndex& L, const uint32_t* U, uint32_t u, int tid, int nth,
                                  bool cta) {
  int bits = 6;
  while ((1u << bits) < 2 * u) ++bits;
  L.bits = bits;
  const uint32_t nb = 1u << (bits - 2);
  uint4* kb = reinterpret_cast<uint4*>(L.keys);
  if (cta) __syncthreads(); else __syncwarp();
  for (uint32_t i = tid; i < nb; i += nth) kb[i] = make_uint4(kEmptySlot, kEmptySlot, kEmptySlot, kEmptySlot);
  if (cta) __syncthreads(); else __syncwarp();
  const uint32_t mask = nb - 1u;
  for (uint32_t i = tid; i < u; i += nth) {
    const uint32_t key = U[i];
    uint32_t h = hbucket(key, bits - 2);
    for (;;) {
      uint32_t* bk = L.keys + 4 * h;
      int j = -1;
      if (atomicCAS(bk, kEmptySlot, key) == kEmptySlot) j = 0;
      else if (atomicCAS(bk + 1, kEmptySlot, key) == kEmptySlot) j = 1;
      else if (atomicCAS(bk + 2, kEmptySlot, key) == kEmptySlot) j = 2;
      else if (atomicCAS(bk + 3, kEmptySlot, key) == kEmptySlot) j = 3;
      if (j >= 0) {
        L.idx[4 * h + j] = static_cast<uint16_t>(i);
        break;
      }
      h = (h + 1) & mask;
    }
  }
  if (cta) __syncthreads(); else __syncwarp();
}

__device__ __forceinline__ int local_find(const LocalIndex& L, uint32_t y) {
  const int bbits = L.bits - 2;
  const uint32_t mask = (1u << bbits) - 1u;
  const uint4* kb = reinterpret_cast<const uint4*>(L.keys);
  uint32_t h = hbucket(y, bbits);
  for (;;) {
    const uint4 q = kb[h];
    if (q.x == y) return L.idx[4 * h];
    if (q.y == y) return L.idx[4 * h + 1];
    if (q.z == y) return L.idx[4 * h + 2];
    if (q.w == y) return L.idx[4 * h + 3];
    if (q.w == kEmptySlot) return -1;
    h = (h + 1) & mask;
  }
}

// Row a of the local graph: bits of N(U[a]) & U restricted to values in
// [U[0], hi) into rowbuf (nwords words, zeroed by the caller), then stored to
// row (coalesced).  One warp per row.
__device__ void local_row(const Ctx& c, const LocalIndex& L, const uint32_t* U, uint32_t u,
                          uint32_t a, bool lower_only, uint32_t* rowbuf, uint32_t nwords,
                          uint32_t* row) {
  const uint32_t x = U[a];
  const uint32_t lo = U[0];
  const uint32_t hi = lower_only ? x : U[u - 1] + 1u;
  const uint32_t* p;
  uint32_t deg;
  nbrs(c, x, p, deg);
  uint32_t start = 0;
  if (deg && lo < hi) {
    const uint32_t first = __ldg(p);
    if (first < lo) start = warp_lower_bound<true>(p, deg, lo);
    for (uint32_t t0 = start; t0 < deg; t0 += 32 * kUnroll) {
      uint32_t y[kUnroll];
#pragma unroll
      for (int k = 0; k < kUnroll; ++k) {
        const uint32_t i = t0 + k * 32 + c.lane;
        y[k] = i < deg ? __ldg(p + i) : kEmptySlot;
      }
#pragma unroll
      for (int k = 0; k < kUnroll; ++k) {
        if (y[k] < hi) {
          const int id = local_find(L, y[k]);
          if (id >= 0) atomicOr(&rowbuf[id >> 5], 1u << (id & 31));
        }
      }
      if (__any_sync(kFull, y[kUnroll - 1] >= hi)) break;
    }
  }
  __syncwarp();
  for (uint32_t w = c.lane; w < nwords; w += 32) {
    row[w] = rowbuf[w];
    rowbuf[w] = 0u;
  }
  __syncwarp();
}

// First set bit (ascending) of the WPL*32-word bitmap held as rem[k] in lane
// `lane` (word index k*32 + lane); clears it and returns its bit index, or -1.
template <int WPL>
__device__ __forceinline__ int local_pop_next(uint32_t (&rem)[WPL], int lane) {
#pragma unroll
  for (int k = 0; k < WPL; ++k) {
    const unsigned nz = __ballot_sync(kFull, rem[k] != 0u);
    if (nz) {
      const int f = __ffs(nz) - 1;
      const uint32_t w = __shfl_sync(kFull, rem[k], f);
      const int bit = __ffs(w) - 1;
      if (lane == f) rem[k] &= rem[k] - 1u;
      return (k * 32 + f) * 32 + bit;
    }
  }
  return -1;
}

template <int WPL>
__device__ __forceinline__ void prefix_mask(uint32_t q, int lane, uint32_t (&m)[WPL]) {
#pragma unroll
  for (int k = 0; k < WPL; ++k) {
    const uint32_t w0 = (k * 32 + lane) * 32u;
    m[k] = q >= w0 + 32u ? ~0u : (q <= w0 ? 0u : ((1u << (q - w0)) - 1u));
  }
}

// Levels 2..n-1 on the local graph (rows of `stride` words).  Level-2 ids
// are taken when (ordinal % a2_stride) == a2_first, so CTA warps can share a
// unit.  Returns this warp's count (all lanes hold it).
template <int WPL>
__device__ uint64_t local_dfs(const Ctx& c, const Program& P, const uint32_t* rows, uint32_t stride,
                              uint32_t u, uint32_t q0, uint32_t q1, uint32_t a2_first,
                              uint32_t a2_stride) {
  const int n = P.depth;
  const int lane = c.lane;
  uint32_t acc[kMaxLevels][WPL];
  uint32_t rem[kMaxLevels][WPL];
  int a[kMaxLevels] = {};
  auto bound_q = [&](int i) -> uint32_t {
    const int p = P.parent[i];
    return p < 0 ? u : (p == 0 ? q0 : (p == 1 ? q1 : static_cast<uint32_t>(a[p])));
  };
  uint32_t m[WPL];
  prefix_mask<WPL>(bound_q(2), lane, m);
#pragma unroll
  for (int k = 0; k < WPL; ++k) rem[2][k] = m[k];
  uint64_t total = 0;
  uint32_t ord2 = 0;
  int level = 2;
  while (level >= 2) {
    const int x = local_pop_next<WPL>(rem[level], lane);
    if (x < 0) {
      --level;
      continue;
    }
    if (level == 2 && (ord2++ % a2_stride) != a2_first) continue;
    a[level] = x;
    const uint32_t* row = rows + static_cast<uint64_t>(x) * stride;
    uint32_t nacc[WPL];
#pragma unroll
    for (int k = 0; k < WPL; ++k) {
      const uint32_t w = k * 32 + lane;
      const uint32_t r = w < stride ? row[w] : 0u;
      nacc[k] = level == 2 ? r : (acc[level][k] & r);
    }
    if (level + 1 == n - 1) {
      prefix_mask<WPL>(bound_q(n - 1), lane, m);
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < WPL; ++k) cnt += __popc(nacc[k] & m[k]);
      total += cnt;
    } else {
      ++level;
      prefix_mask<WPL>(bound_q(level), lane, m);
#pragma unroll
      for (int k = 0; k < WPL; ++k) {
        acc[level][k] = nacc[k];
        rem[level][k] = nacc[k] & m[k];
      }
    }
  }
  return warp_sum64(total);
}

// The universe U: the longest stored k=1 node (all are N(v0) & N(v1) bounded).
__device__ __forceinline__ int clique_universe(const WarpState& s, const Program& P) {
  int best = -1;
  for (int t = P.node_begin[1]; t < P.node_end[1]; ++t)
    if (best < 0 || s.len[t] > s.len[best]) best = t;
  return best;
}

// Rows only need bits below their own id when every deeper level is bounded
// by the level before it (the standard clique restrictions v_i < v_{i-1}).
__device__ __forceinline__ bool clique_lower_only(const Program& P) {
  for (int i = 3; i < P.depth; ++i)
    if (P.parent[i] != i - 1) return false;
  return true;
}

// Warp tier: count the unit in the warp's state (k=1 nodes built).
__device__ uint64_t clique_local_warp(const Ctx& c, const Program& P, uint32_t* rows) {
  const WarpState& s = *c.s;
  const int un = clique_universe(s, P);
  const uint32_t* U = s.ptr[un];
  const uint32_t u = s.len[un];
  if (u < 2) return 0;  // levels 2..n-1 need n-2 >= 3 distinct elements of U
  LocalIndex L;
  L.keys = c.hash;
  L.idx = reinterpret_cast<uint16_t*>(c.hash + 2 * kLocalWarpMax);
  uint32_t* rowbuf = c.hash + 2 * kLocalWarpMax + kLocalWarpMax;  // after keys (2u) and idx (u/2 words)
  local_index_build(L, U, u, c.lane, 32, false);
  const uint32_t nwords = (u + 31) / 32;
  if (c.lane < kLocalWarpRowWords) rowbuf[c.lane] = 0u;
  __syncwarp();
  const bool lower = clique_lower_only(P);
  for (uint32_t a = 0; a < u; ++a)
    local_row(c, L, U, u, a, lower, rowbuf, nwords, rows + static_cast<uint64_t>(a) * kLocalWarpRowWords);
  __syncwarp();
  const uint32_t q0 = warp_lower_bound<false>(U, u, s.vals[0]);
  const uint32_t q1 = warp_lower_bound<false>(U, u, s.vals[1]);
  return local_dfs<1>(c, P, rows, kLocalWarpRowWords, u, q0, q1, 0, 1);
}

// SHAPE: kShapeGeneric runs every path; kShapeBatch4 is the depth-4 plan
// with a batched leaf (clique4, rectangle, every 4-vertex motif): the unit's
// loop-0/1 sets, then one leaf batch -- the deeper-loop DFS, per-sibling
// leaves and clique-local paths are compiled out, which keeps the hot code
// small enough for the instruction caches at 64 resident warps per SM.
enum { kShapeGeneric = 0, kShapeBatch4 = 1 };

template <bool METER, bool TRACE, int SHAPE>
__global__ void __launch_bounds__(kThreads, SHAPE == kShapeBatch4 ? 8 : 3) count_kernel(const KernelArgs a) {
  __shared__ WarpState states[kWarpsPerBlock];
  extern __shared__ uint32_t dyn_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + wib;
  const Program& P = a.prog;
  Ctx c;
  c.off = a.off;
  c.adj = a.adj;
  c.s = &states[wib];
  c.scratch = a.scratch + gw * static_cast<uint64_t>(P.nslots) * a.cap;
  c.cap = a.cap;
  c.lane = lane;
  c.nv = static_cast<float>(a.nverts);
  c.tune = a.tune;
  c.list_cost = a.list_cost;
  c.heavy_stream = a.heavy_stream;
  c.heavy_min = a.heavy_min;
  c.gbm = a.warp_bitmaps ? a.warp_bitmaps + gw * a.bitmap_words : nullptr;
  c.gbm_words = static_cast<uint32_t>(a.bitmap_words);
  c.hslots = SHAPE == kShapeBatch4 ? kBatchHashSlots : kHashSlots;
  c.hash = dyn_smem + wib * c.hslots;
  const bool batch = P.batch;
  HeavyQueue hq;
  hq.items = a.heavy_items;
  hq.cap = a.heavy_cap;
  hq.count = &a.ctr->heavy_count;
  uint64_t trbuf[TRACE ? kTrCount : 1];
  if (TRACE)
    for (int i = 0; i < kTrCount; ++i) trbuf[i] = 0;
  uint64_t* tr = trbuf;
  long long tclk = 0;
  unsigned long long t_start = 0;
  if (TRACE) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  WarpState& s = states[wib];

  uint64_t cnt = 0, elems = 0, units = 0;
  bool ovf = false;
  uint32_t pos[kMaxLevels];

  for (;;) {
    unsigned long long chunk = 0;
    if (lane == 0) chunk = atomicAdd(&a.ctr->next_chunk, 1ull);
    chunk = __shfl_sync(kFull, chunk, 0);
    uint64_t gchunk = chunk;
    if (a.num_shards > 1) {
      if (chunk >= a.map_pref[a.map_k]) break;
      uint32_t k = 0;
      while (a.map_pref[k + 1] <= chunk) ++k;  // map_k <= kShardSplit: a short scan
      gchunk = a.map_begin[k] + (chunk - a.map_pref[k]);
    }
    const uint64_t e0 = a.unit_begin + gchunk * kChunk;
    if (e0 >= a.unit_end) break;
    const uint64_t e = e0 + lane;
    bool valid = e < a.unit_end;
    const uint32_t u0 = valid ? __ldg(a.src + e) : 0u;
    const uint32_t u1 = valid ? __ldg(a.adj + e) : 0u;
    if (P.unit_bound) valid = valid && (u1 < u0);
    unsigned m = __ballot_sync(kFull, valid);
    units += __popc(m);
    if (P.depth == 2) {
      checked_acc(cnt, __popc(m), ovf);
      continue;
    }
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t v0 = __shfl_sync(kFull, u0, l);
      const uint32_t v1 = __shfl_sync(kFull, u1, l);
      if (lane == 0) {
        s.vals[0] = v0;
        s.vals[1] = v1;
      }
      __syncwarp();
      if (METER) elems += meter_level(c, P, 2);
      if (SHAPE == kShapeBatch4 && !METER && (a.tune & 1024u) && hq.items) {
        // (tune 1024) hub-hub units go straight to the CTA tier: their loop-1
        // sets would be rebuilt there anyway
        const uint32_t d0 = static_cast<uint32_t>(__ldg(c.off + v0 + 1) - __ldg(c.off + v0));
        const uint32_t d1 = static_cast<uint32_t>(__ldg(c.off + v1 + 1) - __ldg(c.off + v1));
        if (min(d0, d1) >= 2048u) {
          unsigned long long slot = 0;
          if (lane == 0) slot = atomicAdd(hq.count, 1ull);
          slot = __shfl_sync(kFull, slot, 0);
          if (slot < hq.cap) {
            if (lane < 2) hq.items[slot * kHeavyItemWords + lane] = lane ? v1 : v0;
            else if (lane == kHeavyItemWords - 1) hq.items[slot * kHeavyItemWords + lane] = 0u;
            continue;
          }
        }
      }
      if (TRACE) tclk = clock64();
      for (int t = P.node_begin[0]; t < P.node_end[0]; ++t) build_node(c, P, t);
      for (int t = P.node_begin[1]; t < P.node_end[1]; ++t) build_node(c, P, t);
      if (TRACE) tr[kTrBuildCycles] += clock64() - tclk;
      if (SHAPE == kShapeBatch4) {
        if (METER) elems += meter_batch(c, P);
        if (TRACE) tclk = clock64();
        checked_acc(cnt, leaf_batch<TRACE>(c, P, hq, tr), ovf);
        if (TRACE) tr[kTrBatchCycles] += clock64() - tclk;
        continue;
      } else {
      if (P.depth == 3) {
        checked_acc(cnt, leaf_count(c, P), ovf);
        continue;
      }
      if (!METER && P.clique && a.local_rows && !(a.tune & 2u)) {
        const uint32_t u = s.len[clique_universe(s, P)];
        if (u <= kLocalWarpMax) {
          checked_acc(cnt, clique_local_warp(c, P, a.local_rows + gw * kLocalWarpMax * kLocalWarpRowWords),
                      ovf);
          continue;
        }
        if (u <= kLocalCtaMax && hq.items) {  // CTA tier
          unsigned long long slot = 0;
          if (lane == 0) slot = atomicAdd(hq.count, 1ull);
          slot = __shfl_sync(kFull, slot, 0);
          if (slot < hq.cap) {
            if (lane < 2) hq.items[slot * kHeavyItemWords + lane] = s.vals[lane];
            if (lane == kHeavyItemWords - 1) hq.items[slot * kHeavyItemWords + lane] = kCliqueItem;
            continue;
          }
        }
      }
      if (batch && P.depth == 4) {
        if (METER) elems += meter_batch(c, P);
        if (TRACE) tclk = clock64();
        checked_acc(cnt, leaf_batch<TRACE>(c, P, hq, tr), ovf);
        if (TRACE) tr[kTrBatchCycles] += clock64() - tclk;
        continue;
      }
      int level = 2;
      pos[2] = 0;
      while (level >= 2) {
        const int cn = P.cand[level];
        if (pos[level] >= s.len[cn]) {
          --level;
          continue;
        }
        const uint32_t x = s.ptr[cn][pos[level]];
        ++pos[level];
        __syncwarp();
        if (lane == 0) s.vals[level] = x;
        __syncwarp();
        if (METER) elems += meter_level(c, P, level + 1);
        if (TRACE) tclk = clock64();
        for (int t = P.node_begin[level]; t < P.node_end[level]; ++t) build_node(c, P, t);
        if (TRACE) tr[kTrBuildCycles] += clock64() - tclk;
        if (level == P.depth - 2) {
          if (TRACE) tclk = clock64();
          checked_acc(cnt, leaf_count(c, P), ovf);
          if (TRACE) {
            tr[kTrLeafCycles] += clock64() - tclk;
            tr[kTrLeaves] += 1;
          }
        } else if (batch && level == P.depth - 3) {
          if (METER) elems += meter_batch(c, P);
          if (TRACE) tclk = clock64();
          checked_acc(cnt, leaf_batch<TRACE>(c, P, hq, tr), ovf);
          if (TRACE) tr[kTrBatchCycles] += clock64() - tclk;
        } else {
          ++level;
          pos[level] = 0;
        }
      }
      }  // SHAPE
    }
  }
  if (lane == 0) {
    if (cnt) {
      const unsigned long long old = atomicAdd(&a.ctr->count, static_cast<unsigned long long>(cnt));
      if (old + cnt < old) ovf = true;
    }
    if (METER && elems) atomicAdd(&a.ctr->elements, static_cast<unsigned long long>(elems));
    if (units) atomicAdd(&a.ctr->units, static_cast<unsigned long long>(units));
    if (ovf) atomicOr(&a.ctr->overflow, 1u);
    if (TRACE) {
      tr[kTrUnits] = units;
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      const unsigned long long busy = now - t_start;
      tr[kTrWarpBusySum] = busy;
      atomicMax(&a.ctr->trace[kTrWarpBusyMax], busy);
      for (int i = 0; i < kTrCount; ++i)
        if (tr[i]) atomicAdd(&a.ctr->trace[i], static_cast<unsigned long long>(tr[i]));
    }
  }
}

// ---------------------------------------------------------------- CTA tier ---
// The deferred batches, one per CTA at a time: 16 warps share a 64 KB
// bucketised table.  Node builds are CTA-wide two-pass filters (count per
// warp slice, scan, write), and the leaf stream is a CTA-wide load-balanced
// search: per tile of 512 lists a block scan of the list lengths, then every
// thread expands kLbsRun consecutive elements of the concatenation (one owner
// search per run, kLbsRun independent loads in flight).  Probe sets beyond
// the table are split into value-range chunks (the streamed lists are
// range-restricted per chunk, so every element is still probed exactly once).

#ifndef SMG_LBS_RUN
#define SMG_LBS_RUN 8
#endif
constexpr int kLbsRun = SMG_LBS_RUN;
constexpr int kTile = kHeavyThreads;

struct HeavyShared {
  WarpState st;
  unsigned long long item;
  unsigned long long red_a[kHeavyWarps], red_b[kHeavyWarps];
  uint32_t wsum[kHeavyWarps + 1];
  uint32_t wsum2[kHeavyWarps + 1];
  uint32_t offs[kTile + 1];
  const uint32_t* lptr[kTile];
  uint32_t llo[kTile], lhi[kTile];
  uint32_t search_idx[kTile];
  uint32_t nsearch;
  uint32_t chunk_next;  // cta_stream: next long-list chunk to claim
  uint32_t coffs[kTile + 1];  // long-list chunk offsets (cta_stream)
  uint32_t llen[kTile];        // long-list lengths (cta_stream)
};

// Two block-wide exclusive scans sharing one set of barriers.  The caller
// must sync before the next use of sh.wsum/wsum2.
__device__ void cta_excl_scan2(uint32_t v, uint32_t w, HeavyShared& sh, uint32_t* rv, uint32_t* rw,
                               uint32_t* tv, uint32_t* tw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t iv = warp_incl_scan(v, lane), iw = warp_incl_scan(w, lane);
  if (lane == 31) {
    sh.wsum[warp] = iv;
    sh.wsum2[warp] = iw;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = lane < kHeavyWarps ? sh.wsum[lane] : 0u;
    const uint32_t y = lane < kHeavyWarps ? sh.wsum2[lane] : 0u;
    const uint32_t xi = warp_incl_scan(x, lane), yi = warp_incl_scan(y, lane);
    if (lane < kHeavyWarps) {
      sh.wsum[lane] = xi - x;
      sh.wsum2[lane] = yi - y;
    }
    if (lane == kHeavyWarps - 1) {
      sh.wsum[kHeavyWarps] = xi;
      sh.wsum2[kHeavyWarps] = yi;
    }
  }
  __syncthreads();
  *rv = sh.wsum[warp] + iv - v;
  *rw = sh.wsum2[warp] + iw - w;
  *tv = sh.wsum[kHeavyWarps];
  *tw = sh.wsum2[kHeavyWarps];
}

// Fill the CTA table with arr[0..n) (all threads; includes the syncs).
__device__ ProbeSet cta_table(uint32_t* table, const uint32_t* arr, uint32_t n) {
  ProbeSet p;
  p.arr = arr;
  p.n = n;
  p.lo = arr[0];
  p.hi = arr[n - 1];
  p.hash = table;
  p.bits = table_bits(n);
  __syncthreads();
  fill_table(table, p, threadIdx.x, kHeavyThreads);
  __syncthreads();
  insert_table(table, p, threadIdx.x, kHeavyThreads);
  __syncthreads();
  return p;
}

// CTA-wide build of node t (see build_node).
__device__ void cta_build_node(const Ctx& c, const Program& P, int t, HeavyShared& sh,
                               uint32_t* table) {
  const Node& nd = P.nodes[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* in;
  uint32_t inlen;
  node_input_cta(c, nd, in, inlen);
  if (nd.raw || nd.nops != 1) {
    if (warp == 0) build_node(c, P, t);  // raw slice, or a multi-op start node (rare)
    __syncthreads();
    return;
  }
  uint32_t* out = c.scratch + static_cast<uint64_t>(nd.slot) * c.cap;
  const WarpState& s = sh.st;
  const uint32_t v = s.vals[nd.ops[0].level];
  const uint32_t* L;
  uint32_t nL;
  nbrs(c, v, L, nL);
  const uint32_t* X = in;
  uint32_t nX = inlen;
  ProbeSet pr;
  pr.arr = L;
  pr.n = 0;
  pr.bits = 0;
  bool keep_found = true;
  uint32_t exclude = kEmptySlot;
  if (inlen == 0) {
    nX = 0;
  } else if (nd.ops[0].mode == kOpIsect) {
    if (nd.bound >= 0) nL = cta_lower_bound<true>(L, nL, s.vals[nd.bound]);
    if (nL == 0) {
      nX = 0;
    } else {
      const bool in_small = inlen <= nL;
      const uint32_t* Sm = in_small ? in : L;
      const uint32_t nSm = in_small ? inlen : nL;
      const uint32_t* Lg = in_small ? L : in;
      const uint32_t nLg = in_small ? nL : inlen;
      if (2 * nSm <= kHeavySlots && nLg >= 4 * nSm) {
        pr = cta_table(table, Sm, nSm);
        X = Lg;
        nX = nLg;
      } else if (2 * nSm <= kHeavySlots && nSm > 32) {
        pr = cta_table(table, Sm, nSm);
        X = Lg;
        nX = nLg;
      } else {
        pr.arr = Lg;
        pr.n = nLg;
        pr.lo = Lg[0];
        pr.hi = Lg[nLg - 1];
        X = Sm;
        nX = nSm;
      }
    }
  } else {
    keep_found = false;
    exclude = v;
    const uint32_t a = cta_lower_bound<true>(L, nL, in[0]);
    const uint32_t b = a + cta_lower_bound<true>(L + a, nL - a, in[inlen - 1] + 1u);
    if (b > a) {
      if (2 * (b - a) <= kHeavySlots) {
        pr = cta_table(table, L + a, b - a);
      } else {
        pr.arr = L + a;
        pr.n = b - a;
        pr.lo = pr.arr[0];
        pr.hi = pr.arr[pr.n - 1];
      }
    }
  }
  // One filter pass over per-warp slices, each compacted into the staging
  // slot at its own input offset; after a scan of the slice counts every warp
  // copies its run to the final position (no second probe pass).
  uint32_t* stage = c.scratch + static_cast<uint64_t>(P.nslots) * c.cap;
  const uint32_t chunk = ((nX + kHeavyWarps - 1) / kHeavyWarps + 255) / 256 * 256;
  const uint32_t lo = min(nX, warp * chunk), hi = min(nX, lo + chunk);
  const uint32_t cnt = filter_list<false, 8>(c, X + lo, hi - lo, pr, keep_found, exclude, stage + lo);
  if (lane == 0) sh.wsum[warp] = cnt;
  __syncthreads();
  uint32_t off = 0, total = 0;
  for (int w = 0; w < kHeavyWarps; ++w) {
    off += w < warp ? sh.wsum[w] : 0u;
    total += sh.wsum[w];
  }
  for (uint32_t i = lane; i < cnt; i += 32) out[off + i] = stage[lo + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    sh.st.ptr[t] = out;
    sh.st.len[t] = total;
  }
  __syncthreads();
}

// CTA-wide load-balanced stream: sum_{s in S} |N(s) & [lo_s, hi_s) & P|.
// Returns this thread's partial count.
__device__ __forceinline__ bool probe_bitmap(const ProbeSet& P, uint32_t y) {
  const uint32_t d = y - P.bm_base;
  return (P.bm[d >> 5] >> (d & 31)) & 1u;
}

#ifndef SMG_CTA_LONG
#define SMG_CTA_LONG 256
#endif
#ifndef SMG_CTA_CHUNK
#define SMG_CTA_CHUNK 1024
#endif
constexpr uint32_t kCtaLong = SMG_CTA_LONG;    // lists this long are streamed in warp chunks
constexpr uint32_t kCtaChunk = SMG_CTA_CHUNK;  // elements per warp chunk (rounds of 8 coalesced loads)

// CTA-wide stream: sum_{s in S} |N(s) & [lo_s, hi_s) & P| with P a bitmap.
// Per tile of kTile lists every thread resolves one list's window (prefix
// truncation by binary search on both ends).  Long lists are cut into
// kCtaChunk-element chunks that whole warps stream with coalesced loads (one
// owner search per chunk); short lists are expanded by a load-balanced
// search (runs of kLbsRun elements per thread); skewed pairs binary-search
// P's window into N(s).  Returns this thread's partial count.
template <bool TRACE>
__device__ uint64_t cta_stream(const Ctx& c, const uint32_t* S, uint32_t nS, const ProbeSet& P,
                               int rel, HeavyShared& sh, uint64_t* tr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t hits = 0;
  for (uint32_t tile = 0; tile < nS; tile += kTile) {
    const uint32_t i = tile + threadIdx.x;
    if (threadIdx.x == 0) {
      sh.nsearch = 0;
      sh.chunk_next = 0;
    }
    uint32_t len = 0, start = 0, lo_val = P.lo, hi_val = P.hi + 1u;
    const uint32_t* base = c.adj;
    if (i < nS) {
      const uint32_t s = S[i];
      if (rel == 1) hi_val = min(hi_val, s);
      if (rel == 2) lo_val = max(lo_val, s + 1u);
      const unsigned long long b = __ldg(c.off + s), e = __ldg(c.off + s + 1);
      base = c.adj + b;
      const uint32_t deg = static_cast<uint32_t>(e - b);
      if (lo_val < hi_val && deg) {
        const uint32_t first = __ldg(base), last = __ldg(base + deg - 1);
        if (last >= lo_val && first < hi_val) {
          uint32_t end = deg;
          if (deg > 32) {
            // Window ends by binary search (a chain of dependent loads), unless
            // the part outside the window is small enough to stream and filter
            // (ids spread evenly over a list's value range).
            const float span = static_cast<float>(last - first) + 1.f;
            if (first < lo_val && static_cast<float>(lo_val - first) > span * 0.0625f)
              start = window_start(base, deg, first, last, lo_val);
            if (last >= hi_val && static_cast<float>(last - hi_val) > span * 0.0625f)
              end = window_end(base, deg, first, last, hi_val);
          }
          len = end > start ? end - start : 0u;
        }
      }
    }
    __syncthreads();  // nsearch reset visible
    const bool search = len > kLongList && static_cast<uint64_t>(P.n) * ilog2p1(len) * 2u < len;
    if (search) sh.search_idx[atomicAdd(&sh.nsearch, 1u)] = threadIdx.x;
    const bool is_long = !search && len >= kCtaLong;
    const uint32_t slen = search || is_long ? 0u : len;
    const uint32_t nch = is_long ? (len + kCtaChunk - 1) / kCtaChunk : 0u;
    uint32_t total, tch, off, coff;
    cta_excl_scan2(slen, nch, sh, &off, &coff, &total, &tch);
    sh.offs[threadIdx.x] = off;
    sh.coffs[threadIdx.x] = coff;
    if (threadIdx.x == 0) {
      sh.offs[kTile] = total;
      sh.coffs[kTile] = tch;
    }
    sh.lptr[threadIdx.x] = base + start;
    sh.llo[threadIdx.x] = lo_val;
    sh.lhi[threadIdx.x] = hi_val;
    sh.llen[threadIdx.x] = len;
    __syncthreads();
    if (TRACE && threadIdx.x == 0) {
      tr[kTrHeavyElems] += total;
      tr[kTrHeavyTiles] += 1;
    }
    // 1) short lists: load-balanced runs
    for (uint32_t e0 = threadIdx.x * kLbsRun; e0 < total; e0 += kTile * kLbsRun) {
      // owner of e0: the last j with offs[j] <= e0; its list state is kept in
      // registers and reloaded only when the run crosses into the next list
      uint32_t j = 0;
#pragma unroll
      for (uint32_t step = kTile / 2; step >= 1; step >>= 1)
        if (sh.offs[j + step] <= e0) j += step;
      const uint32_t* lp = sh.lptr[j] - sh.offs[j];
      uint32_t lo = sh.llo[j], hi = sh.lhi[j], next = sh.offs[j + 1];
      uint32_t y[kLbsRun];
      uint32_t ylo[kLbsRun], yhi[kLbsRun];
#pragma unroll
      for (int k = 0; k < kLbsRun; ++k) {
        const uint32_t e = e0 + k;
        y[k] = kEmptySlot;
        ylo[k] = lo;
        yhi[k] = hi;
        if (e < total) {
          while (next <= e) {
            ++j;
            lp = sh.lptr[j] - sh.offs[j];
            lo = sh.llo[j];
            hi = sh.lhi[j];
            next = sh.offs[j + 1];
          }
          y[k] = __ldg(lp + e);
          ylo[k] = lo;
          yhi[k] = hi;
        }
      }
#pragma unroll
      for (int k = 0; k < kLbsRun; ++k)
        if (y[k] >= ylo[k] && y[k] < yhi[k] && probe_bitmap(P, y[k])) ++hits;
    }
    // 2) long lists: whole warps claim chunks dynamically (after their share
    //    of the short-list runs, so the tile ends balanced)
    for (;;) {
      uint32_t q = 0;
      if (lane == 0) q = atomicAdd(&sh.chunk_next, 1u);
      q = __shfl_sync(kFull, q, 0);
      if (q >= tch) break;
      uint32_t j = 0;
#pragma unroll
      for (uint32_t step = kTile / 2; step >= 1; step >>= 1)
        if (sh.coffs[j + step] <= q) j += step;
      const uint32_t* lp = sh.lptr[j];
      const uint32_t ll = sh.llen[j], jlo = sh.llo[j], jhi = sh.lhi[j];
      const uint32_t e0 = (q - sh.coffs[j]) * kCtaChunk;
      const uint32_t e1 = min(ll, e0 + kCtaChunk);
      if (TRACE && lane == 0) tr[kTrStreamElems] += e1 - e0;
      constexpr int kU = 8;  // loads in flight per lane
      for (uint32_t t = e0 + lane; t < e1; t += 32 * kU) {
        uint32_t y[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
          const uint32_t idx = t + 32 * k;
          y[k] = idx < e1 ? __ldg(lp + idx) : kEmptySlot;
        }
#pragma unroll
        for (int k = 0; k < kU; ++k)
          if (y[k] >= jlo && y[k] < jhi && probe_bitmap(P, y[k])) ++hits;
      }
    }
    // 3) skewed pairs: one warp per list, P's window binary-searched into N(s)
    for (uint32_t q = warp; q < sh.nsearch; q += kHeavyWarps) {
      const uint32_t jt = sh.search_idx[q];
      const uint32_t jlo = sh.llo[jt], jhi = sh.lhi[jt];
      const uint32_t pa = warp_lower_bound<false>(P.arr, P.n, jlo);
      const uint32_t pb = pa + warp_lower_bound<false>(P.arr + pa, P.n - pa, jhi);
      const uint32_t s = S[tile + jt];
      const unsigned long long b = __ldg(c.off + s), e = __ldg(c.off + s + 1);
      const uint32_t* lb = c.adj + b;
      const uint32_t deg = static_cast<uint32_t>(e - b);
      for (uint32_t qq = pa + lane; qq < pb; qq += 32)
        if (contains_dev(lb, deg, P.arr[qq])) ++hits;
    }
    __syncthreads();
  }
  return hits;
}

template <bool TRACE>
__global__ void __launch_bounds__(kHeavyThreads, kHeavyMinBlocks) heavy_kernel(const KernelArgs a) {
  __shared__ HeavyShared sh;
  extern __shared__ uint4 table4[];
  // dynamic smem: [bitmap, kBitmapWords) [node table / clique-local region)
  uint32_t* bm = reinterpret_cast<uint32_t*>(table4);
  uint32_t* table = bm + kBitmapWords;
  for (uint32_t i = threadIdx.x; i < kBitmapWords / 4; i += kHeavyThreads)
    table4[i] = make_uint4(0u, 0u, 0u, 0u);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const Program& P = a.prog;
  Ctx c;
  c.off = a.off;
  c.adj = a.adj;
  c.s = &sh.st;
  c.scratch = a.heavy_scratch + static_cast<uint64_t>(blockIdx.x) * (P.nslots + 1) * a.cap;  // + staging slot
  c.cap = a.cap;
  c.lane = lane;
  c.nv = static_cast<float>(a.nverts);
  c.tune = a.tune;
  c.list_cost = a.list_cost;
  c.heavy_stream = 0;
  c.heavy_min = 0;
  c.gbm = nullptr;
  c.hslots = kHashSlots;
  c.hash = table;
  uint64_t trbuf[TRACE ? kTrCount : 1];
  if (TRACE)
    for (int i = 0; i < kTrCount; ++i) trbuf[i] = 0;
  uint64_t* tr = trbuf;
  const unsigned long long nitems = min(*(volatile unsigned long long*)&a.ctr->heavy_count, a.heavy_cap);
  uint64_t cnt = 0;
  bool ovf = false;
  const bool yltx = P.batch_yltx != 0;
  for (;;) {
    if (threadIdx.x == 0) sh.item = atomicAdd(&a.ctr->heavy_next, 1ull);
    __syncthreads();
    const unsigned long long it = sh.item;
    if (it >= nitems) break;
    long long t0 = TRACE ? clock64() : 0;
    if (threadIdx.x < P.depth - 2) sh.st.vals[threadIdx.x] = a.heavy_items[it * kHeavyItemWords + threadIdx.x];
    const bool clique_item = a.heavy_items[it * kHeavyItemWords + kHeavyItemWords - 1] == kCliqueItem;
    __syncthreads();
    if (clique_item) {
      // CTA clique-local: k=0,1 nodes, U, index table, rows by all warps, split DFS
      for (int t = P.node_begin[0]; t < P.node_end[1]; ++t) cta_build_node(c, P, t, sh, table);
      const int un = clique_universe(sh.st, P);
      const uint32_t* U = sh.st.ptr[un];
      const uint32_t u = sh.st.len[un];
      // the local index and row buffers borrow the (idle) bitmap region
      LocalIndex L;
      L.keys = bm;
      L.idx = reinterpret_cast<uint16_t*>(bm + kLocalCtaSlots);
      uint32_t* rowbuf = bm + kLocalCtaSlots + kLocalCtaSlots / 2 + warp * kLocalRowWords;
      local_index_build(L, U, u, threadIdx.x, kHeavyThreads, true);
      for (uint32_t w = lane; w < kLocalRowWords; w += 32) rowbuf[w] = 0u;
      __syncwarp();
      const uint32_t nwords = (u + 31) / 32;
      const bool lower = clique_lower_only(P);
      uint32_t* rows = a.heavy_rows + static_cast<uint64_t>(blockIdx.x) * kLocalCtaMax * kLocalRowWords;
      for (uint32_t r = warp; r < u; r += kHeavyWarps)
        local_row(c, L, U, u, r, lower, rowbuf, nwords, rows + static_cast<uint64_t>(r) * kLocalRowWords);
      __threadfence_block();
      __syncthreads();
      const uint32_t q0 = cta_lower_bound<false>(U, u, sh.st.vals[0]);
      const uint32_t q1 = cta_lower_bound<false>(U, u, sh.st.vals[1]);
      const uint64_t part = local_dfs<kLocalRowWords / 32>(c, P, rows, kLocalRowWords, u, q0, q1, warp,
                                                          kHeavyWarps);
      if (lane == 0) sh.red_a[warp] = part;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint64_t sum = 0;
        for (int w = 0; w < kHeavyWarps; ++w) sum += sh.red_a[w];
        checked_acc(cnt, sum, ovf);
        if (TRACE) {
          tr[kTrHeavyItems] += 1;
          tr[kTrHeavyCycles] += clock64() - t0;
        }
      }
      for (uint32_t i = threadIdx.x; i < kBitmapWords / 4; i += kHeavyThreads)
        table4[i] = make_uint4(0u, 0u, 0u, 0u);  // batch items expect a zero bitmap
      __syncthreads();
      continue;
    }
    for (int t = P.node_begin[0]; t < P.node_end[P.depth - 3]; ++t) cta_build_node(c, P, t, sh, table);
    long long t1 = TRACE ? clock64() : 0;
    if (TRACE && threadIdx.x == 0) tr[kTrHeavyBuild] += t1 - t0;
    const BatchSets b = batch_sets(sh.st, P);
    if (b.nA == 0 || b.nB == 0) {  // no leaf pairs (only early-deferred units can get here)
      if (threadIdx.x == 0 && TRACE) tr[kTrHeavyItems] += 1;
      __syncthreads();
      continue;
    }
    // side choice from the degree sums (CTA-wide)
    bool flip = false;
    if (!b.same) {
      uint64_t sum_s = 0;
      auto cta_dsum = [&](const uint32_t* X, uint32_t n) -> uint64_t {
        const uint64_t d = degree_sum(c, X, n, warp * 32, kHeavyThreads);
        __syncthreads();
        if (lane == 0) sh.red_a[warp] = d;
        __syncthreads();
        uint64_t t = 0;
        for (int w = 0; w < kHeavyWarps; ++w) t += sh.red_a[w];
        return t;
      };
      flip = choose_stream_b(c, b, cta_dsum, sum_s);
      __syncthreads();
    }
    const uint32_t* Parr = flip ? b.A : b.B;
    const uint32_t Pn = flip ? b.nA : b.nB;
    const uint32_t* S = flip ? b.B : b.A;
    const uint32_t nS = flip ? b.nB : b.nA;
    const int rel = yltx ? (flip ? 2 : 1) : 0;
    uint64_t core = 0;
    // The probe set as a bitmap, one id slice of kBitmapSpan at a time (one
    // slice whenever n <= 2^20); the streamed lists are clipped to the slice's
    // part of P, so every element is probed once.
    for (uint32_t i0 = 0; i0 < Pn;) {
      const uint32_t base = Parr[i0];
      const uint64_t lim = static_cast<uint64_t>(base) + kBitmapSpan;
      const uint32_t i1 = static_cast<uint64_t>(Parr[Pn - 1]) < lim
                              ? Pn
                              : i0 + cta_lower_bound<false>(Parr + i0, Pn - i0, static_cast<uint32_t>(lim));
      for (uint32_t i = i0 + threadIdx.x; i < i1; i += kHeavyThreads) {
        const uint32_t d = Parr[i] - base;
        atomicOr(&bm[d >> 5], 1u << (d & 31));
      }
      __syncthreads();
      ProbeSet ps;
      ps.arr = Parr + i0;
      ps.n = i1 - i0;
      ps.lo = Parr[i0];
      ps.hi = Parr[i1 - 1];
      ps.hash = nullptr;
      ps.bits = 0;
      ps.bm = bm;
      ps.bm_base = base;
      core += cta_stream<TRACE>(c, S, nS, ps, rel, sh, tr);
      __syncthreads();
      for (uint32_t i = i0 + threadIdx.x; i < i1; i += kHeavyThreads) bm[(Parr[i] - base) >> 5] = 0u;
      __syncthreads();
      i0 = i1;
    }
    core = warp_sum64(core);
    if (TRACE && threadIdx.x == 0) tr[kTrHeavyStream] += clock64() - t1;
    const uint64_t dpart = P.batch_diff ? diff_terms(c, P, b, warp * 32, kHeavyThreads, warp == 0) : 0;
    if (lane == 0) {
      sh.red_a[warp] = core;
      sh.red_b[warp] = dpart;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t sc = 0, sd = 0;
      for (int w = 0; w < kHeavyWarps; ++w) {
        sc += sh.red_a[w];
        sd += sh.red_b[w];
      }
      checked_acc(cnt, P.batch_diff ? sd - sc : sc, ovf);
      if (TRACE) {
        tr[kTrHeavyItems] += 1;
        tr[kTrHeavyCycles] += clock64() - t0;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (cnt) {
      const unsigned long long old = atomicAdd(&a.ctr->count, static_cast<unsigned long long>(cnt));
      if (old + cnt < old) ovf = true;
    }
    if (ovf) atomicOr(&a.ctr->overflow, 1u);
    // the last CTA out rewinds the queue cursor, so a replay of this launch
    // (profiler kernel replay) sees the same queue
    __threadfence();
    if (atomicAdd(&a.ctr->heavy_done, 1u) == gridDim.x - 1) {
      a.ctr->heavy_next = 0;
      a.ctr->heavy_done = 0;
    }
  }
  if (TRACE && lane == 0) {
    for (int i = 0; i < kTrCount; ++i)
      if (tr[i] && ((i != kTrHeavyItems && i != kTrHeavyCycles && i != kTrHeavyBuild &&
                     i != kTrHeavyStream && i != kTrHeavyElems && i != kTrHeavyTiles) || threadIdx.x == 0))
        atomicAdd(&a.ctr->trace[i], static_cast<unsigned long long>(tr[i]));
  }
}

// ------------------------------------------------------------- listing ---
// enumerate_instances (engine.cpp:181-191, enumerate_from :117-134): the same
// depth-first nested loops without leaf batching.  The reference emits in
// level-0 ascending, then lexicographic order; edge units in CSR slot order
// are exactly (v0 asc, v1 asc) and every candidate set is sorted, so a unit's
// embeddings are contiguous in the global order.  Pass COUNT stores each
// unit's embedding count; after a scan, pass WRITE writes each unit's tuples
// at its offset, dropping those at or beyond `limit`.
template <bool WRITE>
__global__ void __launch_bounds__(kThreads) enum_kernel(const KernelArgs a, uint64_t slot_lo,
                                                        uint64_t slot_hi,
                                                        unsigned long long* unit_val,
                                                        unsigned long long limit, uint32_t* out) {
  __shared__ WarpState states[kWarpsPerBlock];
  extern __shared__ uint32_t dyn_smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + wib;
  const Program& P = a.prog;
  Ctx c;
  c.off = a.off;
  c.adj = a.adj;
  c.s = &states[wib];
  c.scratch = a.scratch + gw * static_cast<uint64_t>(P.nslots + 1) * a.cap;
  c.cap = a.cap;
  c.lane = lane;
  c.nv = static_cast<float>(a.nverts);
  c.tune = a.tune;
  c.list_cost = a.list_cost;
  c.heavy_stream = a.heavy_stream;
  c.heavy_min = a.heavy_min;
  c.gbm = a.warp_bitmaps ? a.warp_bitmaps + gw * a.bitmap_words : nullptr;
  c.gbm_words = static_cast<uint32_t>(a.bitmap_words);
  c.hslots = kHashSlots;
  c.hash = dyn_smem + wib * kHashSlots;
  uint32_t* leafbuf = c.scratch + static_cast<uint64_t>(P.nslots) * a.cap;
  WarpState& s = states[wib];
  const int n = P.depth;
  uint32_t pos[kMaxLevels];
  for (;;) {
    unsigned long long e = 0;
    if (lane == 0) e = slot_lo + atomicAdd(&a.ctr->next_chunk, 1ull);
    e = __shfl_sync(kFull, e, 0);
    if (e >= slot_hi) break;
    const uint32_t v0 = __ldg(a.src + e), v1 = __ldg(a.adj + e);
    const bool valid = !P.unit_bound || v1 < v0;
    unsigned long long base = WRITE ? unit_val[e - slot_lo] : 0ull;
    if (!valid || (WRITE && base >= limit)) {
      if (!WRITE && lane == 0) unit_val[e - slot_lo] = 0;
      continue;
    }
    unsigned long long written = 0;
    if (lane == 0) {
      s.vals[0] = v0;
      s.vals[1] = v1;
    }
    __syncwarp();
    auto emit_leaf = [&]() {
      // materialise the leaf set, then (WRITE) its tuples
      const uint32_t* in;
      uint32_t inlen;
      node_input(c, P.leaf, in, inlen);
      const uint32_t len = apply_ops<false>(c, P.leaf, in, inlen, leafbuf);
      __syncwarp();
      if (WRITE) {
        for (uint32_t i = lane; i < len; i += 32) {
          const unsigned long long idx = base + written + i;
          if (idx < limit) {
            uint32_t* t = out + idx * n;
            for (int j = 0; j < n - 1; ++j) t[j] = s.vals[j];
            t[n - 1] = leafbuf[i];
          }
        }
      }
      written += len;
      __syncwarp();
    };
    if (n == 2) {
      if (WRITE && lane == 0 && base < limit) {
        out[base * 2] = v0;
        out[base * 2 + 1] = v1;
      }
      written = 1;
    } else {
      for (int t = P.node_begin[0]; t < P.node_end[0]; ++t) build_node(c, P, t);
      for (int t = P.node_begin[1]; t < P.node_end[1]; ++t) build_node(c, P, t);
      if (n == 3) {
        emit_leaf();
      } else {
        int level = 2;
        pos[2] = 0;
        while (level >= 2) {
          if (WRITE && base + written >= limit) break;
          const int cn = P.cand[level];
          if (pos[level] >= s.len[cn]) {
            --level;
            continue;
          }
          const uint32_t x = s.ptr[cn][pos[level]];
          ++pos[level];
          __syncwarp();
          if (lane == 0) s.vals[level] = x;
          __syncwarp();
          for (int t = P.node_begin[level]; t < P.node_end[level]; ++t) build_node(c, P, t);
          if (level == n - 2) {
            emit_leaf();
          } else {
            ++level;
            pos[level] = 0;
          }
        }
      }
    }
    if (!WRITE && lane == 0) unit_val[e - slot_lo] = written;
  }
}

// E of level 1 over roots [lo, hi): |{x in N(v0) : x < beta_1}|.
__global__ void meter_roots_kernel(const unsigned long long* __restrict__ off,
                                   const uint32_t* __restrict__ adj, uint32_t lo, uint32_t hi,
                                   int bounded, Counters* ctr) {
  uint64_t acc = 0;
  for (uint64_t v = lo + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < hi;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long b = off[v], e = off[v + 1];
    const uint32_t len = static_cast<uint32_t>(e - b);
    acc += bounded ? lower_bound_dev(adj + b, len, static_cast<uint32_t>(v)) : len;
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&ctr->elements, static_cast<unsigned long long>(acc));
}

// src[e] = v for e in [off[v], off[v+1]).
__global__ void fill_src_kernel(const unsigned long long* __restrict__ off, uint64_t n,
                                uint32_t* __restrict__ src) {
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t v = warp; v < n; v += nwarps) {
    const unsigned long long b = off[v], e = off[v + 1];
    for (unsigned long long i = b + lane; i < e; i += 32) src[i] = static_cast<uint32_t>(v);
  }
}

// CSR validation on the device (the reference's Graph invariants,
// graph.hpp:18-20, 55-58): pass 1 checks the offsets and reduces the maximum
// degree; pass 2 (only after pass 1 succeeded, so every slice is in bounds)
// checks every slot: id < n, no self loop, strictly ascending, and the
// reverse slot exists (symmetry, by binary search in the neighbour's list).
// The first error found sets `err` (codes below); the host maps it to
// SMG_EINPUT.
enum { kCsrOk = 0, kCsrOffsets = 1, kCsrRange = 2, kCsrLoop = 3, kCsrOrder = 4, kCsrAsym = 5, kCsrDegree = 6 };

__global__ void validate_offsets_kernel(const unsigned long long* __restrict__ off, uint64_t n,
                                        uint64_t slots, unsigned int* err, unsigned long long* maxd) {
  unsigned long long m = 0;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long b = off[v], e = off[v + 1];
    if (e < b || e > slots) {
      atomicCAS(err, 0u, static_cast<unsigned>(kCsrOffsets));
      continue;
    }
    m = max(m, e - b);
  }
  for (int d = 16; d >= 1; d >>= 1) m = max(m, __shfl_xor_sync(kFull, m, d));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(maxd, m);
}

__global__ void validate_slots_kernel(const unsigned long long* __restrict__ off,
                                      const uint32_t* __restrict__ adj, const uint32_t* __restrict__ src,
                                      uint64_t n, uint64_t slots, unsigned int* err) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < slots;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = src[i], x = adj[i];
    unsigned code = kCsrOk;
    if (x >= n) {
      code = kCsrRange;
    } else if (x == v) {
      code = kCsrLoop;
    } else if (i > off[v] && adj[i - 1] >= x) {
      code = kCsrOrder;
    } else {
      const unsigned long long b = off[x], e = off[x + 1];
      if (!contains_dev(adj + b, static_cast<uint32_t>(e - b), v)) code = kCsrAsym;
    }
    if (code) atomicCAS(err, 0u, code);
  }
}

// Shard map: cost proxy of a chunk of kChunk level-1 units =
// sum over its slots (v0, v1) of 1 + min(deg v0, deg v1) (the smaller list
// bounds the unit's level-2 set), counting only units that pass level 1's
// bound when the plan has one.  Exclusive prefix sums over chunks cut the
// unit range into J super-chunks of equal cost: bound[j] = first chunk k with
// P[k] * J >= j * total.  paper_1911_12877_b200/distributed.py mirrors this
// exactly on the host (shard_slots).
__global__ void chunk_cost_kernel(const unsigned long long* __restrict__ off, const uint32_t* __restrict__ adj,
                                  const uint32_t* __restrict__ src, uint64_t slots, uint64_t nchunks,
                                  int unit_bound, unsigned long long* __restrict__ cost) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < nchunks;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long c = 0;
    const uint64_t e1 = (k + 1) * kChunk < slots ? (k + 1) * kChunk : slots;
    for (uint64_t e = k * kChunk; e < e1; ++e) {
      const uint32_t v0 = src[e], v1 = adj[e];
      if (unit_bound && !(v1 < v0)) continue;
      const unsigned long long d0 = off[v0 + 1] - off[v0], d1 = off[v1 + 1] - off[v1];
      c += 1 + min(d0, d1);
    }
    cost[k] = c;
  }
}

__global__ void shard_bounds_kernel(const unsigned long long* __restrict__ pref, uint64_t nchunks, uint32_t J,
                                    unsigned long long* __restrict__ bound) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > J) return;
  const unsigned long long total = pref[nchunks];
  const unsigned long long target = total * j;  // compare P[k] * J >= target
  uint64_t lo = 0, hi = nchunks;                 // first k in [0, nchunks] with P[k] * J >= target
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (pref[mid] * J >= target) hi = mid; else lo = mid + 1;
  }
  bound[j] = j == J ? nchunks : lo;
}

// ------------------------------------------------------------------ host ---

thread_local std::string g_last_error;
const uint32_t g_tune = [] {
  const char* e = std::getenv("SMG_TUNE");
  return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
}();
const uint32_t g_heavy_stream = [] {
  const char* e = std::getenv("SMG_HEAVY_STREAM");
  return e ? static_cast<uint32_t>(std::atol(e)) : 0u;
}();
const uint32_t g_heavy_min = [] {
  const char* e = std::getenv("SMG_HEAVY_MIN");
  return e ? static_cast<uint32_t>(std::atol(e)) : static_cast<uint32_t>(kHeavyMinStream);
}();
const float g_list_cost = [] {
  const char* e = std::getenv("SMG_LIST_COST");
  return e ? static_cast<float>(std::atof(e)) : kListCost;
}();
// SMG_FAST=0 disables the folded kernels (tindex.cu) for every call.
const int g_fast = [] {
  const char* e = std::getenv("SMG_FAST");
  return (e && *e == '0') ? 0 : 1;
}();
const int g_trace = [] {
  const char* e = std::getenv("SMG_TRACE");
  return (e && *e && *e != '0') ? 1 : 0;
}();

constexpr int kTryGeneric = -77;  // internal: the specialised kernel does not apply, run the generic executor

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define SMG_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t err_ = (call);                                                           \
    if (err_ != cudaSuccess)                                                             \
      return fail(SMG_EIO, std::string(#call) + ": " + cudaGetErrorString(err_));        \
  } while (0)

struct Replica {
  int device = -1;
  int num_sms = 0;
  unsigned long long* off = nullptr;
  uint32_t* adj = nullptr;
  uint32_t* src = nullptr;
  uint32_t* scratch = nullptr;
  size_t scratch_bytes = 0;
  uint32_t* heavy_items = nullptr;     // CTA-tier queue
  uint32_t* heavy_scratch = nullptr;
  uint32_t* warp_bitmaps = nullptr;    // per-warp id bitmaps (zeroed once, kept zero by the kernels)
  size_t warp_bitmaps_bytes = 0;
  uint32_t* local_rows = nullptr;      // clique-local rows (warp tier)
  size_t local_rows_bytes = 0;
  uint32_t* heavy_rows = nullptr;      // clique-local rows (CTA tier)
  size_t heavy_rows_bytes = 0;
  size_t heavy_scratch_bytes = 0;
  Counters* ctr = nullptr;  // device
  Counters* host_ctr = nullptr;  // pinned
  cudaStream_t stream = nullptr;       // owned
  cudaStream_t user_stream = nullptr;  // set by smg_graph_set_stream (not owned)
  cudaStream_t active() const { return user_stream ? user_stream : stream; }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t phase_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // created on first use (m4_count)
  double phase_ms[4] = {0, 0, 0, 0};  // last m4_count: 4-clique count, C4 pass, edge pass, vertex pass
  // cost-balanced shard map, cached per (num_shards, unit_bound)
  uint32_t map_shards = 0;
  int map_unit_bound = -1;
  std::vector<unsigned long long> map_bounds;          // host copy, J + 1 chunk boundaries
  unsigned long long* map_dev = nullptr;               // this replica's (begin[K], pref[K+1]) per shard
  TIndex tix;                                          // triangle index (folded kernels), built on demand
  uint32_t* fast_scratch = nullptr;                    // per-warp scratch of the folded kernels
  size_t fast_scratch_bytes = 0;
  unsigned long long* fast_acc = nullptr;              // per-slot accumulators (two-center kinds)
  size_t fast_acc_bytes = 0;
  int fast_acc_kind = 0;                               // kind whose accumulators fast_acc holds
  // folded full-count mode: per-CTA signed partials, global closed-form terms
  unsigned long long* part_dev = nullptr;
  unsigned long long* part_host = nullptr;             // pinned
  size_t part_words = 0;
  bool k4pairs_valid = false, k5_valid = false;
  unsigned long long k4pairs = 0, k5 = 0;              // cached: the graph is immutable
  int post_kind = 0;                                   // > 0: finish() combines the partials
  unsigned post_blocks = 0;
  __int128 post_global = 0;
  uint32_t* fast_dense = nullptr;                      // per-CTA dense codegree tables
  size_t fast_dense_bytes = 0;
  // degree-ordered copy of the CSR (orient_reindex ids: 0 = highest degree),
  // built on first use for the label-free full counts (cliques, 4-cycles)
  DevCSR ocsr;
  K4Work k4w;                                          // buffers of the per-root 4-clique count (k4.cu)
  uint32_t* tcount = nullptr;                          // per-slot triangle counts it leaves for the edge pass
  size_t tcount_bytes = 0;
  bool tiers_valid = false;                            // hub / group tier bounds of the ordered copy
  uint32_t hub_count = 0, group_end = 0;
  uint32_t* gtab = nullptr;                            // group-tier tables of the 4-cycle pass
  size_t gtab_bytes = 0;
  unsigned long long* gbar = nullptr;
  bool view_oriented = false;                          // off/adj/src currently point at ocsr
  bool map_oriented = false;                           // labelling the cached shard map belongs to
  std::mutex mu;
};

}  // namespace smg

struct smg_graph {
  uint64_t n = 0;
  uint64_t slots = 0;
  uint64_t max_degree = 0;
  std::vector<smg::Replica*> reps;
};

namespace smg {

// Work buffers (per-warp scratch, the CTA-tier queue and scratch, the warp
// bitmaps, clique-local rows) are sized by the launch, not by the graph, so a
// destroyed replica parks them per device and the next replica on that device
// adopts them: a new smg_graph (e.g. one per call through the C++ adapter or
// the e2e bench path) does not pay gigabytes of cudaMalloc/cudaFree + memset.
// The bitmaps are all-zero whenever no kernel runs, so they can be reused.
struct WorkSet {
  uint32_t* scratch = nullptr;
  size_t scratch_bytes = 0;
  uint32_t* heavy_items = nullptr;
  uint32_t* heavy_scratch = nullptr;
  size_t heavy_scratch_bytes = 0;
  uint32_t* local_rows = nullptr;
  size_t local_rows_bytes = 0;
  uint32_t* warp_bitmaps = nullptr;
  size_t warp_bitmaps_bytes = 0;
  uint32_t* heavy_rows = nullptr;
  size_t heavy_rows_bytes = 0;
  // closed-form 4-vertex counts (m4_count): dense per-CTA tables and group
  // tables (both kept zero by the kernels), barrier counters, partial sums
  uint32_t* fast_dense = nullptr;
  size_t fast_dense_bytes = 0;
  uint32_t* gtab = nullptr;
  size_t gtab_bytes = 0;
  unsigned long long* gbar = nullptr;
  unsigned long long* part_dev = nullptr;
  unsigned long long* part_host = nullptr;
  size_t part_words = 0;
  uint32_t* tcount = nullptr;  // per-slot triangle counts (k4.cu -> m4_edge_counts_kernel)
  size_t tcount_bytes = 0;
  K4Work k4w;                  // counters, events and row scratch of k4_count (lmax is per graph: reset on adopt)
};
std::mutex g_pool_mu;
WorkSet g_pool[64];  // one parked set per device ordinal
bool g_pool_used[64] = {};

void free_work(WorkSet& w) {
  if (w.scratch) cudaFree(w.scratch);
  if (w.heavy_items) cudaFree(w.heavy_items);
  if (w.heavy_scratch) cudaFree(w.heavy_scratch);
  if (w.local_rows) cudaFree(w.local_rows);
  if (w.warp_bitmaps) cudaFree(w.warp_bitmaps);
  if (w.heavy_rows) cudaFree(w.heavy_rows);
  if (w.fast_dense) cudaFree(w.fast_dense);
  if (w.gtab) cudaFree(w.gtab);
  if (w.gbar) cudaFree(w.gbar);
  if (w.part_dev) cudaFree(w.part_dev);
  if (w.part_host) cudaFreeHost(w.part_host);
  if (w.tcount) cudaFree(w.tcount);
  k4_free(&w.k4w);
  w = WorkSet();
}

void park_work(Replica& r) {
  WorkSet w;
  w.scratch = r.scratch;
  w.scratch_bytes = r.scratch_bytes;
  w.heavy_items = r.heavy_items;
  w.heavy_scratch = r.heavy_scratch;
  w.heavy_scratch_bytes = r.heavy_scratch_bytes;
  w.local_rows = r.local_rows;
  w.local_rows_bytes = r.local_rows_bytes;
  w.warp_bitmaps = r.warp_bitmaps;
  w.warp_bitmaps_bytes = r.warp_bitmaps_bytes;
  w.heavy_rows = r.heavy_rows;
  w.heavy_rows_bytes = r.heavy_rows_bytes;
  w.fast_dense = r.fast_dense;
  w.fast_dense_bytes = r.fast_dense_bytes;
  w.gtab = r.gtab;
  w.gtab_bytes = r.gtab_bytes;
  w.gbar = r.gbar;
  w.part_dev = r.part_dev;
  w.part_host = r.part_host;
  w.part_words = r.part_words;
  w.tcount = r.tcount;
  w.tcount_bytes = r.tcount_bytes;
  r.tcount = nullptr;
  r.tcount_bytes = 0;
  w.k4w = r.k4w;
  r.k4w = K4Work();
  r.fast_dense = nullptr;
  r.gtab = nullptr;
  r.gbar = nullptr;
  r.part_dev = nullptr;
  r.part_host = nullptr;
  r.fast_dense_bytes = r.gtab_bytes = r.part_words = 0;
  if (r.device < 0 || r.device >= 64) {
    free_work(w);
    return;
  }
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (g_pool_used[r.device]) free_work(g_pool[r.device]);  // keep the newest set
  g_pool[r.device] = w;
  g_pool_used[r.device] = true;
}

void adopt_work(Replica& r) {
  if (r.device < 0 || r.device >= 64) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool_used[r.device]) return;
  WorkSet& w = g_pool[r.device];
  r.scratch = w.scratch;
  r.scratch_bytes = w.scratch_bytes;
  r.heavy_items = w.heavy_items;
  r.heavy_scratch = w.heavy_scratch;
  r.heavy_scratch_bytes = w.heavy_scratch_bytes;
  r.local_rows = w.local_rows;
  r.local_rows_bytes = w.local_rows_bytes;
  r.warp_bitmaps = w.warp_bitmaps;
  r.warp_bitmaps_bytes = w.warp_bitmaps_bytes;
  r.heavy_rows = w.heavy_rows;
  r.heavy_rows_bytes = w.heavy_rows_bytes;
  r.fast_dense = w.fast_dense;
  r.fast_dense_bytes = w.fast_dense_bytes;
  r.gtab = w.gtab;
  r.gtab_bytes = w.gtab_bytes;
  r.gbar = w.gbar;
  r.part_dev = w.part_dev;
  r.part_host = w.part_host;
  r.part_words = w.part_words;
  r.tcount = w.tcount;
  r.tcount_bytes = w.tcount_bytes;
  r.k4w = w.k4w;
  r.k4w.lmax = 0;  // the longest list is a property of the graph
  w = WorkSet();
  g_pool_used[r.device] = false;
}

int ensure_scratch(Replica& r, size_t bytes) {
  if (r.scratch_bytes >= bytes) return SMG_OK;
  if (r.scratch) cudaFree(r.scratch);
  r.scratch = nullptr;
  r.scratch_bytes = 0;
  if (bytes == 0) return SMG_OK;
  SMG_CUDA(cudaMalloc(&r.scratch, bytes));
  r.scratch_bytes = bytes;
  return SMG_OK;
}

struct Launch {
  bool meter = false;
  uint64_t unit_begin = 0, unit_end = 0;
  uint32_t root_lo = 0, root_hi = 0;
  bool meter_roots = false;
  uint32_t shard = 0, num_shards = 1;
};

// The cost-balanced shard map of `num_shards` shards for plans with/without
// a level-1 bound, built on r's device and cached on the replica (the graph is
// immutable).  Caller holds r.mu.
int ensure_shard_map(const smg_graph& g, Replica& r, uint32_t num_shards, int unit_bound) {
  if (r.map_shards == num_shards && r.map_unit_bound == unit_bound && r.map_dev &&
      r.map_oriented == r.view_oriented)
    return SMG_OK;
  r.map_shards = 0;  // invalid until rebuilt for this labelling
  r.map_oriented = r.view_oriented;
  const uint64_t nch = (g.slots + kChunk - 1) / kChunk;
  const uint32_t J = num_shards * kShardSplit;
  cudaStream_t st = r.active();
  unsigned long long *cost = nullptr, *pref = nullptr, *bnd = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  std::vector<unsigned long long> bounds(J + 1, 0);
  cudaError_t e = cudaMalloc(&cost, (nch + 1) * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&pref, (nch + 1) * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&bnd, (J + 1) * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cost, pref, nch + 1, st);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 4));
  if (e == cudaSuccess) e = cudaMemsetAsync(cost, 0, (nch + 1) * sizeof(unsigned long long), st);
  if (e == cudaSuccess && nch) {
    chunk_cost_kernel<<<r.num_sms * 8, 256, 0, st>>>(r.off, r.adj, r.src, g.slots, nch, unit_bound, cost);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cost, pref, nch + 1, st);
  if (e == cudaSuccess) {
    shard_bounds_kernel<<<(J + 256) / 256, 256, 0, st>>>(pref, nch, J, bnd);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(bounds.data(), bnd, (J + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(cost);
  cudaFree(pref);
  cudaFree(bnd);
  cudaFree(tmp);
  if (e != cudaSuccess) return fail(SMG_EIO, std::string("shard map: ") + cudaGetErrorString(e));
  // per shard s: begin[K] then pref[K+1]; super-chunk j belongs to shard j % S
  const uint32_t K = kShardSplit, W = 2 * K + 1;
  std::vector<unsigned long long> h(static_cast<size_t>(num_shards) * W, 0);
  for (uint32_t sh = 0; sh < num_shards; ++sh) {
    unsigned long long* b = h.data() + static_cast<size_t>(sh) * W;
    unsigned long long* pr = b + K;
    pr[0] = 0;
    for (uint32_t k = 0; k < K; ++k) {
      const uint32_t j = k * num_shards + sh;
      b[k] = bounds[j];
      pr[k + 1] = pr[k] + (bounds[j + 1] - bounds[j]);
    }
  }
  if (r.map_dev) cudaFree(r.map_dev);
  r.map_dev = nullptr;
  r.map_shards = 0;
  SMG_CUDA(cudaMalloc(&r.map_dev, h.size() * sizeof(unsigned long long)));
  SMG_CUDA(cudaMemcpy(r.map_dev, h.data(), h.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  r.map_bounds = bounds;
  r.map_shards = num_shards;
  r.map_unit_bound = unit_bound;
  return SMG_OK;
}

// Enqueue one shard on replica r (asynchronous).  Caller holds r.mu.
template <bool METER, bool TRACE, int SHAPE>
int enqueue_t(const smg_graph& g, Replica& r, const Program& prog, const Launch& L) {
  const uint64_t cap = std::max<uint64_t>(32, (g.max_degree + 31) / 32 * 32);
  const bool heavy = prog.batch != 0;
  const size_t dyn = SHAPE == kShapeBatch4 ? kBatchDynSmem : kDynSmem;
  SMG_CUDA(cudaFuncSetAttribute(count_kernel<METER, TRACE, SHAPE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
  int per_sm = 0;
  SMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_kernel<METER, TRACE, SHAPE>, kThreads,
                                                         dyn));
  per_sm = std::max(1, per_sm);
  uint64_t blocks = static_cast<uint64_t>(r.num_sms) * per_sm;
  // Keep the per-warp scratch within a budget (sets are at most max_degree).
  const uint64_t per_block = static_cast<uint64_t>(prog.nslots) * cap * 4 * kWarpsPerBlock;
  const uint64_t budget = 24ull << 30;
  if (per_block > 0) blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, budget / per_block));
  int rc = ensure_scratch(r, per_block * blocks);
  if (rc) return rc;
  if (heavy) {
    if (!r.heavy_items)
      SMG_CUDA(cudaMalloc(&r.heavy_items, kHeavyQueueCap * kHeavyItemWords * sizeof(uint32_t)));
    const size_t hs = static_cast<size_t>(r.num_sms) * 4 * (prog.nslots + 1) * cap * 4;  // <= 4 CTAs/SM
    if (r.heavy_scratch_bytes < hs) {
      if (r.heavy_scratch) cudaFree(r.heavy_scratch);
      r.heavy_scratch = nullptr;
      r.heavy_scratch_bytes = 0;
      SMG_CUDA(cudaMalloc(&r.heavy_scratch, std::max<size_t>(hs, 4)));
      r.heavy_scratch_bytes = hs;
    }
  }
  // Per-warp global work areas (radix index / bitmap of a big probe set): only
  // plans with a batched leaf use them, and only if they fit next to
  // everything else (else the kernels fall back to bisection probes).
  const uint64_t bm_words = (g.n + 31) / 32;
  bool use_bitmaps = false;
  if (heavy && !(g_tune & 64u)) {
    const size_t bytes = blocks * kWarpsPerBlock * bm_words * sizeof(uint32_t);
    if (r.warp_bitmaps_bytes >= bytes) {
      use_bitmaps = true;
    } else {
      if (r.warp_bitmaps) cudaFree(r.warp_bitmaps);
      r.warp_bitmaps = nullptr;
      r.warp_bitmaps_bytes = 0;
      size_t free_b = 0, total_b = 0;
      SMG_CUDA(cudaMemGetInfo(&free_b, &total_b));
      if (bytes + (2ull << 30) <= free_b && cudaMalloc(&r.warp_bitmaps, bytes) == cudaSuccess) {
        SMG_CUDA(cudaMemset(r.warp_bitmaps, 0, bytes));
        SMG_CUDA(cudaDeviceSynchronize());
        r.warp_bitmaps_bytes = bytes;
        use_bitmaps = true;
      } else {
        cudaGetLastError();
        r.warp_bitmaps = nullptr;
      }
    }
  }
  const bool clique = !METER && prog.clique;
  if (clique) {
    const size_t lr = blocks * kWarpsPerBlock * kLocalWarpMax * kLocalWarpRowWords * sizeof(uint32_t);
    const size_t hr = static_cast<size_t>(r.num_sms) * 4 * kLocalCtaMax * kLocalRowWords * sizeof(uint32_t);
    if (r.local_rows_bytes < lr) {
      if (r.local_rows) cudaFree(r.local_rows);
      r.local_rows = nullptr;
      r.local_rows_bytes = 0;
      SMG_CUDA(cudaMalloc(&r.local_rows, lr));
      r.local_rows_bytes = lr;
    }
    if (r.heavy_rows_bytes < hr) {
      if (r.heavy_rows) cudaFree(r.heavy_rows);
      r.heavy_rows = nullptr;
      r.heavy_rows_bytes = 0;
      SMG_CUDA(cudaMalloc(&r.heavy_rows, hr));
      r.heavy_rows_bytes = hr;
    }
  }
  cudaStream_t st = r.active();
  SMG_CUDA(cudaMemsetAsync(r.ctr, 0, sizeof(Counters), st));
  SMG_CUDA(cudaEventRecord(r.ev0, st));
  if (METER && L.meter_roots && L.root_hi > L.root_lo) {
    const uint32_t nr = L.root_hi - L.root_lo;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((nr + 255) / 256, 4096));
    meter_roots_kernel<<<grid, 256, 0, st>>>(r.off, r.adj, L.root_lo, L.root_hi, prog.unit_bound, r.ctr);
  }
  KernelArgs a;
  a.off = r.off;
  a.adj = r.adj;
  a.src = r.src;
  a.scratch = r.scratch;
  a.cap = cap;
  a.unit_begin = L.unit_begin;
  a.unit_end = L.unit_end;
  a.nverts = g.n;
  a.tune = g_tune;
  a.heavy_stream = g_heavy_stream;
  a.heavy_min = g_heavy_min;
  a.list_cost = g_list_cost;
  a.shard = L.shard;
  a.num_shards = L.num_shards;
  a.map_begin = nullptr;
  a.map_pref = nullptr;
  a.map_k = 0;
  if (L.num_shards > 1) {
    int mrc = ensure_shard_map(g, r, L.num_shards, prog.unit_bound);
    if (mrc) return mrc;
    a.map_begin = r.map_dev + static_cast<size_t>(L.shard) * (2 * kShardSplit + 1);
    a.map_pref = a.map_begin + kShardSplit;
    a.map_k = kShardSplit;
  }
  a.ctr = r.ctr;
  a.heavy_items = heavy ? r.heavy_items : nullptr;
  a.heavy_cap = heavy ? kHeavyQueueCap : 0;
  a.heavy_scratch = r.heavy_scratch;
  a.local_rows = clique ? r.local_rows : nullptr;
  a.warp_bitmaps = use_bitmaps ? r.warp_bitmaps : nullptr;
  a.bitmap_words = bm_words;
  a.heavy_rows = clique ? r.heavy_rows : nullptr;
  a.prog = prog;
  if (L.unit_end > L.unit_begin) {
    count_kernel<METER, TRACE, SHAPE><<<static_cast<unsigned>(blocks), kThreads, dyn, st>>>(a);
    if (heavy) {
      static_assert(kHeavyCliqueSmem <= kBitmapWords * 4, "clique-local region must fit the bitmap region");
      const size_t hsm = kHeavySmem;
      SMG_CUDA(cudaFuncSetAttribute(heavy_kernel<TRACE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(hsm)));
      int hper = 0;
      SMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hper, heavy_kernel<TRACE>, kHeavyThreads, hsm));
      hper = std::min(kHeavyMinBlocks, std::max(1, hper));
      heavy_kernel<TRACE><<<r.num_sms * hper, kHeavyThreads, hsm, st>>>(a);
    }
  }
  SMG_CUDA(cudaGetLastError());
  SMG_CUDA(cudaEventRecord(r.ev1, st));
  SMG_CUDA(cudaMemcpyAsync(r.host_ctr, r.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  return SMG_OK;
}

int enqueue(const smg_graph& g, Replica& r, const Program& prog, const Launch& L);
int finish(Replica& r, uint64_t* count, uint64_t* elems, uint64_t* units, bool* ovf, double* ms,
           int64_t* count_hi = nullptr);

int ensure_oriented(const smg_graph& g, Replica& r);
int k5_oriented(const smg_graph& g, Replica& r, uint32_t shard, uint32_t num_shards, unsigned long long* count,
                unsigned long long* units, double* ms);

// Number of 5-cliques: a closed-form term of the folded full counts.  The
// per-root count of k4.cu on the degree-ordered copy; the clique plan
// (v0 > v1 > ... > v4: each K5 once) through the generic executor's
// clique-local path if a list exceeds that kernel's capacity.  Cached on the
// replica.  Caller holds r.mu.
int replica_k5(const smg_graph& g, Replica& r, unsigned long long* out) {
  if (!r.k5_valid) {
    unsigned long long c5 = 0, u5 = 0;
    double ms5 = 0;
    const int krc = k5_oriented(g, r, 0, 1, &c5, &u5, &ms5);
    if (krc == SMG_OK) {
      r.k5 = c5;
      r.k5_valid = true;
      *out = r.k5;
      return SMG_OK;
    }
    if (krc != kTryGeneric) return krc;
    smg_plan p;
    std::memset(&p, 0, sizeof(p));
    p.depth = 5;
    for (int i = 0; i < SMG_MAX_LEVELS; ++i) p.parent[i] = -1;
    for (int i = 1; i < 5; ++i) {
      p.isect_mask[i] = static_cast<uint8_t>((1u << i) - 1u);
      p.parent[i] = static_cast<int8_t>(i - 1);
    }
    p.flags = SMG_PLAN_USE_BOUNDS | SMG_PLAN_USE_RESTRICTIONS;
    Program prog;
    const std::string err = compile_program(p, &prog);
    if (!err.empty()) return fail(SMG_EIO, "internal clique plan: " + err);
    Launch L;
    L.unit_begin = 0;
    L.unit_end = g.slots;
    L.root_lo = 0;
    L.root_hi = static_cast<uint32_t>(g.n);
    int rc = enqueue(g, r, prog, L);
    if (rc) return rc;
    uint64_t c = 0, el = 0, u = 0;
    bool ovf = false;
    double ms = 0;
    rc = finish(r, &c, &el, &u, &ovf, &ms);
    if (rc) return rc;
    if (ovf) return fail(SMG_EOVERFLOW, "5-clique count exceeds 64 bits");
    r.k5 = c;
    r.k5_valid = true;
  }
  *out = r.k5;
  return SMG_OK;
}

// The folded closed-form path (tindex.cu) for plans fast_kind() recognises:
// builds the triangle index on first use (cached on the replica), then one
// persistent kernel over the level-1 unit slots.  Same Counters, events and
// result path as enqueue().  Caller holds r.mu.
int enqueue_fast(const smg_graph& g, Replica& r, int kind, const smg_plan& plan, const Launch& L) {
  SMG_CUDA(cudaSetDevice(r.device));
  cudaStream_t st = r.active();
  std::string err;
  const auto tb0 = std::chrono::steady_clock::now();
  const bool full = L.root_lo == 0 && L.root_hi == g.n;
  const bool fullmode = full && fast_has_full(kind);
  if (tindex_build(&r.tix, r.off, r.adj, r.src, g.n, g.slots, r.num_sms, st, kind == kFastStar4,
                   kind == kFastTailedDiamondA || fullmode, &err)) {
    tindex_free(&r.tix);
    return fail(SMG_EIO, "triangle index: " + err);
  }
  if (g_trace)
    std::fprintf(stderr, "[smg trace] triangle index ready in %.1f ms (%llu entries, kind %d)\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb0).count(),
                 static_cast<unsigned long long>(r.tix.entries), kind);
  const bool dense = fast_dense(kind);
  const unsigned blocks = static_cast<unsigned>(r.num_sms) * (dense ? 2 : 4);
  const uint64_t words = fast_scratch_words(kind, g.max_degree);
  // per-slot accumulators and dense per-CTA codegree tables (two-center kinds;
  // the rectangle kinds use an accumulator only for root-range calls).  The
  // accumulators of a completed pass stay valid (the graph is immutable), so
  // later root-range calls of the same kind only run the combine.
  const bool rect = kind == kFastRectangle || kind == kFastRectangleMotif;
  const bool arrays = fast_slot_arrays(kind) > 0 && !(rect && full) && !fullmode;
  const bool combine_only = arrays && !full && r.fast_acc_kind == kind;
  const size_t acc_need = arrays ? static_cast<size_t>(fast_slot_arrays(kind)) * std::max<uint64_t>(g.slots, 1) * 8 : 0;
  const size_t dense_need = dense ? static_cast<size_t>(blocks) * g.n * sizeof(uint32_t) : 0;
  if (acc_need > r.fast_acc_bytes) {
    if (r.fast_acc) cudaFree(r.fast_acc);
    r.fast_acc = nullptr;
    r.fast_acc_bytes = 0;
    r.fast_acc_kind = 0;
    SMG_CUDA(cudaMalloc(&r.fast_acc, acc_need));
    r.fast_acc_bytes = acc_need;
  }
  if (dense_need > r.fast_dense_bytes) {
    if (r.fast_dense) cudaFree(r.fast_dense);
    r.fast_dense = nullptr;
    r.fast_dense_bytes = 0;
    SMG_CUDA(cudaMalloc(&r.fast_dense, dense_need));
    SMG_CUDA(cudaMemsetAsync(r.fast_dense, 0, dense_need, st));
    r.fast_dense_bytes = dense_need;
  }
  const size_t need = static_cast<size_t>(blocks) * (kFastThreads / 32) * words * sizeof(uint32_t);
  if (need > r.fast_scratch_bytes) {
    if (r.fast_scratch) cudaFree(r.fast_scratch);
    r.fast_scratch = nullptr;
    r.fast_scratch_bytes = 0;
    SMG_CUDA(cudaMalloc(&r.fast_scratch, need));
    SMG_CUDA(cudaMemsetAsync(r.fast_scratch, 0, need, st));
    r.fast_scratch_bytes = need;
  }
  FastArgs a;
  std::memset(&a, 0, sizeof(a));
  a.off = r.off;
  a.adj = r.adj;
  a.src = r.src;
  a.n = g.n;
  a.slots = g.slots;
  a.root_lo = L.root_lo;
  a.root_hi = L.root_hi;
  a.e_lo = full ? 0 : L.unit_begin;
  a.e_hi = full ? g.slots : L.unit_end;
  a.via_rev = (!full && fast_center_v1(kind)) ? 1 : 0;
  a.num_shards = L.num_shards;
  if (L.num_shards > 1) {
    int mrc = ensure_shard_map(g, r, L.num_shards, plan.parent[1] == 0 ? 1 : 0);
    if (mrc) return mrc;
    a.map_begin = r.map_dev + static_cast<size_t>(L.shard) * (2 * kShardSplit + 1);
    a.map_pref = a.map_begin + kShardSplit;
    a.map_k = kShardSplit;
  }
  a.t = r.tix;
  a.scratch = r.fast_scratch;
  a.scratch_words = words;
  a.dmax = g.max_degree;
  a.next_chunk = &r.ctr->next_chunk;
  a.next2 = &r.ctr->heavy_next;
  a.acc0 = arrays ? r.fast_acc : nullptr;
  a.acc1 = arrays ? r.fast_acc + g.slots : nullptr;
  a.acc2 = arrays ? r.fast_acc + (fast_slot_arrays(kind) - 1) * g.slots : nullptr;
  a.dense = r.fast_dense;
  a.count = &r.ctr->count;
  a.units = &r.ctr->units;
  a.overflow = &r.ctr->overflow;
  r.post_kind = 0;
  if (fullmode) {
    // closed-form terms (shard 0 carries them): sum_entries k4(k4-1) and K5
    __int128 global = 0;
    if (L.shard == 0) {
      if (!r.k4pairs_valid) {
        if (tindex_k4_pairs(r.tix, r.num_sms, st, &r.k4pairs, &err)) return fail(SMG_EIO, err);
        r.k4pairs_valid = true;
      }
      unsigned long long k5 = 0;
      int krc = replica_k5(g, r, &k5);
      if (krc) return krc;
      const __int128 half = static_cast<__int128>(r.k4pairs / 2), k5x60 = static_cast<__int128>(k5) * 60;
      global = k5x60 - half;  // house: -k4p/2 + 60 K5 (with ego/2); tdb, tda: -(k4p/2 - 60 K5)
    }
    const size_t words = 4 * static_cast<size_t>(blocks);
    if (words > r.part_words) {
      if (r.part_dev) cudaFree(r.part_dev);
      if (r.part_host) cudaFreeHost(r.part_host);
      r.part_dev = nullptr;
      r.part_host = nullptr;
      r.part_words = 0;
      SMG_CUDA(cudaMalloc(&r.part_dev, words * sizeof(unsigned long long)));
      SMG_CUDA(cudaMallocHost(&r.part_host, words * sizeof(unsigned long long)));
      r.part_words = words;
    }
    a.part = r.part_dev;
    r.post_global = global;
    r.post_blocks = blocks;
  }
  SMG_CUDA(cudaMemsetAsync(r.ctr, 0, sizeof(Counters), st));
  SMG_CUDA(cudaEventRecord(r.ev0, st));
  if (fullmode) {
    if (kind != kFastTailedDiamondA) SMG_CUDA(cudaMemsetAsync(r.part_dev, 0, r.part_words * 8, st));
    if (g.slots && fast_launch_full(kind, a, blocks, st)) return fail(SMG_EIO, "folded kernel launch failed");
    SMG_CUDA(cudaMemcpyAsync(r.part_host, r.part_dev, 4 * blocks * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st));
    r.post_kind = kind;
  } else if (g.slots && fast_launch(kind, a, blocks, st, combine_only)) {
    return fail(SMG_EIO, "folded kernel launch failed");
  }
  if (arrays) r.fast_acc_kind = kind;
  SMG_CUDA(cudaGetLastError());
  SMG_CUDA(cudaEventRecord(r.ev1, st));
  SMG_CUDA(cudaMemcpyAsync(r.host_ctr, r.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  return SMG_OK;
}

// ---- label-free full counts on the degree-ordered copy of the CSR ---------
// A plan whose restrictions leave exactly one (or a fixed number) of the
// automorphic embeddings of every instance counts the same total under any
// relabelling of the vertices.  That holds for every clique plan (the
// automorphism group is the full symmetric group, so the number of orderings
// of an instance that satisfy a given set of id constraints does not depend
// on the ids) and for the two rectangle plans fast_kind() recognises.  Their
// full counts run on the orient_reindex copy (graph.cpp:137-161: ids by
// descending degree), where every vertex has few smaller-id neighbours, so the
// v_a < v_b cut-offs prune hub lists first.  Root-range calls, metering and
// SMG_GENERIC calls keep the caller's labelling (per-root counts and E are
// label-dependent).  SMG_RELABEL=0 turns it off.
const int g_relabel = [] {
  const char* e = std::getenv("SMG_RELABEL");
  return (e && *e == '0') ? 0 : 1;
}();

// SMG_K4=0: count 4-cliques through the generic executor instead of k4.cu.
const int g_k4 = [] {
  const char* e = std::getenv("SMG_K4");
  return (e && *e == '0') ? 0 : 1;
}();

// SMG_M4_HUB_DEGREE: degree from which a centre of the 4-cycle pass is scattered
// by the whole grid (tests lower it so small graphs take the hub path).
const uint32_t g_m4_hub = [] {
  const char* e = std::getenv("SMG_M4_HUB_DEGREE");
  const long v = e ? std::atol(e) : 0;
  return v > 0 ? static_cast<uint32_t>(std::min<long>(v, 32768)) : kM4HubDegree;  // group tables hold 16-bit counts
}();
// SMG_M4_GROUP_DEGREE: degree from which a centre takes the group tier (0 = off).
const uint32_t g_m4_group = [] {
  const char* e = std::getenv("SMG_M4_GROUP_DEGREE");
  return e ? static_cast<uint32_t>(std::max<long>(0, std::atol(e))) : kM4GroupDegree;
}();

// First vertex of the degree-ordered CSR (degrees descend with the id) whose
// degree is below `threshold`: a binary search over device offsets.
int first_below(const unsigned long long* off, uint64_t n, uint64_t threshold, uint32_t* out) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    unsigned long long o[2];
    SMG_CUDA(cudaMemcpy(o, off + mid, sizeof(o), cudaMemcpyDeviceToHost));
    if (o[1] - o[0] >= threshold) lo = mid + 1;
    else hi = mid;
  }
  *out = static_cast<uint32_t>(lo);
  return SMG_OK;
}

bool clique_plan(const smg_plan& p) {
  if (p.depth < 3) return false;
  for (uint32_t i = 1; i < p.depth; ++i)
    if (p.isect_mask[i] != static_cast<uint8_t>((1u << i) - 1u) || p.diff_mask[i]) return false;
  return true;
}

int ensure_oriented(const smg_graph& g, Replica& r) {
  if (r.ocsr.off) return SMG_OK;
  SMG_CUDA(cudaSetDevice(r.device));
  DevCSR in;
  in.off = r.off;
  in.adj = r.adj;
  in.src = r.src;
  in.n = g.n;
  in.slots = g.slots;
  in.max_degree = g.max_degree;
  std::string err;
  const auto t0 = std::chrono::steady_clock::now();
  DevCSR o;
  if (device_orient(r.device, r.active(), r.num_sms, in, &o, nullptr, &err)) return fail(SMG_EIO, "orient: " + err);
  r.ocsr = o;
  if (g_trace)
    std::fprintf(stderr, "[smg trace] degree-ordered CSR ready in %.1f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  return SMG_OK;
}

// Points the replica's CSR at the degree-ordered copy for its lifetime.
struct OrientedView {
  Replica& r;
  unsigned long long* off;
  uint32_t* adj;
  uint32_t* src;
  explicit OrientedView(Replica& rep) : r(rep), off(rep.off), adj(rep.adj), src(rep.src) {
    r.off = r.ocsr.off;
    r.adj = r.ocsr.adj;
    r.src = r.ocsr.src;
    r.view_oriented = true;
  }
  ~OrientedView() {
    r.off = off;
    r.adj = adj;
    r.src = src;
    r.view_oriented = false;
  }
  OrientedView(const OrientedView&) = delete;
  OrientedView& operator=(const OrientedView&) = delete;
};

// 1: clique plan (generic executor on the oriented view); 2: the 4-vertex
// kinds with a closed form over subgraph counts (m4_launch); 0: keep the
// caller's labelling.
// 5-cliques of the graph (this shard's roots) through k4.cu on the ordered
// copy.  SMG_OK, kTryGeneric (SMG_K4=0 or a list beyond the kernel's capacity),
// or an error.  Synchronous.  Caller holds r.mu.
int k5_oriented(const smg_graph& g, Replica& r, uint32_t shard, uint32_t num_shards, unsigned long long* count,
                unsigned long long* units, double* ms) {
  if (!g_k4 || !g_relabel) return kTryGeneric;
  SMG_CUDA(cudaSetDevice(r.device));
  int rc = ensure_oriented(g, r);
  if (rc) return rc;
  OrientedView view(r);
  std::string kerr;
  const int krc = k4_count(r.off, r.adj, g.n, shard, num_shards, r.num_sms, r.active(), &r.k4w, nullptr, count, units,
                           ms, &kerr, 5);
  if (krc == 1) return fail(SMG_EIO, kerr);
  if (krc == 3) return fail(SMG_EOVERFLOW, "5-clique count exceeds 64 bits");
  return krc == 0 ? SMG_OK : kTryGeneric;
}

bool clique5_plan(const smg_plan& p) {
  return p.depth == 5 && clique_plan(p) && p.parent[1] == 0 && p.parent[2] == 1 && p.parent[3] == 2 &&
         p.parent[4] == 3;
}

// A fully restricted 4-clique plan (v0 > v1 > v2 > v3: each 4-clique once).
bool clique4_plan(const smg_plan& p) {
  return p.depth == 4 && clique_plan(p) && p.parent[1] == 0 && p.parent[2] == 1 && p.parent[3] == 2;
}

int relabel_mode(const smg_plan& plan, uint32_t flags) {
  if (!g_relabel || (flags & (SMG_METER | SMG_GENERIC))) return 0;
  if (g_fast && g_k4 && (clique4_plan(plan) || clique5_plan(plan))) return 2;  // the per-root counts of k4.cu
  if (clique_plan(plan)) return 1;
  if (!g_fast) return 0;
  M4Weights w;
  return m4_weights(fast_kind(plan), &w) ? 2 : 0;
}

// The closed-form kind of a plan relabel_mode() sends to m4_count.
int m4_kind(const smg_plan& plan) {
  return clique4_plan(plan) ? kFastClique4 : clique5_plan(plan) ? kFastClique5 : fast_kind(plan);
}

int enqueue_oriented(const smg_graph& g, Replica& r, const Program& prog, const Launch& L) {
  int rc = ensure_oriented(g, r);
  if (rc) return rc;
  OrientedView view(r);
  return enqueue(g, r, prog, L);
}

// Full counts of 4-vertex kinds as weighted sums of subgraph counts of the
// whole graph (tindex.cu, m4_launch), this shard's shares: one 4-clique count
// (generic executor), one set of passes over the shard's vertices / edges,
// then each plan's weights on the host.  Synchronous.  Caller holds r.mu.
struct M4Out {
  __int128 share = 0;
  uint64_t units = 0;
  double ms = 0;
};

int m4_count(const smg_graph& g, Replica& r, const int* kinds, const smg_plan* const* plans, uint32_t np,
             const Launch& L, M4Out* out) {
  r.post_kind = 0;
  SMG_CUDA(cudaSetDevice(r.device));  // one host thread per device (m4_count_devices): set it here
  if (np == 1 && kinds[0] == kFastClique5) {
    unsigned long long c5 = 0, u5 = 0;
    double ms5 = 0;
    const int krc = k5_oriented(g, r, L.shard, L.num_shards, &c5, &u5, &ms5);
    if (krc) return krc;  // kTryGeneric: the caller runs the generic executor
    out[0].share = static_cast<__int128>(c5);
    out[0].units = u5;
    out[0].ms = ms5;
    return SMG_OK;
  }
  int rc = ensure_oriented(g, r);
  if (rc) return rc;
  OrientedView view(r);
  M4Weights W[16];
  if (np == 0 || np > 16) return fail(SMG_EINPUT, "bad plan count");
  unsigned need = 0;
  for (uint32_t i = 0; i < np; ++i) {
    if (!m4_weights(kinds[i], &W[i])) return fail(SMG_EIO, "internal: kind has no closed form");
    need |= W[i].need();
  }
  // K4 share: per-root local-graph count on the ordered copy (k4.cu); the
  // clique plan v0 > v1 > v2 > v3 through the generic executor when a root's
  // list exceeds that kernel's capacity, or with SMG_K4=0
  unsigned long long k4 = 0, k4_units = 0;
  double k4_ms = 0;
  bool k4_done = false;
  uint32_t* tcount = nullptr;  // triangles per edge, a by-product of the 4-clique kernels (one shard only)
  if (g_k4) {
    if (need && L.num_shards <= 1 && g.slots) {
      const size_t tb = g.slots * sizeof(uint32_t);
      if (tb > r.tcount_bytes) {
        if (r.tcount) cudaFree(r.tcount);
        r.tcount = nullptr;
        r.tcount_bytes = 0;
        if (cudaMalloc(&r.tcount, tb) == cudaSuccess) r.tcount_bytes = tb;
        else cudaGetLastError();  // no room: the edge pass intersects instead
      }
      if (r.tcount) {
        SMG_CUDA(cudaMemsetAsync(r.tcount, 0, tb, r.active()));
        tcount = r.tcount;
      }
    }
    std::string kerr;
    const int krc = k4_count(r.off, r.adj, g.n, L.shard, L.num_shards, r.num_sms, r.active(), &r.k4w, tcount, &k4,
                             &k4_units, &k4_ms, &kerr);
    if (krc == 1) return fail(SMG_EIO, kerr);
    if (krc == 3) return fail(SMG_EOVERFLOW, "4-clique count exceeds 64 bits");
    k4_done = krc == 0;
  }
  if (!k4_done) tcount = nullptr;
  if (!k4_done) {
    smg_plan p;
    std::memset(&p, 0, sizeof(p));
    p.depth = 4;
    for (int i = 0; i < SMG_MAX_LEVELS; ++i) p.parent[i] = -1;
    for (int i = 1; i < 4; ++i) {
      p.isect_mask[i] = static_cast<uint8_t>((1u << i) - 1u);
      p.parent[i] = static_cast<int8_t>(i - 1);
    }
    p.flags = SMG_PLAN_USE_BOUNDS | SMG_PLAN_USE_RESTRICTIONS;
    Program prog;
    const std::string err = compile_program(p, &prog);
    if (!err.empty()) return fail(SMG_EIO, "internal clique plan: " + err);
    Launch K = L;
    K.meter = false;
    K.meter_roots = false;
    rc = enqueue(g, r, prog, K);
    if (rc) return rc;
    uint64_t c = 0, el = 0, u = 0;
    bool ovf = false;
    rc = finish(r, &c, &el, &u, &ovf, &k4_ms);
    if (rc) return rc;
    if (ovf) return fail(SMG_EOVERFLOW, "4-clique count exceeds 64 bits");
    k4 = c;
    k4_units = u;
  }
  cudaStream_t st = r.active();
  const unsigned blocks = static_cast<unsigned>(r.num_sms) * 2;
  // one dense table (n words) per CTA of c4_kernel: as many as fit in half of
  // the free memory (a graph near the 2^32-vertex limit still gets one)
  unsigned c4_blocks = blocks;
  if (need & (1u << kM4C4)) {
    const size_t table = std::max<uint64_t>(g.n, 1) * sizeof(uint32_t);
    if (static_cast<size_t>(blocks) * table > r.fast_dense_bytes) {
      size_t free_b = 0, total_b = 0;
      SMG_CUDA(cudaMemGetInfo(&free_b, &total_b));
      free_b += r.fast_dense_bytes;  // the current buffer is released first
      c4_blocks = static_cast<unsigned>(std::min<size_t>(blocks, std::max<size_t>(1, free_b / 2 / table)));
      if (static_cast<size_t>(c4_blocks) * table > r.fast_dense_bytes) {
        if (r.fast_dense) cudaFree(r.fast_dense);
        r.fast_dense = nullptr;
        r.fast_dense_bytes = 0;
        SMG_CUDA(cudaMalloc(&r.fast_dense, static_cast<size_t>(c4_blocks) * table));
        SMG_CUDA(cudaMemsetAsync(r.fast_dense, 0, static_cast<size_t>(c4_blocks) * table, st));
        r.fast_dense_bytes = static_cast<size_t>(c4_blocks) * table;
      } else {
        c4_blocks = static_cast<unsigned>(r.fast_dense_bytes / table);
      }
    }
  }
  const size_t words = 2 * static_cast<size_t>(kM4Regions) * blocks;
  if (words > r.part_words) {
    if (r.part_dev) cudaFree(r.part_dev);
    if (r.part_host) cudaFreeHost(r.part_host);
    r.part_dev = nullptr;
    r.part_host = nullptr;
    r.part_words = 0;
    SMG_CUDA(cudaMalloc(&r.part_dev, words * sizeof(unsigned long long)));
    SMG_CUDA(cudaMallocHost(&r.part_host, words * sizeof(unsigned long long)));
    r.part_words = words;
  }
  FastArgs a;
  std::memset(&a, 0, sizeof(a));
  if (need & (1u << kM4Paw)) {  // per-vertex triangle sums live in the per-slot accumulator buffer
    const size_t acc_need = std::max<uint64_t>(g.n, 1) * sizeof(unsigned long long);
    if (acc_need > r.fast_acc_bytes) {
      if (r.fast_acc) cudaFree(r.fast_acc);
      r.fast_acc = nullptr;
      r.fast_acc_bytes = 0;
      SMG_CUDA(cudaMalloc(&r.fast_acc, acc_need));
      r.fast_acc_bytes = acc_need;
    }
    r.fast_acc_kind = 0;  // whatever pass it cached is overwritten
    SMG_CUDA(cudaMemsetAsync(r.fast_acc, 0, acc_need, st));
    a.acc0 = r.fast_acc;
  }
  a.off = r.off;
  a.adj = r.adj;
  a.src = r.src;
  a.n = g.n;
  a.slots = g.slots;
  a.root_hi = static_cast<uint32_t>(g.n);
  a.e_hi = g.slots;
  a.num_shards = L.num_shards;
  a.shard = L.shard;
  a.units_per_edge = 1;
  a.c4_blocks = c4_blocks;
  a.tcount = tcount;
  if (need & (1u << kM4C4)) {
    if (!r.tiers_valid) {
      SMG_CUDA(cudaStreamSynchronize(st));
      int trc = first_below(r.off, g.n, g_m4_hub, &r.hub_count);
      if (trc) return trc;
      r.group_end = r.hub_count;
      if (r.hub_count > kM4MaxHubs) {
        // more hubs than the launch loop takes: the rest go one CTA each (32-bit
        // tables); no group tier, its 16-bit counters assume degrees below the hub degree
        r.hub_count = r.group_end = kM4MaxHubs;
      } else if (g_m4_group && g_m4_group < g_m4_hub) {
        trc = first_below(r.off, g.n, g_m4_group, &r.group_end);
        if (trc) return trc;
        r.group_end = std::max(r.group_end, r.hub_count);
      }
      r.tiers_valid = true;
    }
    a.hub_count = r.hub_count;
    a.group_end = r.group_end;
    if (a.group_end > a.hub_count) {
      // as many group tables as stay L2-resident together (about 64 MB), at most 16
      const size_t table = m4_group_table_words(g.n) * sizeof(uint32_t);
      const uint32_t groups = static_cast<uint32_t>(std::min<size_t>(16, std::max<size_t>(1, (64u << 20) / table)));
      const size_t need_bytes = groups * table;
      if (need_bytes > r.gtab_bytes) {
        if (r.gtab) cudaFree(r.gtab);
        r.gtab = nullptr;
        r.gtab_bytes = 0;
        SMG_CUDA(cudaMalloc(&r.gtab, need_bytes));
        SMG_CUDA(cudaMemsetAsync(r.gtab, 0, need_bytes, st));
        r.gtab_bytes = need_bytes;
      }
      if (!r.gbar) SMG_CUDA(cudaMalloc(&r.gbar, 16 * sizeof(unsigned long long)));
      a.groups = groups;
      a.gtab = r.gtab;
      a.gbar = r.gbar;
    }
  }
  a.dmax = g.max_degree;
  a.dense = r.fast_dense;
  a.part = r.part_dev;
  a.next_chunk = &r.ctr->next_chunk;
  a.next2 = &r.ctr->heavy_next;
  a.count = &r.ctr->count;
  a.units = &r.ctr->units;
  a.overflow = &r.ctr->overflow;
  SMG_CUDA(cudaMemsetAsync(r.ctr, 0, sizeof(Counters), st));
  SMG_CUDA(cudaEventRecord(r.ev0, st));
  for (cudaEvent_t& e : r.phase_ev)
    if (!e) SMG_CUDA(cudaEventCreate(&e));
  if (g.slots && need && m4_launch(a, need, blocks, st, r.phase_ev))
    return fail(SMG_EIO, "4-vertex closed-form kernel launch failed");
  if (!(g.slots && need))
    for (cudaEvent_t e : r.phase_ev) SMG_CUDA(cudaEventRecord(e, st));
  SMG_CUDA(cudaGetLastError());
  SMG_CUDA(cudaEventRecord(r.ev1, st));
  SMG_CUDA(cudaMemcpyAsync(r.part_host, r.part_dev, words * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  SMG_CUDA(cudaMemcpyAsync(r.host_ctr, r.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  SMG_CUDA(cudaStreamSynchronize(st));
  float t = 0.f;
  SMG_CUDA(cudaEventElapsedTime(&t, r.ev0, r.ev1));
  r.phase_ms[0] = k4_ms;
  for (int q = 0; q < 3; ++q) {
    float pt = 0.f;
    SMG_CUDA(cudaEventElapsedTime(&pt, r.phase_ev[q], r.phase_ev[q + 1]));
    r.phase_ms[q + 1] = pt;
  }
  __int128 S[kM4Regions];
  for (int q = 0; q < kM4Regions; ++q) {
    S[q] = 0;
    if (!g.slots || !need) continue;
    for (unsigned b = 0; b < blocks; ++b) {
      const size_t i = 2 * (static_cast<size_t>(q) * blocks + b);
      S[q] += static_cast<__int128>((static_cast<unsigned __int128>(r.part_host[i + 1]) << 64) | r.part_host[i]);
    }
  }
  if (g_trace)
    std::fprintf(stderr, "[smg trace] m4 sums: K4=%llu (%.1f ms) C4=%.6g D=%.6g T3=%.6g P4E=%.6g PAW=%.6g STAR=%.6g (%.1f ms)\n",
                 k4, k4_ms, static_cast<double>(S[kM4C4]), static_cast<double>(S[kM4D]),
                 static_cast<double>(S[kM4T3]), static_cast<double>(S[kM4P4E]), static_cast<double>(S[kM4Paw]),
                 static_cast<double>(S[kM4Star]), t);
  for (uint32_t i = 0; i < np; ++i) {
    __int128 v = static_cast<__int128>(k4) * W[i].k4;
    for (int q = 0; q < kM4Regions; ++q) v += S[q] * W[i].w[q];
    out[i].share = v;
    out[i].units = (need ? r.host_ctr->units : k4_units) * (plans[i]->parent[1] == 0 ? 1u : 2u);
    out[i].ms = (static_cast<double>(t) + k4_ms) / np;
  }
  return SMG_OK;
}

void m4_store(const M4Out& o, smg_result* out) {
  out->count = static_cast<uint64_t>(o.share);
  out->count_hi = static_cast<int64_t>(o.share >> 64);
  out->units = o.units;
  out->kernel_ms = o.ms;
  out->per_gpu[0] = out->count;
}

// The folded kernel for this call, or kFastNone.  range: a root-range call.
int fast_for(const smg_plan& plan, uint32_t flags, bool range = false) {
  if (!g_fast || (flags & (SMG_METER | SMG_GENERIC))) return kFastNone;
  const int k = fast_kind(plan);
  if (range && !(flags & SMG_FOLDED_RANGE) && (fast_dense(k) || fast_slot_arrays(k))) return kFastNone;
  return k;
}

int enqueue(const smg_graph& g, Replica& r, const Program& prog, const Launch& L) {
  SMG_CUDA(cudaSetDevice(r.device));
  if (prog.batch && prog.depth == 4) {
    if (L.meter)
      return g_trace ? enqueue_t<true, true, kShapeBatch4>(g, r, prog, L)
                     : enqueue_t<true, false, kShapeBatch4>(g, r, prog, L);
    return g_trace ? enqueue_t<false, true, kShapeBatch4>(g, r, prog, L)
                   : enqueue_t<false, false, kShapeBatch4>(g, r, prog, L);
  }
  if (L.meter)
    return g_trace ? enqueue_t<true, true, kShapeGeneric>(g, r, prog, L)
                   : enqueue_t<true, false, kShapeGeneric>(g, r, prog, L);
  return g_trace ? enqueue_t<false, true, kShapeGeneric>(g, r, prog, L)
                 : enqueue_t<false, false, kShapeGeneric>(g, r, prog, L);
}

// count_hi (may be null): high 64 bits of a signed shard share (folded
// full-count kinds); with count_hi == null a share outside [0, 2^64) is an
// overflow.
int finish(Replica& r, uint64_t* count, uint64_t* elems, uint64_t* units, bool* ovf, double* ms,
           int64_t* count_hi) {
  SMG_CUDA(cudaSetDevice(r.device));
  SMG_CUDA(cudaStreamSynchronize(r.active()));
  float t = 0.f;
  SMG_CUDA(cudaEventElapsedTime(&t, r.ev0, r.ev1));
  *count = r.host_ctr->count;
  *elems = r.host_ctr->elements;
  *units = r.host_ctr->units;
  *ovf = r.host_ctr->overflow != 0;
  *ms = t;
  if (count_hi) *count_hi = 0;
  if (r.post_kind) {
    // centre partials [0, B), ego partials [B, 2B) as (lo, hi) pairs
    __int128 center = 0, ego = 0;
    for (unsigned i = 0; i < 2 * r.post_blocks; ++i) {
      const __int128 v = static_cast<__int128>(
          (static_cast<unsigned __int128>(r.part_host[2 * i + 1]) << 64) | r.part_host[2 * i]);
      (i < r.post_blocks ? center : ego) += v;
    }
    __int128 total = r.post_global;
    if (r.post_kind == kFastTailedDiamondA) total += static_cast<__int128>(r.host_ctr->count);
    else total += center + (r.post_kind == kFastHouse ? ego / 2 : ego);
    r.post_kind = 0;
    *count = static_cast<uint64_t>(total);
    if (count_hi) *count_hi = static_cast<int64_t>(total >> 64);
    else if (total < 0 || (total >> 64) != 0) *ovf = true;
  }
  if (g_trace) {
    static const char* names[kTrCount] = {"units", "build_cycles", "batch_cycles", "batches",
                                          "batches_hashed", "stream_elems", "search_lists",
                                          "probe_set_sum", "stream_set_sum", "leaf_cycles",
                                          "leaves", "bigP_stream_cycles", "deferred",
                                          "heavy_items", "heavy_cycles", "long_lists",
                                          "heavy_build_cycles", "heavy_stream_cycles",
                                          "warp_busy_sum_ns", "warp_busy_max_ns", "heavy_elems",
                                          "heavy_tiles"};
    std::fprintf(stderr, "[smg trace] kernel %.3f ms:", t);
    for (int i = 0; i < kTrCount; ++i)
      std::fprintf(stderr, " %s=%.4g", names[i], static_cast<double>(r.host_ctr->trace[i]));
    std::fprintf(stderr, "\n");
  }
  return SMG_OK;
}

int prepare(const smg_graph* g, const smg_plan* plan, Program* prog) {
  if (!g || !plan) return fail(SMG_EINPUT, "null graph or plan");
  const std::string err = compile_program(*plan, prog);
  if (!err.empty()) return fail(SMG_EINPUT, err);
  return SMG_OK;
}

}  // namespace smg

using namespace smg;

extern "C" {

int smg_abi_version(void) { return 2; }

const char* smg_last_error(void) { return g_last_error.c_str(); }

int smg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int smg_plan_validate(const smg_plan* plan) {
  if (!plan) return fail(SMG_EINPUT, "null plan");
  const std::string err = validate_plan(*plan);
  if (!err.empty()) return fail(SMG_EINPUT, err);
  return SMG_OK;
}

int smg_plan_describe(const smg_plan* plan, char* buf, size_t cap) {
  if (!plan || !buf) return fail(SMG_EINPUT, "null argument");
  Program pr;
  const std::string err = compile_program(*plan, &pr);
  if (!err.empty()) return fail(SMG_EINPUT, err);
  auto node_json = [](const Node& nd) {
    std::string s = "{\"k\":" + std::to_string(nd.k) + ",\"src\":" + std::to_string(nd.src) +
                    ",\"list\":" + std::to_string(nd.list) + ",\"bound\":" + std::to_string(nd.bound) +
                    ",\"raw\":" + std::to_string(nd.raw) + ",\"slot\":" + std::to_string(nd.slot) +
                    ",\"ops\":[";
    for (int o = 0; o < nd.nops; ++o) {
      if (o) s += ",";
      s += "[" + std::to_string(nd.ops[o].level) + "," + std::to_string(nd.ops[o].mode) + "]";
    }
    return s + "]}";
  };
  std::string s = "{\"depth\":" + std::to_string(pr.depth) + ",\"unit_bound\":" +
                  std::to_string(pr.unit_bound) + ",\"nslots\":" + std::to_string(pr.nslots) +
                  ",\"nodes\":[";
  for (int t = 0; t < pr.nnodes; ++t) s += (t ? "," : "") + node_json(pr.nodes[t]);
  s += "],\"cand\":[";
  for (int i = 0; i < pr.depth; ++i) s += (i ? "," : "") + std::to_string(pr.cand[i]);
  s += "],\"node_begin\":[";
  for (int i = 0; i < pr.depth; ++i) s += (i ? "," : "") + std::to_string(pr.node_begin[i]);
  s += "],\"node_end\":[";
  for (int i = 0; i < pr.depth; ++i) s += (i ? "," : "") + std::to_string(pr.node_end[i]);
  s += "],\"leaf\":" + (pr.depth >= 3 ? node_json(pr.leaf) : std::string("null"));
  s += ",\"batch\":" + std::to_string(pr.batch) + ",\"batch_diff\":" + std::to_string(pr.batch_diff) +
       ",\"batch_yltx\":" + std::to_string(pr.batch_yltx) +
       ",\"batch_fixed_bound\":" + std::to_string(pr.batch_fixed_bound) +
       ",\"clique\":" + std::to_string(pr.clique) + ",\"fast\":" + std::to_string(fast_kind(*plan)) +
       // how a full count runs: 0 caller's labels, 1 generic executor on the degree-ordered copy,
       // 2 closed form / per-root clique kernel on the copy (full_kind: FastKind incl. 10, 11)
       ",\"full_count_mode\":" + std::to_string(relabel_mode(*plan, 0)) +
       ",\"full_kind\":" + std::to_string(relabel_mode(*plan, 0) == 2 ? m4_kind(*plan) : 0) + ",\"parent\":[";
  for (int i = 0; i < pr.depth; ++i) s += (i ? "," : "") + std::to_string(pr.parent[i]);
  s += "]}";
  if (s.size() + 1 > cap) return fail(SMG_EINPUT, "buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return SMG_OK;
}

void smg_graph_destroy(smg_graph* g) {
  if (!g) return;
  for (Replica* r : g->reps) {
    if (r->device >= 0) cudaSetDevice(r->device);
    if (r->off) cudaFree(r->off);
    if (r->adj) cudaFree(r->adj);
    if (r->src) cudaFree(r->src);
    park_work(*r);  // per-warp scratch, queues and bitmaps go to the device's pool
    if (r->ctr) cudaFree(r->ctr);
    if (r->map_dev) cudaFree(r->map_dev);
    tindex_free(&r->tix);
    if (r->fast_scratch) cudaFree(r->fast_scratch);
    if (r->fast_acc) cudaFree(r->fast_acc);
    if (r->fast_dense) cudaFree(r->fast_dense);
    if (r->gtab) cudaFree(r->gtab);
    if (r->gbar) cudaFree(r->gbar);
    k4_free(&r->k4w);
    if (r->tcount) cudaFree(r->tcount);
    if (r->ocsr.off) cudaFree(r->ocsr.off);
    if (r->ocsr.adj) cudaFree(r->ocsr.adj);
    if (r->ocsr.src) cudaFree(r->ocsr.src);
    if (r->part_dev) cudaFree(r->part_dev);
    if (r->part_host) cudaFreeHost(r->part_host);
    if (r->host_ctr) cudaFreeHost(r->host_ctr);
    if (r->ev0) cudaEventDestroy(r->ev0);
    if (r->ev1) cudaEventDestroy(r->ev1);
    for (cudaEvent_t e : r->phase_ev)
      if (e) cudaEventDestroy(e);
    if (r->stream) cudaStreamDestroy(r->stream);
    delete r;
  }
  delete g;
}

int smg_graph_create(const uint64_t* offsets, const uint32_t* adjacency, uint64_t n,
                     const int* devices, int num_devices, smg_graph** out) {
  if (!out) return fail(SMG_EINPUT, "null output handle");
  *out = nullptr;
  if (!offsets) return fail(SMG_EINPUT, "null offsets");
  if (n >= (1ull << 32)) return fail(SMG_EINPUT, "vertex ids must fit in 32 bits");
  if (num_devices < 1 || num_devices > SMG_MAX_GPUS) return fail(SMG_EINPUT, "num_devices must be 1..8");
  if (offsets[0] != 0) return fail(SMG_EINPUT, "offsets[0] must be 0");
  const uint64_t slots = offsets[n];
  if (slots && !adjacency) return fail(SMG_EINPUT, "null adjacency");
  int ndev = smg_device_count();
  if (ndev == 0) return fail(SMG_EIO, "no CUDA device available (the engine has no CPU path)");
  smg_graph* g = new smg_graph;
  g->n = n;
  g->slots = slots;
  g->max_degree = 0;
  for (int i = 0; i < num_devices; ++i) {
    const int dev = devices ? devices[i] : i;
    if (dev < 0 || dev >= ndev) {
      smg_graph_destroy(g);
      return fail(SMG_EINPUT, "device index out of range");
    }
    Replica* r = new Replica;
    g->reps.push_back(r);
    r->device = dev;
    adopt_work(*r);
    auto step = [&](cudaError_t e, const char* what) {
      if (e != cudaSuccess) {
        g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
        return false;
      }
      return true;
    };
    bool ok = step(cudaSetDevice(dev), "cudaSetDevice") &&
              step(cudaDeviceGetAttribute(&r->num_sms, cudaDevAttrMultiProcessorCount, dev),
                   "cudaDeviceGetAttribute") &&
              step(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking), "stream") &&
              step(cudaEventCreate(&r->ev0), "event") && step(cudaEventCreate(&r->ev1), "event") &&
              step(cudaMalloc(&r->off, (n + 1) * sizeof(unsigned long long)), "cudaMalloc offsets") &&
              step(cudaMalloc(&r->adj, std::max<uint64_t>(slots, 1) * sizeof(uint32_t)), "cudaMalloc adj") &&
              step(cudaMalloc(&r->src, std::max<uint64_t>(slots, 1) * sizeof(uint32_t)), "cudaMalloc src") &&
              step(cudaMalloc(&r->ctr, sizeof(Counters)), "cudaMalloc counters") &&
              step(cudaMallocHost(&r->host_ctr, sizeof(Counters)), "cudaMallocHost") &&
              step(cudaMemcpyAsync(r->off, offsets, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, r->stream), "H2D offsets") &&
              (slots == 0 || step(cudaMemcpyAsync(r->adj, adjacency, slots * sizeof(uint32_t), cudaMemcpyHostToDevice, r->stream), "H2D adjacency"));
    // Replica 0 is validated on its device (later copies are byte-identical):
    // offsets first (so every slice is in bounds), then the slot map, then
    // the slots themselves.
    unsigned int herr = 0;
    unsigned long long hmax = 0;
    unsigned int* derr = reinterpret_cast<unsigned int*>(&r->ctr->overflow);
    unsigned long long* dmax = &r->ctr->count;
    if (ok && i == 0) {
      ok = step(cudaMemsetAsync(r->ctr, 0, sizeof(Counters), r->stream), "memset");
      if (ok && n > 0) {
        validate_offsets_kernel<<<r->num_sms * 4, 256, 0, r->stream>>>(r->off, n, slots, derr, dmax);
        ok = step(cudaGetLastError(), "validate offsets") &&
             step(cudaMemcpyAsync(&herr, derr, sizeof(herr), cudaMemcpyDeviceToHost, r->stream), "D2H") &&
             step(cudaStreamSynchronize(r->stream), "validate offsets");
      }
    }
    if (ok && !herr && n > 0) {
      fill_src_kernel<<<r->num_sms * 8, 256, 0, r->stream>>>(r->off, n, r->src);
      ok = step(cudaGetLastError(), "fill_src");
    }
    if (ok && i == 0 && !herr && n > 0) {
      if (slots > 0) {
        validate_slots_kernel<<<r->num_sms * 8, 256, 0, r->stream>>>(r->off, r->adj, r->src, n, slots, derr);
        ok = step(cudaGetLastError(), "validate slots");
      }
      ok = ok && step(cudaMemcpyAsync(&herr, derr, sizeof(herr), cudaMemcpyDeviceToHost, r->stream), "D2H") &&
           step(cudaMemcpyAsync(&hmax, dmax, sizeof(hmax), cudaMemcpyDeviceToHost, r->stream), "D2H") &&
           step(cudaStreamSynchronize(r->stream), "validate slots");
    }
    if (ok && i == 0) {
      if (herr || hmax >= (1ull << 32)) {
        static const char* msgs[] = {"degree too large",
                                     "offsets must be non-decreasing and end at the slot count",
                                     "adjacency id out of range", "self loop in adjacency",
                                     "neighbour lists must be strictly ascending",
                                     "adjacency must be symmetric (missing reverse edge)"};
        smg_graph_destroy(g);
        return fail(SMG_EINPUT, msgs[herr < 6 ? herr : 0]);
      }
      g->max_degree = hmax;
    }
    ok = ok && step(cudaStreamSynchronize(r->stream), "upload");
    if (!ok) {
      smg_graph_destroy(g);
      return SMG_EIO;
    }
  }
  *out = g;
  return SMG_OK;
}

// Runtime parts of a replica (stream, events, counters) on `dev`.  Only a
// replica that is kept (`keep`) adopts the device's parked work buffers; a
// temporary one (smg_graph_from_edges' build stream) must not, or they leak.
static int init_replica_runtime(Replica* r, int dev, bool keep) {
  r->device = dev;
  if (keep) adopt_work(*r);
  SMG_CUDA(cudaSetDevice(dev));
  SMG_CUDA(cudaDeviceGetAttribute(&r->num_sms, cudaDevAttrMultiProcessorCount, dev));
  SMG_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
  SMG_CUDA(cudaEventCreate(&r->ev0));
  SMG_CUDA(cudaEventCreate(&r->ev1));
  SMG_CUDA(cudaMalloc(&r->ctr, sizeof(Counters)));
  SMG_CUDA(cudaMallocHost(&r->host_ctr, sizeof(Counters)));
  return SMG_OK;
}

// Wrap a device CSR built on devs[0] into a graph replicated on devs.
static int adopt_device_csr(const DevCSR& csr, const int* devs, int ndevs, smg_graph** out) {
  smg_graph* g = new smg_graph;
  g->n = csr.n;
  g->slots = csr.slots;
  g->max_degree = csr.max_degree;
  for (int i = 0; i < ndevs; ++i) {
    Replica* r = new Replica;
    g->reps.push_back(r);
    int rc = init_replica_runtime(r, devs[i], true);
    if (rc) {
      if (i == 0) {  // still owns the arrays
        cudaFree(csr.off);
        cudaFree(csr.adj);
        cudaFree(csr.src);
      }
      smg_graph_destroy(g);
      return rc;
    }
    if (i == 0) {
      r->off = csr.off;
      r->adj = csr.adj;
      r->src = csr.src;
      continue;
    }
    const size_t ob = (csr.n + 1) * sizeof(unsigned long long), sb = std::max<uint64_t>(csr.slots, 1) * 4;
    cudaError_t e = cudaMalloc(&r->off, ob);
    if (e == cudaSuccess) e = cudaMalloc(&r->adj, sb);
    if (e == cudaSuccess) e = cudaMalloc(&r->src, sb);
    // UVA: device-to-device (NVLink peer path where enabled)
    if (e == cudaSuccess) e = cudaMemcpy(r->off, csr.off, ob, cudaMemcpyDefault);
    if (e == cudaSuccess) e = cudaMemcpy(r->adj, csr.adj, sb, cudaMemcpyDefault);
    if (e == cudaSuccess) e = cudaMemcpy(r->src, csr.src, sb, cudaMemcpyDefault);
    if (e != cudaSuccess) {
      smg_graph_destroy(g);
      return fail(SMG_EIO, std::string("replicate CSR: ") + cudaGetErrorString(e));
    }
  }
  *out = g;
  return SMG_OK;
}

int smg_graph_from_edges(const uint32_t* pairs, uint64_t num_edges, uint64_t n, const int* devices,
                         int num_devices, smg_graph** out, uint64_t* dups, uint64_t* loops) {
  if (!out) return fail(SMG_EINPUT, "null output handle");
  *out = nullptr;
  if (n >= (1ull << 32)) return fail(SMG_EINPUT, "vertex ids must fit in 32 bits");
  if (num_edges && !pairs) return fail(SMG_EINPUT, "null edge array");
  if (num_devices < 1 || num_devices > SMG_MAX_GPUS) return fail(SMG_EINPUT, "num_devices must be 1..8");
  const int ndev = smg_device_count();
  if (ndev == 0) return fail(SMG_EIO, "no CUDA device available (the engine has no CPU path)");
  int devs[SMG_MAX_GPUS];
  for (int i = 0; i < num_devices; ++i) {
    devs[i] = devices ? devices[i] : i;
    if (devs[i] < 0 || devs[i] >= ndev) return fail(SMG_EINPUT, "device index out of range");
  }
  Replica tmp;
  int rc = init_replica_runtime(&tmp, devs[0], false);
  auto release_tmp = [&tmp] {
    if (tmp.stream) cudaStreamDestroy(tmp.stream);
    if (tmp.ev0) cudaEventDestroy(tmp.ev0);
    if (tmp.ev1) cudaEventDestroy(tmp.ev1);
    if (tmp.ctr) cudaFree(tmp.ctr);
    if (tmp.host_ctr) cudaFreeHost(tmp.host_ctr);
    tmp.stream = nullptr;
  };
  if (rc) {
    release_tmp();
    return rc;
  }
  DevCSR csr;
  uint64_t d = 0, l = 0;
  std::string err;
  rc = device_from_edges(devs[0], tmp.stream, tmp.num_sms, pairs, num_edges, n, &csr, &d, &l, &err);
  release_tmp();
  if (rc) return fail(rc == 2 ? SMG_EINPUT : SMG_EIO, err);
  if (dups) *dups = d;
  if (loops) *loops = l;
  return adopt_device_csr(csr, devs, num_devices, out);
}

int smg_graph_orient(const smg_graph* g, int replica, smg_graph** out, uint32_t* new_to_old) {
  if (!g || !out) return fail(SMG_EINPUT, "null argument");
  *out = nullptr;
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  DevCSR in;
  in.off = r.off;
  in.adj = r.adj;
  in.src = r.src;
  in.n = g->n;
  in.slots = g->slots;
  in.max_degree = g->max_degree;
  DevCSR o;
  std::string err;
  const int rc = device_orient(r.device, r.stream, r.num_sms, in, &o, new_to_old, &err);
  if (rc) return fail(SMG_EIO, err);
  const int dev = r.device;
  return adopt_device_csr(o, &dev, 1, out);
}

int smg_graph_download(const smg_graph* g, int replica, uint64_t* offsets, uint32_t* adjacency) {
  if (!g || !offsets) return fail(SMG_EINPUT, "null argument");
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  const Replica& r = *g->reps[replica];
  SMG_CUDA(cudaSetDevice(r.device));
  SMG_CUDA(cudaMemcpy(offsets, r.off, (g->n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (g->slots) {
    if (!adjacency) return fail(SMG_EINPUT, "null adjacency");
    SMG_CUDA(cudaMemcpy(adjacency, r.adj, g->slots * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  }
  return SMG_OK;
}

int smg_graph_set_stream(smg_graph* g, int replica, void* stream) {
  if (!g || replica < 0 || replica >= static_cast<int>(g->reps.size()))
    return fail(SMG_EINPUT, "bad graph or replica");
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  r.user_stream = static_cast<cudaStream_t>(stream);
  return SMG_OK;
}

int smg_phase_times(const smg_graph* g, int replica, double* ms) {
  if (!g || !ms) return fail(SMG_EINPUT, "null argument");
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  for (int q = 0; q < 4; ++q) ms[q] = r.phase_ms[q];
  return SMG_OK;
}

int smg_graph_info(const smg_graph* g, uint64_t* n, uint64_t* slots, uint64_t* maxd, int* ndev) {
  if (!g) return fail(SMG_EINPUT, "null graph");
  if (n) *n = g->n;
  if (slots) *slots = g->slots;
  if (maxd) *maxd = g->max_degree;
  if (ndev) *ndev = static_cast<int>(g->reps.size());
  return SMG_OK;
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int smg_count_shard(const smg_graph* g, const smg_plan* plan, int replica, uint32_t shard,
                    uint32_t num_shards, uint32_t flags, smg_result* out) {
  const double t0 = now_ms();
  if (!out) return fail(SMG_EINPUT, "null result");
  std::memset(out, 0, sizeof(*out));
  Program prog;
  int rc = prepare(g, plan, &prog);
  if (rc) return rc;
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  if (num_shards == 0 || shard >= num_shards) return fail(SMG_EINPUT, "bad shard");
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  Launch L;
  L.meter = (flags & SMG_METER) != 0;
  L.unit_begin = 0;
  L.unit_end = g->slots;
  L.root_lo = 0;
  L.root_hi = static_cast<uint32_t>(g->n);
  L.meter_roots = (shard == 0);
  L.shard = shard;
  L.num_shards = num_shards;
  const int fk = fast_for(*plan, flags);
  const int rm = relabel_mode(*plan, flags);
  if (rm == 2) {
    M4Out o;
    const int mk = m4_kind(*plan);
    rc = m4_count(*g, r, &mk, &plan, 1, L, &o);
    if (rc && rc != kTryGeneric) return rc;
    if (rc == SMG_OK) {
      m4_store(o, out);
      out->wall_ms = now_ms() - t0;
      return SMG_OK;
    }
  }
  rc = rm >= 1 ? enqueue_oriented(*g, r, prog, L)
       : fk    ? enqueue_fast(*g, r, fk, *plan, L)
               : enqueue(*g, r, prog, L);
  if (rc) return rc;
  bool ovf = false;
  rc = finish(r, &out->count, &out->elements, &out->units, &ovf, &out->kernel_ms, &out->count_hi);
  if (rc) return rc;
  out->per_gpu[0] = out->count;
  out->wall_ms = now_ms() - t0;
  if (ovf) return fail(SMG_EOVERFLOW, "embedding count exceeds 64 bits");
  return SMG_OK;
}

int smg_enumerate(const smg_graph* g, const smg_plan* plan, int replica, int has_limit,
                  uint64_t limit, uint32_t* out, uint64_t cap_tuples, uint64_t* n_out) {
  if (!n_out) return fail(SMG_EINPUT, "null n_out");
  *n_out = 0;
  Program prog;
  int rc = prepare(g, plan, &prog);
  if (rc) return rc;
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  if (has_limit && limit == 0) return SMG_OK;  // engine.cpp:184
  const unsigned long long lim = has_limit ? limit : ~0ull;
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  SMG_CUDA(cudaSetDevice(r.device));
  cudaStream_t st = r.active();
  const uint64_t cap = std::max<uint64_t>(32, (g->max_degree + 31) / 32 * 32);
  SMG_CUDA(cudaFuncSetAttribute(enum_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kDynSmem)));
  SMG_CUDA(cudaFuncSetAttribute(enum_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kDynSmem)));
  const uint64_t blocks = static_cast<uint64_t>(r.num_sms) * 2;
  rc = ensure_scratch(r, (prog.nslots + 1) * cap * 4 * kWarpsPerBlock * blocks);
  if (rc) return rc;
  const uint64_t kSlotChunk = 1ull << 22;
  unsigned long long *uval = nullptr, *uoff = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  SMG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, uval, uoff, kSlotChunk + 1, st));
  SMG_CUDA(cudaMalloc(&uval, (kSlotChunk + 1) * sizeof(unsigned long long)));
  SMG_CUDA(cudaMalloc(&uoff, (kSlotChunk + 1) * sizeof(unsigned long long)));
  SMG_CUDA(cudaMalloc(&tmp, tmp_bytes));
  uint32_t* dout = nullptr;
  size_t dout_cap = 0;
  KernelArgs a;
  std::memset(&a, 0, sizeof(a));
  a.off = r.off;
  a.adj = r.adj;
  a.src = r.src;
  a.scratch = r.scratch;
  a.cap = cap;
  a.ctr = r.ctr;
  a.nverts = g->n;
  a.tune = g_tune;
  a.heavy_stream = g_heavy_stream;
  a.heavy_min = g_heavy_min;
  a.list_cost = g_list_cost;
  a.prog = prog;
  unsigned long long total = 0;
  int status = SMG_OK;
  for (uint64_t lo = 0; lo < g->slots && total < lim && status == SMG_OK; lo += kSlotChunk) {
    const uint64_t hi = std::min<uint64_t>(g->slots, lo + kSlotChunk);
    const uint64_t ns = hi - lo;
    cudaError_t e = cudaMemsetAsync(r.ctr, 0, sizeof(Counters), st);
    if (e == cudaSuccess) {
      enum_kernel<false><<<static_cast<unsigned>(blocks), kThreads, kDynSmem, st>>>(a, lo, hi, uval, 0, nullptr);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(uval + ns, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, uval, uoff, ns + 1, st);
    unsigned long long chunk_total = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&chunk_total, uoff + ns, sizeof(chunk_total), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      status = fail(SMG_EIO, std::string("enumerate count pass: ") + cudaGetErrorString(e));
      break;
    }
    const unsigned long long take = std::min<unsigned long long>(chunk_total, lim - total);
    const unsigned long long room = total < cap_tuples ? cap_tuples - total : 0;
    const unsigned long long keep = std::min(take, room);  // tuples copied to the caller
    if (keep && out) {
      const size_t need = keep * prog.depth * sizeof(uint32_t);
      if (need > dout_cap) {
        if (dout) cudaFree(dout);
        dout = nullptr;
        e = cudaMalloc(&dout, need);
        dout_cap = e == cudaSuccess ? need : 0;
      }
      if (e == cudaSuccess) e = cudaMemsetAsync(r.ctr, 0, sizeof(Counters), st);
      if (e == cudaSuccess) {
        // uoff holds the unit offsets within the chunk: write tuples < keep
        enum_kernel<true><<<static_cast<unsigned>(blocks), kThreads, kDynSmem, st>>>(a, lo, hi, uoff, keep, dout);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(out + total * prog.depth, dout, need, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) status = fail(SMG_EIO, std::string("enumerate write pass: ") + cudaGetErrorString(e));
    }
    total += take;
  }
  cudaFree(uval);
  cudaFree(uoff);
  cudaFree(tmp);
  if (dout) cudaFree(dout);
  *n_out = total;
  return status;
}

int smg_shard_bounds(const smg_graph* g, int replica, uint32_t num_shards, int unit_bound, uint64_t* bounds) {
  if (!g || !bounds) return fail(SMG_EINPUT, "null argument");
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  if (num_shards == 0 || num_shards > 4096) return fail(SMG_EINPUT, "bad shard count");
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  SMG_CUDA(cudaSetDevice(r.device));
  int rc = ensure_shard_map(*g, r, num_shards, unit_bound ? 1 : 0);
  if (rc) return rc;
  std::memcpy(bounds, r.map_bounds.data(), r.map_bounds.size() * sizeof(uint64_t));
  return SMG_OK;
}

int smg_count_range(const smg_graph* g, const smg_plan* plan, int replica, uint32_t lo,
                    uint32_t hi, uint32_t flags, smg_result* out) {
  const double t0 = now_ms();
  if (!out) return fail(SMG_EINPUT, "null result");
  std::memset(out, 0, sizeof(*out));
  Program prog;
  int rc = prepare(g, plan, &prog);
  if (rc) return rc;
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  if (lo > hi || hi > g->n) return fail(SMG_EINPUT, "root range out of bounds");
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  uint64_t b = 0, e = 0;
  SMG_CUDA(cudaSetDevice(r.device));
  SMG_CUDA(cudaMemcpy(&b, r.off + lo, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  SMG_CUDA(cudaMemcpy(&e, r.off + hi, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  Launch L;
  L.meter = (flags & SMG_METER) != 0;
  L.unit_begin = b;
  L.unit_end = e;
  L.root_lo = lo;
  L.root_hi = hi;
  L.meter_roots = true;
  {
    const int fk = fast_for(*plan, flags, true);
    rc = fk ? enqueue_fast(*g, r, fk, *plan, L) : enqueue(*g, r, prog, L);
  }
  if (rc) return rc;
  bool ovf = false;
  rc = finish(r, &out->count, &out->elements, &out->units, &ovf, &out->kernel_ms);
  if (rc) return rc;
  out->per_gpu[0] = out->count;
  out->wall_ms = now_ms() - t0;
  if (ovf) return fail(SMG_EOVERFLOW, "embedding count exceeds 64 bits");
  return SMG_OK;
}

// Shares of `np` 4-vertex closed-form plans on the first num_gpus replicas
// (one host thread per device; replicas locked by the caller), summed.
static int m4_count_devices(const smg_graph* g, const int* kinds, const smg_plan* const* plans, uint32_t np,
                            unsigned num_gpus, smg_result* out) {
  std::vector<std::vector<M4Out>> res(num_gpus, std::vector<M4Out>(np));
  std::vector<int> rcs(num_gpus, SMG_OK);
  std::vector<std::string> errs(num_gpus);
  auto run = [&](unsigned d) {
    Launch L;
    L.unit_begin = 0;
    L.unit_end = g->slots;
    L.root_lo = 0;
    L.root_hi = static_cast<uint32_t>(g->n);
    L.shard = d;
    L.num_shards = num_gpus;
    rcs[d] = m4_count(*g, *g->reps[d], kinds, plans, np, L, res[d].data());
    if (rcs[d]) errs[d] = g_last_error;  // thread-local: carry it to the caller's thread
  };
  std::vector<std::thread> th;
  for (unsigned d = 1; d < num_gpus; ++d) th.emplace_back(run, d);
  run(0);
  for (auto& t : th) t.join();
  for (unsigned d = 0; d < num_gpus; ++d)
    if (rcs[d]) return rcs[d] == kTryGeneric ? kTryGeneric : fail(rcs[d], errs[d]);
  for (uint32_t i = 0; i < np; ++i) {
    __int128 total = 0;
    std::memset(&out[i], 0, sizeof(out[i]));
    for (unsigned d = 0; d < num_gpus; ++d) {
      total += res[d][i].share;
      out[i].per_gpu[d] = static_cast<uint64_t>(res[d][i].share);
      out[i].units += res[d][i].units;
      out[i].kernel_ms = std::max(out[i].kernel_ms, res[d][i].ms);
    }
    if (total < 0 || (total >> 64) != 0) return fail(SMG_EOVERFLOW, "embedding count exceeds 64 bits");
    out[i].count = static_cast<uint64_t>(total);
  }
  return SMG_OK;
}

int smg_count(const smg_graph* g, const smg_plan* plan, unsigned num_gpus, uint32_t flags,
              smg_result* out) {
  const double t0 = now_ms();
  if (!out) return fail(SMG_EINPUT, "null result");
  std::memset(out, 0, sizeof(*out));
  Program prog;
  int rc = prepare(g, plan, &prog);
  if (rc) return rc;
  if (num_gpus == 0) num_gpus = 1;  // workers == 0 -> 1 (engine.cpp:146)
  if (num_gpus > g->reps.size()) return fail(SMG_EINPUT, "more GPUs requested than graph replicas");
  std::vector<std::unique_lock<std::mutex>> locks;
  for (unsigned d = 0; d < num_gpus; ++d) locks.emplace_back(g->reps[d]->mu);
  const int fk = fast_for(*plan, flags);
  const int rm = relabel_mode(*plan, flags);
  if (rm == 2) {
    const int mk = m4_kind(*plan);
    rc = m4_count_devices(g, &mk, &plan, 1, num_gpus, out);
    if (rc != kTryGeneric) {
      out->wall_ms = now_ms() - t0;
      return rc;
    }
    std::memset(out, 0, sizeof(*out));
  }
  for (unsigned d = 0; d < num_gpus; ++d) {
    Launch L;
    L.meter = (flags & SMG_METER) != 0;
    L.unit_begin = 0;
    L.unit_end = g->slots;
    L.root_lo = 0;
    L.root_hi = static_cast<uint32_t>(g->n);
    L.meter_roots = (d == 0);
    L.shard = d;
    L.num_shards = num_gpus;
    Replica& rd = *g->reps[d];
    rc = rm >= 1 ? enqueue_oriented(*g, rd, prog, L)
         : fk    ? enqueue_fast(*g, rd, fk, *plan, L)
                 : enqueue(*g, rd, prog, L);
    if (rc) {
      // devices 0..d-1 are still counting into their Counters: drain them
      // before the replica locks are released
      const std::string err = g_last_error;
      for (unsigned e = 0; e < d; ++e) {
        uint64_t c = 0, el = 0, u = 0;
        bool ovf = false;
        double ms = 0;
        finish(*g->reps[e], &c, &el, &u, &ovf, &ms);
      }
      g_last_error = err;
      return rc;
    }
  }
  bool any_ovf = false;
  __int128 total = 0;  // device shares may be signed (folded full-count kinds)
  for (unsigned d = 0; d < num_gpus; ++d) {
    uint64_t c = 0, el = 0, u = 0;
    int64_t hi = 0;
    bool ovf = false;
    double ms = 0;
    rc = finish(*g->reps[d], &c, &el, &u, &ovf, &ms, &hi);
    if (rc) return rc;
    out->per_gpu[d] = c;
    total += static_cast<__int128>((static_cast<unsigned __int128>(static_cast<uint64_t>(hi)) << 64) | c);
    out->elements += el;
    out->units += u;
    out->kernel_ms = std::max(out->kernel_ms, ms);
    any_ovf |= ovf;
  }
  if (total < 0 || (total >> 64) != 0) any_ovf = true;
  out->count = static_cast<uint64_t>(total);
  out->wall_ms = now_ms() - t0;
  if (any_ovf) return fail(SMG_EOVERFLOW, "embedding count exceeds 64 bits");
  return SMG_OK;
}

// The batch kind of a plan inside smg_count_many: a 4-vertex closed-form kind,
// kFastClique4 for a fully restricted 4-clique plan (its count is the K4 the
// closed forms need anyway), or 0 (counted on its own).
static int batch_kind(const smg_plan& p, uint32_t flags) {
  if (clique5_plan(p)) return 0;  // counted on its own (smg_count)
  if (relabel_mode(p, flags) == 2) return m4_kind(p);
  if (!g_relabel || !g_fast || (flags & (SMG_METER | SMG_GENERIC))) return 0;
  return clique4_plan(p) ? kFastClique4 : 0;  // SMG_K4=0: still shares the batch's generic K4
}

// shard_mode: one shard on one replica (smg_count_many_shard), else the first
// num_gpus replicas (smg_count_many).
static int count_many_impl(const smg_graph* g, const smg_plan* plans, uint32_t num_plans, bool shard_mode,
                           int replica, uint32_t shard, uint32_t num_shards, unsigned num_gpus, uint32_t flags,
                           smg_result* out) {
  if (!g || !plans || !out) return fail(SMG_EINPUT, "null argument");
  std::vector<int> kinds;
  std::vector<const smg_plan*> shared;
  std::vector<uint32_t> idx;
  bool closed_form = false;
  for (uint32_t i = 0; i < num_plans; ++i) {
    Program prog;
    int rc = prepare(g, &plans[i], &prog);  // validates every plan before any work
    if (rc) return rc;
    const int k = batch_kind(plans[i], flags);
    if (k && shared.size() < 16) {
      kinds.push_back(k);
      shared.push_back(&plans[i]);
      idx.push_back(i);
      closed_form |= k != kFastClique4;
    }
  }
  if (shared.size() >= 2 && closed_form) {
    const double t0 = now_ms();
    std::vector<smg_result> res(shared.size());
    if (shard_mode) {
      Replica& r = *g->reps[replica];
      std::lock_guard<std::mutex> lock(r.mu);
      Launch L;
      L.unit_begin = 0;
      L.unit_end = g->slots;
      L.root_lo = 0;
      L.root_hi = static_cast<uint32_t>(g->n);
      L.shard = shard;
      L.num_shards = num_shards;
      std::vector<M4Out> o(shared.size());
      int rc = m4_count(*g, r, kinds.data(), shared.data(), static_cast<uint32_t>(shared.size()), L, o.data());
      if (rc) return rc;
      for (size_t k = 0; k < shared.size(); ++k) {
        std::memset(&res[k], 0, sizeof(res[k]));
        m4_store(o[k], &res[k]);
      }
    } else {
      std::vector<std::unique_lock<std::mutex>> locks;
      for (unsigned d = 0; d < num_gpus; ++d) locks.emplace_back(g->reps[d]->mu);
      int rc = m4_count_devices(g, kinds.data(), shared.data(), static_cast<uint32_t>(shared.size()), num_gpus,
                                res.data());
      if (rc) return rc;
    }
    const double wall = now_ms() - t0;
    for (size_t k = 0; k < shared.size(); ++k) {
      out[idx[k]] = res[k];
      out[idx[k]].wall_ms = wall / shared.size();
    }
  } else {
    idx.clear();
  }
  for (uint32_t i = 0; i < num_plans; ++i) {
    if (std::find(idx.begin(), idx.end(), i) != idx.end()) continue;
    int rc = shard_mode ? smg_count_shard(g, &plans[i], replica, shard, num_shards, flags, &out[i])
                        : smg_count(g, &plans[i], num_gpus, flags, &out[i]);
    if (rc) return rc;
  }
  return SMG_OK;
}

// count_instances for a batch of plans on one graph (the motif loop,
// engine.cpp:193-205): out[i] is what smg_count(g, &plans[i], ...) returns.
// The 4-vertex plans with a closed form over subgraph counts share one
// 4-clique count and one set of passes (m4_count); a fully restricted
// 4-clique plan in the batch takes its count from the same K4.
int smg_count_many(const smg_graph* g, const smg_plan* plans, uint32_t num_plans, unsigned num_gpus,
                   uint32_t flags, smg_result* out) {
  if (!g) return fail(SMG_EINPUT, "null graph");
  if (num_gpus == 0) num_gpus = 1;
  if (num_gpus > g->reps.size()) return fail(SMG_EINPUT, "more GPUs requested than graph replicas");
  return count_many_impl(g, plans, num_plans, false, 0, 0, 1, num_gpus, flags, out);
}

// The same for one shard on one replica (one process per GPU): out[i] is what
// smg_count_shard(g, &plans[i], replica, shard, num_shards, ...) returns.
int smg_count_many_shard(const smg_graph* g, const smg_plan* plans, uint32_t num_plans, int replica,
                         uint32_t shard, uint32_t num_shards, uint32_t flags, smg_result* out) {
  if (!g) return fail(SMG_EINPUT, "null graph");
  if (replica < 0 || replica >= static_cast<int>(g->reps.size())) return fail(SMG_EINPUT, "bad replica");
  if (num_shards == 0 || shard >= num_shards) return fail(SMG_EINPUT, "bad shard");
  return count_many_impl(g, plans, num_plans, true, replica, shard, num_shards, 1, flags, out);
}

}  // extern "C"

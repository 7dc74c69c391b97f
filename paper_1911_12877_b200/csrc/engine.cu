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

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/symmine_gpu.h"
#include "program.hpp"

namespace smg {

constexpr int kWarpsPerBlock = 8;
constexpr int kThreads = kWarpsPerBlock * 32;
constexpr uint32_t kChunk = 32;  // edge slots per queue grab
constexpr unsigned kFull = 0xffffffffu;
constexpr int kHashLog2 = 11;  // per-warp shared-memory hash: 2048 slots (8 KB)
constexpr uint32_t kHashSlots = 1u << kHashLog2;
constexpr uint32_t kEmptySlot = 0xffffffffu;  // never a vertex id (ids < n < 2^32)
constexpr size_t kDynSmem = sizeof(uint32_t) * kHashSlots * kWarpsPerBlock;
// CTA tier (heavy_kernel): 16 warps share one 32K-slot (128 KB) table.
constexpr int kHeavyWarps = 16;
constexpr int kHeavyThreads = kHeavyWarps * 32;
constexpr uint32_t kHeavySlots = 1u << 15;
constexpr uint32_t kHeavyChunk = kHeavySlots / 2;  // probe-set elements per table fill
constexpr size_t kHeavySmem = sizeof(uint32_t) * kHeavySlots;
constexpr uint64_t kHeavyMinStream = 4096;  // defer only batches with real streaming work
constexpr uint64_t kHeavyQueueCap = 1ull << 22;

// ---------------------------------------------------------------- device ---

struct Counters {
  unsigned long long next_chunk;
  unsigned long long count;
  unsigned long long elements;
  unsigned long long units;
  unsigned long long heavy_count;  // batches deferred to the CTA tier
  unsigned long long heavy_next;   // CTA-tier queue cursor
  unsigned int overflow;
  unsigned int pad;
  // SMG_TRACE=1: per-phase cycle and event counters (see kTr* below)
  unsigned long long trace[16];  // >= kTrCount
};

enum {
  kTrUnits = 0, kTrBuildCycles, kTrBatchCycles, kTrBatches, kTrBatchesHashed, kTrStreamElems,
  kTrSearchLists, kTrProbeSetSum, kTrStreamSetSum, kTrLeafCycles, kTrLeaves, kTrBigPCycles,
  kTrDeferred, kTrHeavyItems, kTrHeavyCycles, kTrCount
};

struct KernelArgs {
  const unsigned long long* off;  // n+1
  const uint32_t* adj;            // slots
  const uint32_t* src;            // slots: source vertex of each slot
  uint32_t* scratch;
  uint64_t cap;                   // scratch elements per slot
  uint64_t unit_begin, unit_end;  // edge-slot range
  uint32_t shard, num_shards;
  Counters* ctr;
  uint32_t* heavy_items;          // CTA-tier queue (kHeavyItemWords per item), may be null
  unsigned long long heavy_cap;
  uint32_t* heavy_scratch;        // CTA-tier node scratch (nslots * cap per CTA)
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

struct Ctx {
  const unsigned long long* __restrict__ off;
  const uint32_t* __restrict__ adj;
  WarpState* s;
  uint32_t* scratch;
  uint64_t cap;
  uint32_t* hash;
  int lane;
};

__device__ __forceinline__ void nbrs(const Ctx& c, uint32_t v, const uint32_t*& p, uint32_t& len) {
  const unsigned long long b = __ldg(c.off + v);
  const unsigned long long e = __ldg(c.off + v + 1);
  p = c.adj + b;
  len = static_cast<uint32_t>(e - b);
}

// Apply a node's ops to the input set `in` (sorted, already bounded).
// COUNT: return |result| only; else write the sorted result to `out`.
template <bool COUNT>
__device__ uint32_t apply_ops(const Ctx& c, const Node& nd, const uint32_t* in, uint32_t inlen,
                              bool in_is_scratch, uint32_t* out) {
  const WarpState& s = *c.s;
  const unsigned lt_mask = (1u << c.lane) - 1u;
  // Single intersection: iterate the shorter side, probe the longer.
  if (nd.nops == 1 && nd.ops[0].mode == kOpIsect) {
    const uint32_t* b;
    uint32_t blen;
    nbrs(c, s.vals[nd.ops[0].level], b, blen);
    if (nd.bound >= 0) blen = lower_bound_dev(b, blen, s.vals[nd.bound]);
    if (blen < inlen) {
      uint32_t written = 0;
      for (uint32_t base = 0; base < blen; base += 32) {
        const uint32_t i = base + c.lane;
        bool keep = i < blen;
        const uint32_t x = keep ? __ldg(b + i) : 0u;
        if (keep) keep = in_is_scratch ? contains_rw(in, inlen, x) : contains_dev(in, inlen, x);
        const unsigned m = __ballot_sync(kFull, keep);
        if (!COUNT && keep) out[written + __popc(m & lt_mask)] = x;
        written += __popc(m);
      }
      return written;
    }
  }
  // Generic: iterate the input, probe every op list.
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
    const uint32_t x = keep ? (in_is_scratch ? in[i] : __ldg(in + i)) : 0u;
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
                                           uint32_t& inlen, bool& in_scratch) {
  const WarpState& s = *c.s;
  if (nd.src >= 0) {
    in = s.ptr[nd.src];
    inlen = s.len[nd.src];
    in_scratch = true;  // may also be a raw CSR slice; plain loads are fine for both
  } else {
    nbrs(c, s.vals[nd.list], in, inlen);
    in_scratch = false;
  }
  if (nd.bound >= 0) {
    const uint32_t b = s.vals[nd.bound];
    inlen = in_scratch ? lower_bound_rw(in, inlen, b) : lower_bound_dev(in, inlen, b);
  }
}

__device__ void build_node(const Ctx& c, const Program& P, int t) {
  const Node& nd = P.nodes[t];
  const uint32_t* in;
  uint32_t inlen;
  bool in_scratch;
  node_input(c, nd, in, inlen, in_scratch);
  if (nd.raw) {
    if (c.lane == 0) {
      c.s->ptr[t] = in;
      c.s->len[t] = inlen;
    }
    __syncwarp();
    return;
  }
  uint32_t* out = c.scratch + static_cast<uint64_t>(nd.slot) * c.cap;
  const uint32_t len = apply_ops<false>(c, nd, in, inlen, in_scratch, out);
  __syncwarp();
  if (c.lane == 0) {
    c.s->ptr[t] = out;
    c.s->len[t] = len;
  }
  __syncwarp();
}

__device__ __forceinline__ uint32_t leaf_count(const Ctx& c, const Program& P) {
  const uint32_t* in;
  uint32_t inlen;
  bool in_scratch;
  node_input(c, P.leaf, in, inlen, in_scratch);
  if (P.leaf.raw) return inlen;
  return apply_ops<true>(c, P.leaf, in, inlen, in_scratch, nullptr);
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
// 128 KB table and streams the lists with all its warps.

struct ProbeSet {
  const uint32_t* arr;  // sorted (scratch or CSR slice)
  uint32_t n;
  uint32_t lo, hi;      // arr[0], arr[n-1]
  uint32_t* hash;       // shared-memory table, valid when bits > 0
  int bits;
};

__device__ __forceinline__ uint32_t hslot(uint32_t x, int bits) {
  return (x * 0x9E3779B1u) >> (32 - bits);
}

__device__ __forceinline__ bool probe(const ProbeSet& P, uint32_t y) {
  if (P.bits) {
    const uint32_t mask = (1u << P.bits) - 1u;
    uint32_t h = hslot(y, P.bits);
    for (;;) {
      const uint32_t k = P.hash[h];
      if (k == y) return true;
      if (k == kEmptySlot) return false;
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

// Fill `table` with P (threads [tid, tid+nthreads) cooperate; caller syncs
// before and after).  Requires P.n > 0 and 2 * P.n <= table capacity.
__device__ __forceinline__ void fill_table(uint32_t* table, const ProbeSet& P, int tid,
                                           int nthreads) {
  const uint32_t slots = 1u << P.bits;
  for (uint32_t i = tid; i < slots; i += nthreads) table[i] = kEmptySlot;
}

__device__ __forceinline__ void insert_table(uint32_t* table, const ProbeSet& P, int tid,
                                             int nthreads) {
  const uint32_t mask = (1u << P.bits) - 1u;
  for (uint32_t i = tid; i < P.n; i += nthreads) {
    const uint32_t key = P.arr[i];
    uint32_t h = hslot(key, P.bits);
    while (atomicCAS(&table[h], kEmptySlot, key) != kEmptySlot) h = (h + 1) & mask;
  }
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

constexpr int kStreamUnroll = 4;  // independent loads in flight per lane

// sum_{s in S} |{p in P : p in N(s)}| with rel: 0 none, 1 p < s, 2 p > s, over
// the groups of 32 elements of S starting at g_first with stride g_stride.
// Returns this warp's partial (all lanes hold it).
template <bool TRACE>
__device__ uint64_t stream_count(const Ctx& c, const uint32_t* S, uint32_t nS, const ProbeSet& P,
                                 int rel, uint32_t g_first, uint32_t g_stride, uint64_t* tr) {
  uint64_t total = 0;
  for (uint32_t g0 = g_first; g0 < nS; g0 += g_stride) {
    const uint32_t i = g0 + c.lane;
    uint32_t start = 0, len = 0, lo_val = P.lo, hi_val = P.hi + 1u;
    const uint32_t* base = c.adj;
    bool search = false;
    if (i < nS) {
      const uint32_t s = S[i];
      if (rel == 1) hi_val = min(hi_val, s);
      if (rel == 2) lo_val = max(lo_val, s + 1u);
      const unsigned long long b = __ldg(c.off + s), e = __ldg(c.off + s + 1);
      base = c.adj + b;
      const uint32_t deg = static_cast<uint32_t>(e - b);
      if (lo_val < hi_val && deg) {
        if (deg > 32) {
          start = lower_bound_dev(base, deg, lo_val);
          len = lower_bound_dev(base + start, deg - start, hi_val);
        } else {
          len = deg;  // short list: range-filter per element instead
        }
      }
      search = len > 64 && static_cast<uint64_t>(P.n) * (33u - __clz(len)) * 2u < len;
    }
    const uint32_t slen = search ? 0u : len;
    const uint32_t incl = warp_incl_scan(slen, c.lane);
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - slen;
    if (TRACE) {
      tr[kTrStreamElems] += tot;
      tr[kTrSearchLists] += __popc(__ballot_sync(kFull, search));
    }
    uint32_t hits = 0;
    for (uint32_t t = 0; t < tot; t += 32 * kStreamUnroll) {
      uint32_t y[kStreamUnroll];
      bool ok[kStreamUnroll];
#pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u) {
        const uint32_t idx = t + u * 32 + c.lane;
        int j = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const uint32_t ex = __shfl_sync(kFull, excl, j + step);
          if (ex <= idx) j += step;
        }
        const uint32_t o_start = __shfl_sync(kFull, start, j);
        const uint32_t o_excl = __shfl_sync(kFull, excl, j);
        const uint32_t o_lo = __shfl_sync(kFull, lo_val, j);
        const uint32_t o_hi = __shfl_sync(kFull, hi_val, j);
        const uint32_t* o_base = reinterpret_cast<const uint32_t*>(
            __shfl_sync(kFull, reinterpret_cast<unsigned long long>(base), j));
        ok[u] = idx < tot;
        y[u] = ok[u] ? __ldg(o_base + o_start + (idx - o_excl)) : 0u;
        ok[u] = ok[u] && y[u] >= o_lo && y[u] < o_hi;
      }
#pragma unroll
      for (int u = 0; u < kStreamUnroll; ++u)
        if (ok[u] && probe(P, y[u])) ++hits;
    }
    unsigned sm = __ballot_sync(kFull, search);
    while (sm) {
      const int j = __ffs(sm) - 1;
      sm &= sm - 1;
      const uint32_t* jb = reinterpret_cast<const uint32_t*>(
          __shfl_sync(kFull, reinterpret_cast<unsigned long long>(base), j));
      const uint32_t js = __shfl_sync(kFull, start, j);
      const uint32_t jl = __shfl_sync(kFull, len, j);
      const uint32_t jlo = __shfl_sync(kFull, lo_val, j);
      const uint32_t jhi = __shfl_sync(kFull, hi_val, j);
      const uint32_t pa = lower_bound_rw(P.arr, P.n, jlo);
      const uint32_t pb = lower_bound_rw(P.arr, P.n, jhi);
      for (uint32_t q = pa + c.lane; q < pb; q += 32)
        if (contains_dev(jb + js, jl, P.arr[q])) ++hits;
    }
    total += hits;
  }
  return warp_sum64(total);
}

// Sum of deg over X[g_first + lane], stride (partial; all lanes hold it).
__device__ __forceinline__ uint64_t degree_sum(const Ctx& c, const uint32_t* X, uint32_t n,
                                               uint32_t first, uint32_t stride) {
  uint64_t acc = 0;
  for (uint32_t i = first + c.lane; i < n; i += stride) {
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
  if (P.batch_fixed_bound >= 0) b.nB = lower_bound_rw(b.B, b.nB, s.vals[P.batch_fixed_bound]);
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

struct HeavyQueue {
  uint32_t* items;          // kHeavyItemWords per item
  unsigned long long cap;
  unsigned long long* count;
};
constexpr int kHeavyItemWords = 6;  // v_0 .. v_{n-3}, n <= 8

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
      const uint64_t da = degree_sum(c, b.A, b.nA, 0, 32), db = degree_sum(c, b.B, b.nB, 0, 32);
      flip = db < da;
      sum_s = flip ? db : da;
    }
    ProbeSet ps;
    ps.arr = flip ? b.A : b.B;
    ps.n = flip ? b.nA : b.nB;
    ps.lo = ps.arr[0];
    ps.hi = ps.arr[ps.n - 1];
    ps.hash = c.hash;
    ps.bits = 0;
    if (ps.n * 2 > kHashSlots) {
      // Too big for the warp's table.  Queue it for the CTA tier unless the
      // streaming side is trivially small (then binary search is cheaper).
      if (b.same) sum_s = degree_sum(c, b.A, b.nA, 0, 32);
      if (sum_s > kHeavyMinStream && hq.items) {
        unsigned long long slot = 0;
        if (c.lane == 0) slot = atomicAdd(hq.count, 1ull);
        slot = __shfl_sync(kFull, slot, 0);
        if (slot < hq.cap) {
          if (c.lane < P.depth - 2) hq.items[slot * kHeavyItemWords + c.lane] = s.vals[c.lane];
          if (TRACE) tr[kTrDeferred] += 1;
          return 0;
        }
      }
    } else {
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
    core = flip ? stream_count<TRACE>(c, b.B, b.nB, ps, yltx ? 2 : 0, 0, 32, tr)
                : stream_count<TRACE>(c, b.A, b.nA, ps, yltx ? 1 : 0, 0, 32, tr);
    if (TRACE && !ps.bits) tr[kTrBigPCycles] += clock64() - t0;
  }
  if (!P.batch_diff) return core;
  return diff_terms(c, P, b, 0, 32, true) - core;
}

template <bool METER, bool TRACE>
__global__ void __launch_bounds__(kThreads) count_kernel(const KernelArgs a) {
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
  c.hash = dyn_smem + wib * kHashSlots;
  const bool batch = !METER && P.batch;
  HeavyQueue hq;
  hq.items = a.heavy_items;
  hq.cap = a.heavy_cap;
  hq.count = &a.ctr->heavy_count;
  uint64_t trbuf[TRACE ? kTrCount : 1];
  if (TRACE)
    for (int i = 0; i < kTrCount; ++i) trbuf[i] = 0;
  uint64_t* tr = trbuf;
  long long tclk = 0;
  WarpState& s = states[wib];

  uint64_t cnt = 0, elems = 0, units = 0;
  bool ovf = false;
  uint32_t pos[kMaxLevels];

  for (;;) {
    unsigned long long chunk = 0;
    if (lane == 0) chunk = atomicAdd(&a.ctr->next_chunk, 1ull);
    chunk = __shfl_sync(kFull, chunk, 0);
    const uint64_t gchunk = chunk * a.num_shards + a.shard;
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
      if (TRACE) tclk = clock64();
      for (int t = P.node_begin[0]; t < P.node_end[0]; ++t) build_node(c, P, t);
      for (int t = P.node_begin[1]; t < P.node_end[1]; ++t) build_node(c, P, t);
      if (TRACE) tr[kTrBuildCycles] += clock64() - tclk;
      if (P.depth == 3) {
        checked_acc(cnt, leaf_count(c, P), ovf);
        continue;
      }
      if (batch && P.depth == 4) {
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
          if (TRACE) tclk = clock64();
          checked_acc(cnt, leaf_batch<TRACE>(c, P, hq, tr), ovf);
          if (TRACE) tr[kTrBatchCycles] += clock64() - tclk;
        } else {
          ++level;
          pos[level] = 0;
        }
      }
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
      for (int i = 0; i < kTrCount; ++i)
        if (tr[i]) atomicAdd(&a.ctr->trace[i], static_cast<unsigned long long>(tr[i]));
    }
  }
}

// CTA tier: the deferred batches, one per CTA at a time, with a 128 KB table
// shared by kHeavyWarps warps.  Probe sets beyond the table are split into
// value-range chunks (the streamed lists are range-restricted per chunk, so
// every element is still probed exactly once).
template <bool TRACE>
__global__ void __launch_bounds__(kHeavyThreads) heavy_kernel(const KernelArgs a) {
  __shared__ WarpState st;
  __shared__ unsigned long long item_sh;
  __shared__ unsigned long long red_a[kHeavyWarps], red_b[kHeavyWarps];
  extern __shared__ uint32_t table[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const Program& P = a.prog;
  Ctx c;
  c.off = a.off;
  c.adj = a.adj;
  c.s = &st;
  c.scratch = a.heavy_scratch + static_cast<uint64_t>(blockIdx.x) * P.nslots * a.cap;
  c.cap = a.cap;
  c.lane = lane;
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
    if (threadIdx.x == 0) item_sh = atomicAdd(&a.ctr->heavy_next, 1ull);
    __syncthreads();
    const unsigned long long it = item_sh;
    if (it >= nitems) break;
    long long t0 = TRACE ? clock64() : 0;
    if (warp == 0) {
      if (lane < P.depth - 2) st.vals[lane] = a.heavy_items[it * kHeavyItemWords + lane];
      __syncwarp();
      for (int t = P.node_begin[0]; t < P.node_end[P.depth - 3]; ++t) build_node(c, P, t);
    }
    __syncthreads();
    const BatchSets b = batch_sets(st, P);
    // side choice from the degree sums (CTA-wide)
    bool flip = false;
    if (!b.same) {
      const uint64_t da = degree_sum(c, b.A, b.nA, warp * 32, kHeavyThreads);
      const uint64_t db = degree_sum(c, b.B, b.nB, warp * 32, kHeavyThreads);
      if (lane == 0) {
        red_a[warp] = da;
        red_b[warp] = db;
      }
      __syncthreads();
      uint64_t sa = 0, sb = 0;
      for (int w = 0; w < kHeavyWarps; ++w) {
        sa += red_a[w];
        sb += red_b[w];
      }
      flip = sb < sa;
      __syncthreads();
    }
    const uint32_t* Parr = flip ? b.A : b.B;
    const uint32_t Pn = flip ? b.nA : b.nB;
    const uint32_t* S = flip ? b.B : b.A;
    const uint32_t nS = flip ? b.nB : b.nA;
    const int rel = yltx ? (flip ? 2 : 1) : 0;
    uint64_t core = 0;
    for (uint32_t pc = 0; pc < Pn; pc += kHeavyChunk) {
      ProbeSet ps;
      ps.arr = Parr + pc;
      ps.n = min(kHeavyChunk, Pn - pc);
      ps.lo = ps.arr[0];
      ps.hi = ps.arr[ps.n - 1];
      ps.hash = table;
      ps.bits = table_bits(ps.n);
      fill_table(table, ps, threadIdx.x, kHeavyThreads);
      __syncthreads();
      insert_table(table, ps, threadIdx.x, kHeavyThreads);
      __syncthreads();
      core += stream_count<TRACE>(c, S, nS, ps, rel, warp * 32, kHeavyWarps * 32, tr);
      __syncthreads();
    }
    const uint64_t dpart = P.batch_diff ? diff_terms(c, P, b, warp * 32, kHeavyThreads, warp == 0) : 0;
    if (lane == 0) {
      red_a[warp] = core;
      red_b[warp] = dpart;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t sc = 0, sd = 0;
      for (int w = 0; w < kHeavyWarps; ++w) {
        sc += red_a[w];
        sd += red_b[w];
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
  }
  if (TRACE && lane == 0) {
    for (int i = 0; i < kTrCount; ++i)
      if (tr[i] && (i != kTrHeavyItems && i != kTrHeavyCycles || threadIdx.x == 0))
        atomicAdd(&a.ctr->trace[i], static_cast<unsigned long long>(tr[i]));
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

// ------------------------------------------------------------------ host ---

thread_local std::string g_last_error;
const int g_trace = [] {
  const char* e = std::getenv("SMG_TRACE");
  return (e && *e && *e != '0') ? 1 : 0;
}();

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
  size_t heavy_scratch_bytes = 0;
  Counters* ctr = nullptr;  // device
  Counters* host_ctr = nullptr;  // pinned
  cudaStream_t stream = nullptr;       // owned
  cudaStream_t user_stream = nullptr;  // set by smg_graph_set_stream (not owned)
  cudaStream_t active() const { return user_stream ? user_stream : stream; }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
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

// Enqueue one shard on replica r (asynchronous).  Caller holds r.mu.
template <bool METER, bool TRACE>
int enqueue_t(const smg_graph& g, Replica& r, const Program& prog, const Launch& L) {
  const uint64_t cap = std::max<uint64_t>(32, (g.max_degree + 31) / 32 * 32);
  const bool heavy = !METER && prog.batch;
  SMG_CUDA(cudaFuncSetAttribute(count_kernel<METER, TRACE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDynSmem)));
  int per_sm = 0;
  SMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_kernel<METER, TRACE>, kThreads,
                                                         kDynSmem));
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
    const size_t hs = static_cast<size_t>(r.num_sms) * prog.nslots * cap * 4;
    if (r.heavy_scratch_bytes < hs) {
      if (r.heavy_scratch) cudaFree(r.heavy_scratch);
      r.heavy_scratch = nullptr;
      r.heavy_scratch_bytes = 0;
      SMG_CUDA(cudaMalloc(&r.heavy_scratch, std::max<size_t>(hs, 4)));
      r.heavy_scratch_bytes = hs;
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
  a.shard = L.shard;
  a.num_shards = L.num_shards;
  a.ctr = r.ctr;
  a.heavy_items = heavy ? r.heavy_items : nullptr;
  a.heavy_cap = heavy ? kHeavyQueueCap : 0;
  a.heavy_scratch = r.heavy_scratch;
  a.prog = prog;
  if (L.unit_end > L.unit_begin) {
    count_kernel<METER, TRACE><<<static_cast<unsigned>(blocks), kThreads, kDynSmem, st>>>(a);
    if (heavy) {
      SMG_CUDA(cudaFuncSetAttribute(heavy_kernel<TRACE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kHeavySmem)));
      heavy_kernel<TRACE><<<r.num_sms, kHeavyThreads, kHeavySmem, st>>>(a);
    }
  }
  SMG_CUDA(cudaGetLastError());
  SMG_CUDA(cudaEventRecord(r.ev1, st));
  SMG_CUDA(cudaMemcpyAsync(r.host_ctr, r.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  return SMG_OK;
}

int enqueue(const smg_graph& g, Replica& r, const Program& prog, const Launch& L) {
  SMG_CUDA(cudaSetDevice(r.device));
  if (L.meter) return g_trace ? enqueue_t<true, true>(g, r, prog, L) : enqueue_t<true, false>(g, r, prog, L);
  return g_trace ? enqueue_t<false, true>(g, r, prog, L) : enqueue_t<false, false>(g, r, prog, L);
}

int finish(Replica& r, uint64_t* count, uint64_t* elems, uint64_t* units, bool* ovf, double* ms) {
  SMG_CUDA(cudaSetDevice(r.device));
  SMG_CUDA(cudaStreamSynchronize(r.active()));
  float t = 0.f;
  SMG_CUDA(cudaEventElapsedTime(&t, r.ev0, r.ev1));
  *count = r.host_ctr->count;
  *elems = r.host_ctr->elements;
  *units = r.host_ctr->units;
  *ovf = r.host_ctr->overflow != 0;
  *ms = t;
  if (g_trace) {
    static const char* names[kTrCount] = {"units", "build_cycles", "batch_cycles", "batches",
                                          "batches_hashed", "stream_elems", "search_lists",
                                          "probe_set_sum", "stream_set_sum", "leaf_cycles",
                                          "leaves", "bigP_stream_cycles", "deferred",
                                          "heavy_items", "heavy_cycles"};
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

int smg_abi_version(void) { return 1; }

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
       ",\"batch_fixed_bound\":" + std::to_string(pr.batch_fixed_bound) + "}";
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
    if (r->scratch) cudaFree(r->scratch);
    if (r->heavy_items) cudaFree(r->heavy_items);
    if (r->heavy_scratch) cudaFree(r->heavy_scratch);
    if (r->ctr) cudaFree(r->ctr);
    if (r->host_ctr) cudaFreeHost(r->host_ctr);
    if (r->ev0) cudaEventDestroy(r->ev0);
    if (r->ev1) cudaEventDestroy(r->ev1);
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
  uint64_t maxd = 0;
  for (uint64_t v = 0; v < n; ++v) {
    if (offsets[v + 1] < offsets[v]) return fail(SMG_EINPUT, "offsets must be non-decreasing");
    const uint64_t d = offsets[v + 1] - offsets[v];
    if (d > maxd) maxd = d;
    for (uint64_t i = offsets[v]; i < offsets[v + 1]; ++i) {
      const uint32_t x = adjacency[i];
      if (x >= n) return fail(SMG_EINPUT, "adjacency id out of range");
      if (x == v) return fail(SMG_EINPUT, "self loop in adjacency");
      if (i > offsets[v] && adjacency[i - 1] >= x)
        return fail(SMG_EINPUT, "neighbour lists must be strictly ascending");
    }
  }
  if (maxd >= (1ull << 32)) return fail(SMG_EINPUT, "degree too large");
  int ndev = smg_device_count();
  if (ndev == 0) return fail(SMG_EIO, "no CUDA device available (the engine has no CPU path)");
  smg_graph* g = new smg_graph;
  g->n = n;
  g->slots = slots;
  g->max_degree = maxd;
  for (int i = 0; i < num_devices; ++i) {
    const int dev = devices ? devices[i] : i;
    if (dev < 0 || dev >= ndev) {
      smg_graph_destroy(g);
      return fail(SMG_EINPUT, "device index out of range");
    }
    Replica* r = new Replica;
    g->reps.push_back(r);
    r->device = dev;
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
    if (ok && n > 0) {
      fill_src_kernel<<<r->num_sms * 8, 256, 0, r->stream>>>(r->off, n, r->src);
      ok = step(cudaGetLastError(), "fill_src");
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

int smg_graph_set_stream(smg_graph* g, int replica, void* stream) {
  if (!g || replica < 0 || replica >= static_cast<int>(g->reps.size()))
    return fail(SMG_EINPUT, "bad graph or replica");
  Replica& r = *g->reps[replica];
  std::lock_guard<std::mutex> lock(r.mu);
  r.user_stream = static_cast<cudaStream_t>(stream);
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
  rc = enqueue(*g, r, prog, L);
  if (rc) return rc;
  bool ovf = false;
  rc = finish(r, &out->count, &out->elements, &out->units, &ovf, &out->kernel_ms);
  if (rc) return rc;
  out->per_gpu[0] = out->count;
  out->wall_ms = now_ms() - t0;
  if (ovf) return fail(SMG_EOVERFLOW, "embedding count exceeds 64 bits");
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
  rc = enqueue(*g, r, prog, L);
  if (rc) return rc;
  bool ovf = false;
  rc = finish(r, &out->count, &out->elements, &out->units, &ovf, &out->kernel_ms);
  if (rc) return rc;
  out->per_gpu[0] = out->count;
  out->wall_ms = now_ms() - t0;
  if (ovf) return fail(SMG_EOVERFLOW, "embedding count exceeds 64 bits");
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
    rc = enqueue(*g, *g->reps[d], prog, L);
    if (rc) return rc;
  }
  bool any_ovf = false;
  for (unsigned d = 0; d < num_gpus; ++d) {
    uint64_t c = 0, el = 0, u = 0;
    bool ovf = false;
    double ms = 0;
    rc = finish(*g->reps[d], &c, &el, &u, &ovf, &ms);
    if (rc) return rc;
    out->per_gpu[d] = c;
    const uint64_t s = out->count + c;
    if (s < out->count) any_ovf = true;
    out->count = s;
    out->elements += el;
    out->units += u;
    out->kernel_ms = std::max(out->kernel_ms, ms);
    any_ovf |= ovf;
  }
  out->wall_ms = now_ms() - t0;
  if (any_ovf) return fail(SMG_EOVERFLOW, "embedding count exceeds 64 bits");
  return SMG_OK;
}

}  // extern "C"

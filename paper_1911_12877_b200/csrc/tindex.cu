// tindex.cu -- triangle index + closed-form ("folded") unit counts for the
// star-shaped plans, on B200 (sm_100a).
//
// The reference counts every plan by nested merges (Executor::count_from,
// proj/src/engine.cpp:89-115).  For plans whose levels >= 2 all lie in N(v1)
// (every level intersects v1's list), a unit (v0, v1) is a count inside the ego
// network L = G[N(v1)], where v0 is itself a vertex of L.  Its rows are the
// common-neighbour lists T(v1, x) = N(v1) & N(x) -- the triangle index built
// here -- and the plan's difference-heavy leaves fold into closed forms over
// local degrees, local codegrees and prefix sums, so the deepest two loops are
// never enumerated.  Every result is the exact per-unit count of the plan (the
// same value count_from(2) returns for that unit); tests compare unit by unit
// with the reference (tests/test_fast.py) and with the generic executor.
//
//  * star4 (motif plan L1 ([0],[],-) L2 ([1],[0],0) L3 ([1],[0,2],2)):
//      X = (N1 & [0,v0)) - N(v0);  count = C(|X|,2) - e(X),
//      e(X) = e(W) - sum_{t in T'} |T(v1,t) & [0,v0)| + e(T'),
//      W = N1 & [0,v0), T' = T(v1,v0) & [0,v0), e(W) a prefix sum over N1 of
//      |T(v1,x) & [0,x)| (lowpref).
//  * tailed diamond (a) (L1 ([0],[],-) L2 ([0,1],[],-) L3 ([1,2],[0],0)
//    L4 ([1],[0,2,3],-)): with P = N_L(v0), A(v2) = N_L(v2) & [0,v0) - P,
//    alpha(x) = |N_L(x) & P| (x < v0, x not in N_L[v0]):
//      count = (d1 - |P|) sum alpha - sum_{v2 in P} |A(v2)| (d_L v2 - |N_L v2 & P|)
//              - sum d_L(x) alpha(x) + sum alpha(x)^2 + S5 - S6,
//      S5 = sum_{v2 in P, x in A(v2)} |N_L(x) & N_L(v2)|  (k4 per index entry),
//      S6 = sum_{v2 in P, x in A(v2)} |N_L(x) & N_L(v2) & P|.
//    (inclusion-exclusion of the leaf L - N_L[v0] - N_L[v2] - N_L[v3]).
//  * tailed triangle (motif plan): count = sum_{v2 in P, v2 < v0}
//      (d1 - |P| - |T(v1,v2)| + |T(v1,v2) & P|),  P = T(v1, v0).
//  * diamond (motif plan, ego network of v0): count = sum_{v2 in P, v2 < v0}
//      |T(v0,v2) & [0,v1) - P|,  P = T(v0, v1).
//  * path4 (motif plan): count = |A1| |A0| - e(A1, A0), the e() of the house
//    decomposition below.
//  * rectangle, named plan (center c = v1 < u = v0) and motif plan (center
//    c = v0 > u = v1): with the incremental table cnt(x) = |N(x) & N(c) & [0,u)|
//    (the centre's neighbours y < u scattered, in ascending order),
//      count = sum_{x in N(u) & [0,c) - T(u,c)} cnt(x)
//              - sum_{t in T(u,c) & [0,u)} |T(u,t) & [0,c) - T(u,c)|.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include "tindex.hpp"

namespace smg {

namespace {

typedef unsigned long long ull;
constexpr unsigned kAll = 0xffffffffu;
constexpr uint32_t kSlotChunk = 32;

__device__ __forceinline__ uint32_t lb32(const uint32_t* __restrict__ a, uint32_t n, uint32_t x) {
  if (n == 0) return 0;
  const uint32_t* base = a;
  while (n > 1) {
    const uint32_t half = n >> 1;
    base = (base[half] < x) ? base + half : base;
    n -= half;
  }
  return static_cast<uint32_t>(base - a) + (*base < x ? 1u : 0u);
}

// |A[0,na) & B[0,nb)| for ascending lists: the shorter list is binary-searched
// into the longer one (the search window only moves right).
__device__ __forceinline__ uint32_t isect_count(const uint32_t* A, uint32_t na, const uint32_t* B, uint32_t nb) {
  if (na > nb) {
    const uint32_t* t = A;
    A = B;
    B = t;
    const uint32_t s = na;
    na = nb;
    nb = s;
  }
  uint32_t c = 0, lo = 0;
  for (uint32_t i = 0; i < na && lo < nb; ++i) {
    const uint32_t x = A[i];
    lo += lb32(B + lo, nb - lo, x);
    if (lo < nb && B[lo] == x) ++c;
  }
  return c;
}

__device__ __forceinline__ ull warp_sum(ull v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(kAll, v, d);
  return v;
}

// ------------------------------------------------------------ the index ---

__global__ void rev_kernel(const ull* __restrict__ off, const uint32_t* __restrict__ adj,
                           const uint32_t* __restrict__ src, uint64_t slots, ull* __restrict__ rev) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < slots;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t u = src[e], v = adj[e];
    const ull b = off[v];
    rev[e] = b + lb32(adj + b, static_cast<uint32_t>(off[v + 1] - b), u);
  }
}

// Common neighbours of every undirected edge {u < v} (slot e = (u, v)): count
// (WRITE = false) into tri[e], or write the positions into T(e) (in N(u)) and
// T(rev e) (in N(v)), both ascending.  Lists of <= 8 elements on the smaller
// side are handled by one lane; the rest by the whole warp (each lane
// binary-searches one element of the smaller list into the larger).
template <bool WRITE>
__global__ void __launch_bounds__(256) tri_kernel(const ull* __restrict__ off, const uint32_t* __restrict__ adj,
                                                  const uint32_t* __restrict__ src, uint64_t slots,
                                                  uint32_t* __restrict__ tri, const ull* __restrict__ toff,
                                                  uint32_t* __restrict__ tent, const ull* __restrict__ rev,
                                                  ull* next) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    ull chunk = 0;
    if (lane == 0) chunk = atomicAdd(next, 1ull);
    chunk = __shfl_sync(kAll, chunk, 0);
    const uint64_t e = chunk * kSlotChunk + lane;
    if (chunk * kSlotChunk >= slots) break;
    bool mine = e < slots;
    uint32_t u = 0, v = 0;
    if (mine) {
      u = src[e];
      v = adj[e];
      mine = u < v;
    }
    ull bu = 0, bv = 0;
    uint32_t du = 0, dv = 0;
    if (mine) {
      bu = off[u];
      du = static_cast<uint32_t>(off[u + 1] - bu);
      bv = off[v];
      dv = static_cast<uint32_t>(off[v + 1] - bv);
    }
    const bool small = mine && min(du, dv) <= 8;
    if (small) {
      const bool su = du <= dv;  // iterate N(u)
      const uint32_t* S = adj + (su ? bu : bv);
      const uint32_t* L = adj + (su ? bv : bu);
      const uint32_t ns = su ? du : dv, nl = su ? dv : du;
      uint32_t k = 0, lo = 0;
      ull w0 = 0, w1 = 0;
      if (WRITE) {
        w0 = toff[e];
        w1 = toff[rev[e]];
      }
      for (uint32_t i = 0; i < ns && lo < nl; ++i) {
        const uint32_t x = S[i];
        lo += lb32(L + lo, nl - lo, x);
        if (lo < nl && L[lo] == x) {
          if (WRITE) {
            tent[w0 + k] = su ? i : lo;
            tent[w1 + k] = su ? lo : i;
          }
          ++k;
        }
      }
      if (!WRITE) tri[e] = k;
    }
    unsigned big = __ballot_sync(kAll, mine && !small);
    while (big) {
      const int j = __ffs(big) - 1;
      big &= big - 1;
      const ull je = __shfl_sync(kAll, static_cast<ull>(e), j);
      const ull jbu = __shfl_sync(kAll, bu, j), jbv = __shfl_sync(kAll, bv, j);
      const uint32_t jdu = __shfl_sync(kAll, du, j), jdv = __shfl_sync(kAll, dv, j);
      const bool su = jdu <= jdv;
      const uint32_t* S = adj + (su ? jbu : jbv);
      const uint32_t* L = adj + (su ? jbv : jbu);
      const uint32_t ns = su ? jdu : jdv, nl = su ? jdv : jdu;
      ull w0 = 0, w1 = 0;
      if (WRITE) {
        w0 = toff[je];
        w1 = toff[rev[je]];
      }
      uint32_t k = 0;
      for (uint32_t base = 0; base < ns; base += 32) {
        const uint32_t i = base + lane;
        bool hit = false;
        uint32_t p = 0;
        if (i < ns) {
          const uint32_t x = S[i];
          p = lb32(L, nl, x);
          hit = p < nl && L[p] == x;
        }
        const unsigned m = __ballot_sync(kAll, hit);
        if (WRITE && hit) {
          const uint32_t at = k + __popc(m & ((1u << lane) - 1u));
          tent[w0 + at] = su ? i : p;
          tent[w1 + at] = su ? p : i;
        }
        k += __popc(m);
      }
      if (!WRITE && lane == 0) tri[je] = k;
    }
  }
}

__global__ void mirror_tri_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ adj,
                                  const ull* __restrict__ rev, uint64_t slots, uint32_t* tri,
                                  ull* __restrict__ wide) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < slots;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t t;
    if (src[e] > adj[e]) {
      t = tri[rev[e]];
      tri[e] = t;
    } else {
      t = tri[e];
    }
    wide[e] = t;
  }
}

// |T(e) & [0, pos of adj[e] in N(src e))| (the edges of G[N(c)] below x at x).
__global__ void low_kernel(const ull* __restrict__ off, const uint32_t* __restrict__ src,
                           const uint32_t* __restrict__ tri, const ull* __restrict__ toff,
                           const uint32_t* __restrict__ tent, uint64_t slots, ull* __restrict__ low) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < slots;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t j = static_cast<uint32_t>(e - off[src[e]]);
    low[e] = lb32(tent + toff[e], tri[e], j);
  }
}

__global__ void lowpref_kernel(const ull* __restrict__ off, const uint32_t* __restrict__ src,
                               const ull* __restrict__ scan, uint64_t slots, ull* __restrict__ lowpref) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < slots;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    lowpref[e] = scan[e] - scan[off[src[e]]];
}

// k4 of entry w of T(c, x): |T(c, x) & T(c, w)| (one warp per slot, lanes over entries).
__global__ void __launch_bounds__(256) k4_kernel(const ull* __restrict__ off, const uint32_t* __restrict__ src,
                                                 const uint32_t* __restrict__ tri, const ull* __restrict__ toff,
                                                 const uint32_t* __restrict__ tent, uint64_t slots,
                                                 uint32_t* __restrict__ k4, ull* next) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    ull f = 0;
    if (lane == 0) f = atomicAdd(next, 1ull);
    f = __shfl_sync(kAll, f, 0);
    if (f >= slots) break;
    const uint32_t tf = tri[f];
    if (tf == 0) continue;
    const ull c0 = off[src[f]];
    const uint32_t* Tf = tent + toff[f];
    for (uint32_t j = lane; j < tf; j += 32) {
      const ull g = c0 + Tf[j];
      k4[toff[f] + j] = isect_count(Tf, tf, tent + toff[g], tri[g]);
    }
  }
}

// --------------------------------------------------------- fast kernels ---

__device__ __forceinline__ bool grab_chunk(const FastArgs& a, int lane, uint64_t& e0) {
  ull chunk = 0;
  if (lane == 0) chunk = atomicAdd(a.next_chunk, 1ull);
  chunk = __shfl_sync(kAll, chunk, 0);
  uint64_t g = chunk;
  if (a.num_shards > 1) {
    if (chunk >= a.map_pref[a.map_k]) return false;
    uint32_t k = 0;
    while (a.map_pref[k + 1] <= chunk) ++k;
    g = a.map_begin[k] + (chunk - a.map_pref[k]);
  }
  e0 = a.e_lo + g * kSlotChunk;
  return e0 < a.e_hi;
}

__device__ __forceinline__ bool owns_chunk(const FastArgs& a, uint64_t q) {
  if (a.num_shards <= 1) return true;
  for (uint32_t k = 0; k < a.map_k; ++k) {
    const ull b = a.map_begin[k], len = a.map_pref[k + 1] - a.map_pref[k];
    if (q >= b && q < b + len) return true;
  }
  return false;
}

// a centre belongs to the shard that owns the chunk of its first slot
__device__ __forceinline__ bool owns_center(const FastArgs& a, ull c) {
  return a.num_shards <= 1 || owns_chunk(a, a.off[c] / kSlotChunk);
}

// The unit slot of walked slot e0 + lane (valid = inside the walk).
__device__ __forceinline__ uint64_t unit_slot(const FastArgs& a, uint64_t ep, bool& valid) {
  valid = ep < a.e_hi;
  return valid ? (a.via_rev ? a.t.rev[ep] : ep) : 0;
}

__device__ __forceinline__ void checked_add(ull& acc, ull add, bool& ovf) {
  const ull r = acc + add;
  ovf |= r < acc;
  acc = r;
}

__device__ __forceinline__ void flush(const FastArgs& a, ull cnt, ull units, bool ovf, int lane) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {  // checked warp sum of the checked per-lane partials
    const ull o = __shfl_xor_sync(kAll, cnt, d);
    checked_add(cnt, o, ovf);
  }
  if (lane == 0) {
    if (cnt) {
      const ull old = atomicAdd(a.count, cnt);
      if (old + cnt < old) ovf = true;
    }
    if (units) atomicAdd(a.units, units);
  }
  ovf = __any_sync(kAll, ovf);
  if (lane == 0 && ovf) atomicOr(a.overflow, 1u);
}

// star4 unit terms over T' entries [j0, k) with stride: s1 (sum of |T(c,t) & [0,i)|)
// and s2 (edges inside T' counted at their larger end).
__device__ __forceinline__ void star4_terms(const FastArgs& a, ull c0, const uint32_t* tl, uint32_t i, uint32_t k,
                                            uint32_t j0, uint32_t stride, ull& s1, ull& s2) {
  for (uint32_t j = j0; j < k; j += stride) {
    const uint32_t q = tl[j];
    const ull f = c0 + q;
    const uint32_t* Tf = a.t.tent + a.t.toff[f];
    const uint32_t tf = a.t.tri[f];
    s1 += lb32(Tf, tf, i);
    s2 += isect_count(Tf, lb32(Tf, tf, q), tl, j);
  }
}

__global__ void __launch_bounds__(kFastThreads) star4_kernel(const FastArgs a) {
  const int lane = threadIdx.x & 31;
  ull cnt = 0, units = 0;
  bool ovf = false;
  uint64_t e0;
  while (grab_chunk(a, lane, e0)) {
    bool mine;
    const uint64_t e = unit_slot(a, e0 + lane, mine);
    uint32_t c = 0, p = 0;
    if (mine) {
      c = a.src[e];
      p = a.adj[e];
      mine = p >= a.root_lo && p < a.root_hi;  // unit (v0, v1) = (p, c)
    }
    units += __popc(__ballot_sync(kAll, mine));
    ull c0 = 0, base = 0;
    uint32_t i = 0, k = 0;
    const uint32_t* tl = nullptr;
    if (mine) {
      c0 = a.off[c];
      i = static_cast<uint32_t>(e - c0);
      tl = a.t.tent + a.t.toff[e];
      k = lb32(tl, a.t.tri[e], i);
      const ull X = i - k;
      base = X * (X - 1) / 2 - a.t.lowpref[e];  // mod 2^64; the true total is >= 0
    }
    const bool small = mine && k <= 4;
    if (small) {
      ull s1 = 0, s2 = 0;
      star4_terms(a, c0, tl, i, k, 0, 1, s1, s2);
      checked_add(cnt, base + s1 - s2, ovf);
    }
    unsigned big = __ballot_sync(kAll, mine && !small);
    while (big) {
      const int j = __ffs(big) - 1;
      big &= big - 1;
      const ull jc0 = __shfl_sync(kAll, c0, j);
      const uint32_t ji = __shfl_sync(kAll, i, j), jk = __shfl_sync(kAll, k, j);
      const uint32_t* jtl = reinterpret_cast<const uint32_t*>(
          __shfl_sync(kAll, reinterpret_cast<ull>(tl), j));
      ull s1 = 0, s2 = 0;
      star4_terms(a, jc0, jtl, ji, jk, lane, 32, s1, s2);
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == j) checked_add(cnt, base + s1 - s2, ovf);
    }
  }
  flush(a, cnt, units, ovf, lane);
}

// Tailed triangle (center v1: slot (v1, v0)) and diamond (center v0: slot
// (v0, v1)): one sum over v2 in P & [0, v0) of T-list terms; lanes take units,
// units with |P| > 4 go to the whole warp.
template <int KIND>
__device__ __forceinline__ ull star_terms(const FastArgs& a, ull c0, const uint32_t* P, uint32_t np, uint32_t i0,
                                          uint32_t p1, uint32_t j0, uint32_t stride) {
  ull s = 0;
  for (uint32_t j = j0; j < np; j += stride) {
    const uint32_t q2 = P[j];
    if (q2 >= i0) break;  // v2 < v0 (positions ascend with ids)
    const ull f = c0 + q2;
    const uint32_t* T2 = a.t.tent + a.t.toff[f];
    const uint32_t t2 = a.t.tri[f];
    if (KIND == kFastTailedTriangle) {
      s += static_cast<ull>(p1) - np - t2 + isect_count(T2, t2, P, np);  // p1 carries d1 here
    } else {
      const uint32_t lo = lb32(T2, t2, p1);
      s += lo - isect_count(T2, lo, P, lb32(P, np, p1));
    }
  }
  return s;
}

template <int KIND>
__global__ void __launch_bounds__(kFastThreads) star_kernel(const FastArgs a) {
  const int lane = threadIdx.x & 31;
  ull cnt = 0, units = 0;
  bool ovf = false;
  uint64_t e0;
  while (grab_chunk(a, lane, e0)) {
    bool mine;
    const uint64_t e = unit_slot(a, e0 + lane, mine);
    uint32_t c = 0, p = 0, v0 = 0;
    if (mine) {
      c = a.src[e];
      p = a.adj[e];
      v0 = KIND == kFastTailedTriangle ? p : c;  // tt: slot (v1, v0); diamond: slot (v0, v1)
      mine = v0 >= a.root_lo && v0 < a.root_hi;
    }
    units += __popc(__ballot_sync(kAll, mine));
    ull c0 = 0;
    uint32_t np = 0, i0 = 0, p1 = 0;
    const uint32_t* P = nullptr;
    if (mine) {
      c0 = a.off[c];
      P = a.t.tent + a.t.toff[e];
      np = a.t.tri[e];
      if (KIND == kFastTailedTriangle) {
        i0 = static_cast<uint32_t>(e - c0);                      // pos of v0 in N(v1)
        p1 = static_cast<uint32_t>(a.off[c + 1] - c0);           // d1
      } else {
        i0 = lb32(a.adj + c0, static_cast<uint32_t>(a.off[c + 1] - c0), c);  // #N(v0) below v0
        p1 = static_cast<uint32_t>(e - c0);                                   // pos of v1 in N(v0)
      }
    }
    const bool small = mine && np <= 4;
    if (small) checked_add(cnt, star_terms<KIND>(a, c0, P, np, i0, p1, 0, 1), ovf);
    unsigned big = __ballot_sync(kAll, mine && !small);
    while (big) {
      const int j = __ffs(big) - 1;
      big &= big - 1;
      const ull jc0 = __shfl_sync(kAll, c0, j);
      const uint32_t jnp = __shfl_sync(kAll, np, j), ji0 = __shfl_sync(kAll, i0, j), jp1 = __shfl_sync(kAll, p1, j);
      const uint32_t* jP = reinterpret_cast<const uint32_t*>(__shfl_sync(kAll, reinterpret_cast<ull>(P), j));
      const ull s = warp_sum(star_terms<KIND>(a, jc0, jP, jnp, ji0, jp1, lane, 32));
      if (lane == j) checked_add(cnt, s, ovf);
    }
  }
  flush(a, cnt, units, ovf, lane);
}

// Tailed diamond (a): one warp per unit with P = T(v1, v0) non-empty.
// FULL: the S6 term is left out (summed in closed form by the caller).
template <bool FULL>
__global__ void __launch_bounds__(kFastThreads) tda_kernel(const FastArgs a) {
  const uint64_t dmax = a.dmax;
  __shared__ uint32_t ntouched[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  uint32_t* alpha = a.scratch + gw * a.scratch_words;
  uint32_t* touched = alpha + dmax;
  uint32_t* bm = touched + dmax;
  ull cnt = 0, units = 0;
  bool ovf = false;
  uint64_t e0;
  while (grab_chunk(a, lane, e0)) {
    bool mine;
    const uint64_t e = unit_slot(a, e0 + lane, mine);
    uint32_t p = 0;
    if (mine) {
      p = a.adj[e];
      mine = p >= a.root_lo && p < a.root_hi;
    }
    units += __popc(__ballot_sync(kAll, mine));
    unsigned todo = __ballot_sync(kAll, mine && a.t.tri[mine ? e : 0] > 0);
    while (todo) {
      const int jl = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t ue = __shfl_sync(kAll, static_cast<ull>(e), jl);
      const uint32_t c = a.src[ue];
      const ull c0 = a.off[c];
      const uint32_t d1 = static_cast<uint32_t>(a.off[c + 1] - c0);
      const uint32_t i0 = static_cast<uint32_t>(ue - c0);
      const uint32_t* P = a.t.tent + a.t.toff[ue];
      const uint32_t np = a.t.tri[ue];
      if (lane == 0) ntouched[wib] = 0;
      for (uint32_t j = lane; j < np; j += 32) atomicOr(&bm[P[j] >> 5], 1u << (P[j] & 31));
      __syncwarp();
      ull S2 = 0, S5 = 0, S6 = 0;
      for (uint32_t jj = 0; jj < np; ++jj) {
        const uint32_t q2 = P[jj];
        const ull f2 = c0 + q2;
        const uint32_t* T2 = a.t.tent + a.t.toff[f2];
        const uint32_t t2 = a.t.tri[f2];
        const uint32_t lb = lb32(T2, t2, i0);
        uint32_t acnt = 0, c02 = 0;
        for (uint32_t r = lane; r < t2; r += 32) {
          const uint32_t x = T2[r];
          const bool inP = (bm[x >> 5] >> (x & 31)) & 1u;
          if (inP) {
            ++c02;
            if (FULL) continue;
            // w = x in P & T(v2): S6 += |T2[0,lb) & T(c,w) - P|
            const ull g = c0 + x;
            const uint32_t* Tg = a.t.tent + a.t.toff[g];
            const uint32_t tg = lb32(Tg, a.t.tri[g], i0);
            const uint32_t* S = lb <= tg ? T2 : Tg;
            const uint32_t* L = lb <= tg ? Tg : T2;
            const uint32_t ns = lb <= tg ? lb : tg, nl = lb <= tg ? tg : lb;
            uint32_t lo = 0;
            for (uint32_t s = 0; s < ns && lo < nl; ++s) {
              const uint32_t y = S[s];
              lo += lb32(L + lo, nl - lo, y);
              if (lo < nl && L[lo] == y && !((bm[y >> 5] >> (y & 31)) & 1u)) ++S6;
            }
          } else if (r < lb) {
            ++acnt;
            if (atomicAdd(&alpha[x], 1u) == 0u) touched[atomicAdd(&ntouched[wib], 1u)] = x;
            S5 += a.t.k4[a.t.toff[f2] + r];
          }
        }
        const ull A = warp_sum(acnt), C = warp_sum(c02);
        if (lane == 0) S2 += A * (t2 - C);
      }
      __syncwarp();
      const uint32_t nt = ntouched[wib];
      ull pairs = 0, S3 = 0, S4 = 0;
      for (uint32_t z = lane; z < nt; z += 32) {
        const uint32_t x = touched[z];
        touched[z] = 0u;  // every scratch word is zero between units (layouts differ per kind)
        const ull al = alpha[x];
        alpha[x] = 0u;
        pairs += al;
        S3 += static_cast<ull>(a.t.tri[c0 + x]) * al;
        S4 += al * al;
      }
      for (uint32_t j = lane; j < np; j += 32) bm[P[j] >> 5] = 0u;
      pairs = warp_sum(pairs);
      S2 = warp_sum(S2);
      S3 = warp_sum(S3);
      S4 = warp_sum(S4);
      S5 = warp_sum(S5);
      S6 = warp_sum(S6);
      __syncwarp();
      if (lane == jl) {
        const ull unit = static_cast<ull>(d1 - np) * pairs - S2 - S3 + S4 + S5 - S6;  // mod 2^64
        checked_add(cnt, unit, ovf);
      }
    }
  }
  flush(a, cnt, units, ovf, lane);
}

// ------------------------------------------------- two-center kinds ---
// house and tailed diamond (b) are not star-shaped: their units need a
// codegree table of one unit vertex (dense, per CTA, one center at a time:
// the 2-hop scatter of N(center) is shared by every unit of that center) and
// local codegree tables inside ego networks (per warp, over positions of one
// adjacency list).  Partial sums land in per-slot accumulators; a last pass
// combines them per unit.  Derivations (checked unit by unit against the
// reference, tests/test_fast.py):
//  house, unit (v0, v1), v1 < v0, A1 = N1 - N[v0], A0 = N0 - N[v1], T = T(v0,v1):
//    count = |T| e(A1, A0) - H(v0, v1) - H(v1, v0) + W(v0, v1)
//    H(a, b) = sum_{x in N(b) - N[a]} al(x) (c_a(x) - al(x) - 1), al(x) = |N(x) & T(a,b)|
//    e(A1, A0) = sum_{x in A1} (c_a(x) - al(x) - 1)            (a = v0, b = v1)
//    W = sum_{t in T} C4 of (v0, v1) inside G[N(t)]  (ego_w_kernel)
//  tailed diamond (b), unit (v0, v1), P = T(v0, v1), v2 in P & [0, v0),
//    Y(v2) = T(v0,v2) - N[v1]:  leaf(v3) = d1 - |P| - tri(v1,v2) - c_v1(v3)
//      + |P & N2| + |P & N3| + |N1 & N2 & N3| - |P & N2 & N3|  (inclusion-exclusion)
//    the N1 & N2 & N3 term is summed per v2 inside G[N(v2)] (ego_w_kernel).
struct WarpScratch {
  uint32_t* t0;
  uint32_t* t1;
  uint32_t* touched;
  uint32_t* bm;
};

__device__ __forceinline__ WarpScratch warp_scratch(const FastArgs& a) {
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  WarpScratch w;
  w.t0 = a.scratch + gw * a.scratch_words;
  w.t1 = w.t0 + a.dmax;
  w.touched = w.t1 + a.dmax;
  w.bm = w.touched + a.dmax;
  return w;
}

__device__ __forceinline__ bool bit(const uint32_t* bm, uint32_t x) { return (bm[x >> 5] >> (x & 31)) & 1u; }

// CTA-wide 2-hop scatter of center c into the dense table: cnt[z] += 1 per
// path c - y - z (val = 1), or cnt[z] = 0 (reset, val = 0).
__device__ __forceinline__ void dense_scatter(const FastArgs& a, uint32_t* cnt, ull co, uint32_t dc, bool reset) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t yy = wib; yy < dc; yy += nw) {
    const uint32_t y = a.adj[co + yy];
    const ull yo = a.off[y];
    const uint32_t dy = static_cast<uint32_t>(a.off[y + 1] - yo);
    for (uint32_t k = lane; k < dy; k += 32) {
      if (reset) cnt[a.adj[yo + k]] = 0u;
      else atomicAdd(&cnt[a.adj[yo + k]], 1u);
    }
  }
}

// Next center for this CTA (all threads call; returns the same value to all).
__device__ __forceinline__ ull next_center(const FastArgs& a, ull* sh) {
  __syncthreads();
  if (threadIdx.x == 0) *sh = atomicAdd(a.next2, 1ull);
  __syncthreads();
  return *sh;
}

// house: e(A1,A0)|T| -> acc0[(a,b)] (b < a), H(a,b) -> acc1[(a,b)], center a.
// path4 (PATH4): |A1||A0| - e(A1,A0) -> acc0[(a,b)] (b < a), no H.
template <bool PATH4>
__global__ void __launch_bounds__(kFastThreads) house_eh_kernel(const FastArgs a) {
  __shared__ ull center_sh;
  __shared__ uint32_t nt_sh[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* cnt = a.dense + static_cast<uint64_t>(blockIdx.x) * a.n;
  const WarpScratch w = warp_scratch(a);
  for (;;) {
    const ull ca = next_center(a, &center_sh);
    if (ca >= a.n) break;
    const ull ao = a.off[ca];
    const uint32_t da = static_cast<uint32_t>(a.off[ca + 1] - ao);
    if (da == 0) continue;
    dense_scatter(a, cnt, ao, da, false);
    __syncthreads();
    for (uint32_t bb = wib; bb < da; bb += nw) {
      const ull e = ao + bb;
      const uint32_t b = a.adj[e];
      if (PATH4 && !(b < ca)) continue;  // path4 needs e() of units (a, b), b < a, only
      const ull r = a.t.rev[e];
      const ull bo = a.off[b];
      const uint32_t db = static_cast<uint32_t>(a.off[b + 1] - bo);
      const uint32_t pa = static_cast<uint32_t>(r - bo);
      const uint32_t* Tba = a.t.tent + a.t.toff[r];
      const uint32_t nT = a.t.tri[r];
      if (lane == 0) nt_sh[wib] = 0;
      for (uint32_t j = lane; j < nT; j += 32) atomicOr(&w.bm[Tba[j] >> 5], 1u << (Tba[j] & 31));
      __syncwarp();
      for (uint32_t j = 0; j < nT; ++j) {  // al(x) = |T(b,x) & T(b,a)|, x in N(b)
        const ull f = bo + Tba[j];
        const uint32_t* Tf = a.t.tent + a.t.toff[f];
        const uint32_t tf = a.t.tri[f];
        for (uint32_t k = lane; k < tf; k += 32) {
          const uint32_t x = Tf[k];
          if (atomicAdd(&w.t0[x], 1u) == 0u) w.touched[atomicAdd(&nt_sh[wib], 1u)] = x;
        }
      }
      __syncwarp();
      const bool needE = b < ca;
      ull Esum = 0, sumA = 0, H = 0;
      if (needE)
        for (uint32_t x = lane; x < db; x += 32)
          if (!bit(w.bm, x) && x != pa) Esum += cnt[a.adj[bo + x]];
      const uint32_t nt = nt_sh[wib];
      for (uint32_t z = lane; z < nt; z += 32) {
        const uint32_t x = w.touched[z];
        w.touched[z] = 0u;
        const ull al = w.t0[x];
        w.t0[x] = 0u;
        if (!bit(w.bm, x) && x != pa) {
          sumA += al;
          H += al * (static_cast<ull>(cnt[a.adj[bo + x]]) - al - 1);
        }
      }
      __syncwarp();
      for (uint32_t j = lane; j < nT; j += 32) w.bm[Tba[j] >> 5] = 0u;
      Esum = warp_sum(Esum);
      sumA = warp_sum(sumA);
      H = warp_sum(H);
      __syncwarp();
      if (lane == 0) {
        const ull A1 = static_cast<ull>(db - nT - 1);  // |N(b) - N[a]|
        const ull E = Esum - sumA - A1;
        if (PATH4) {
          if (needE) a.acc0[e] = A1 * static_cast<ull>(da - nT - 1) - E;
        } else {
          a.acc1[e] = H;
          if (needE) a.acc0[e] = static_cast<ull>(nT) * E;
        }
      }
    }
    __syncthreads();
    dense_scatter(a, cnt, ao, da, true);
  }
}

// tailed diamond (b), center v1 (dense c_v1): every term of a unit (v0, v1)
// except the N1 & N2 & N3 one -> acc0[(v0, v1)].
__global__ void __launch_bounds__(kFastThreads) tdb_unit_kernel(const FastArgs a) {
  __shared__ ull center_sh;
  __shared__ uint32_t nt_sh[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* cnt = a.dense + static_cast<uint64_t>(blockIdx.x) * a.n;
  const WarpScratch w = warp_scratch(a);
  for (;;) {
    const ull v1 = next_center(a, &center_sh);
    if (v1 >= a.n) break;
    const ull o1 = a.off[v1];
    const uint32_t d1 = static_cast<uint32_t>(a.off[v1 + 1] - o1);
    if (d1 == 0) continue;
    dense_scatter(a, cnt, o1, d1, false);
    __syncthreads();
    for (uint32_t bb = wib; bb < d1; bb += nw) {
      const uint32_t v0 = a.adj[o1 + bb];
      const ull e = a.t.rev[o1 + bb];  // the unit's slot (v0, v1)
      const ull oo = a.off[v0];
      const uint32_t d0 = static_cast<uint32_t>(a.off[v0 + 1] - oo);
      const uint32_t p1 = static_cast<uint32_t>(e - oo);
      const uint32_t* P = a.t.tent + a.t.toff[e];
      const uint32_t np = a.t.tri[e];
      if (np == 0) {
        if (lane == 0) a.acc0[e] = 0;
        continue;
      }
      const uint32_t i0 = lb32(a.adj + oo, d0, v0);  // v2 < v0  <=>  position < i0
      if (lane == 0) nt_sh[wib] = 0;
      for (uint32_t j = lane; j < np; j += 32) atomicOr(&w.bm[P[j] >> 5], 1u << (P[j] & 31));
      __syncwarp();
      ull T1 = 0, T5 = 0;
      for (uint32_t j = 0; j < np; ++j) {
        const uint32_t q2 = P[j];
        const bool bounded = q2 < i0;
        const ull f2 = oo + q2;
        const uint32_t* T02 = a.t.tent + a.t.toff[f2];
        const uint32_t t02 = a.t.tri[f2];
        uint32_t c = 0;
        for (uint32_t k = lane; k < t02; k += 32) {
          const uint32_t x = T02[k];
          if (bit(w.bm, x)) {
            ++c;
            if (bounded) {  // w = x in P & N(v2): |T(v0,w) & T02 - P - {v1}|
              const ull g = oo + x;
              const uint32_t* Tg = a.t.tent + a.t.toff[g];
              const uint32_t tg = a.t.tri[g];
              const uint32_t* S = t02 <= tg ? T02 : Tg;
              const uint32_t* L = t02 <= tg ? Tg : T02;
              const uint32_t ns = t02 <= tg ? t02 : tg, nl = t02 <= tg ? tg : t02;
              uint32_t lo = 0;
              for (uint32_t s = 0; s < ns && lo < nl; ++s) {
                const uint32_t y = S[s];
                lo += lb32(L + lo, nl - lo, y);
                if (lo < nl && L[lo] == y && !bit(w.bm, y) && y != p1) ++T5;
              }
            }
          } else if (x != p1) {
            if (atomicAdd(&w.t0[x], 1u) == 0u) w.touched[atomicAdd(&nt_sh[wib], 1u)] = x;  // |N3 & P|
            if (bounded) atomicAdd(&w.t1[x], 1u);                                          // b(v3)
          }
        }
        if (bounded) {
          const ull C = warp_sum(c);
          if (lane == 0) {
            const uint32_t v2 = a.adj[f2];
            const uint32_t tri12 = a.t.tri[o1 + lb32(a.adj + o1, d1, v2)];
            const ull Y = t02 - C - 1;
            T1 += Y * (static_cast<ull>(d1) - np - tri12 + C);
          }
        }
      }
      __syncwarp();
      const uint32_t nt = nt_sh[wib];
      ull T2 = 0, T3 = 0;
      for (uint32_t z = lane; z < nt; z += 32) {
        const uint32_t x = w.touched[z];
        w.touched[z] = 0u;
        const ull A = w.t0[x], B = w.t1[x];
        w.t0[x] = 0u;
        w.t1[x] = 0u;
        T2 += B * cnt[a.adj[oo + x]];
        T3 += B * A;
      }
      __syncwarp();
      for (uint32_t j = lane; j < np; j += 32) w.bm[P[j] >> 5] = 0u;
      T1 = warp_sum(T1);
      T2 = warp_sum(T2);
      T3 = warp_sum(T3);
      T5 = warp_sum(T5);
      __syncwarp();
      if (lane == 0) a.acc0[e] = T1 - T2 + T3 - T5;
    }
    __syncthreads();
    dense_scatter(a, cnt, o1, d1, true);
  }
}

// Ego-network pair sums, one warp per slot (t, a): cl(x) = |T(t,x) & T(t,a)|
// over positions of N(t), then for b in T(t,a):
//   house (b < a):  sum_{x in T(t,b) - T(t,a) - {a}} (cl(x) - 1 - |T(t,x) & T(t,a) & T(t,b)|) -> acc2[(a, b)]
//   tdb   (b > t):  sum_{x in T(t,b) - T(t,a) - {a}} cl(x)                                   -> acc2[(b, a)]
template <int KIND>
__global__ void __launch_bounds__(kFastThreads) ego_w_kernel(const FastArgs a) {
  __shared__ uint32_t nt_sh[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const WarpScratch w = warp_scratch(a);
  uint64_t e0;
  while (grab_chunk(a, lane, e0)) {
    const uint64_t me = e0 + lane;
    // house needs |N_L(a)| >= 2 (b and a 4-cycle vertex); tdb any non-empty row
    unsigned todo = __ballot_sync(kAll, me < a.slots && a.t.tri[me < a.slots ? me : 0] > (KIND == kFastHouse ? 1u : 0u));
    while (todo) {
      const int jl = __ffs(todo) - 1;
      todo &= todo - 1;
      const ull e = e0 + jl;
      const uint32_t t = a.src[e], av = a.adj[e];
      const ull to = a.off[t];
      const uint32_t pa = static_cast<uint32_t>(e - to);
      const uint32_t* Ta = a.t.tent + a.t.toff[e];
      const uint32_t na = a.t.tri[e];
      if (lane == 0) nt_sh[wib] = 0;
      for (uint32_t j = lane; j < na; j += 32) atomicOr(&w.bm[Ta[j] >> 5], 1u << (Ta[j] & 31));
      __syncwarp();
      for (uint32_t j = 0; j < na; ++j) {
        const ull f = to + Ta[j];
        const uint32_t* Tf = a.t.tent + a.t.toff[f];
        const uint32_t tf = a.t.tri[f];
        for (uint32_t k = lane; k < tf; k += 32) {
          const uint32_t x = Tf[k];
          if (atomicAdd(&w.t0[x], 1u) == 0u) w.touched[atomicAdd(&nt_sh[wib], 1u)] = x;
        }
      }
      __syncwarp();
      for (uint32_t j = 0; j < na; ++j) {
        const uint32_t pb = Ta[j];
        const uint32_t bv = a.adj[to + pb];
        if (KIND == kFastHouse ? !(pb < pa) : !(bv > t)) continue;
        const ull f = to + pb;
        const uint32_t* Tb = a.t.tent + a.t.toff[f];
        const uint32_t nb = a.t.tri[f];
        ull sum = 0, tri3 = 0;
        for (uint32_t k = lane; k < nb; k += 32) {
          const uint32_t x = Tb[k];
          if (!bit(w.bm, x)) {
            if (x != pa) sum += KIND == kFastHouse ? static_cast<ull>(w.t0[x]) - 1 : static_cast<ull>(w.t0[x]);
          } else if (KIND == kFastHouse) {  // w = x in T(t,a) & T(t,b): |T(t,w) & T(t,b) - T(t,a) - {a}|
            const ull g = to + x;
            const uint32_t* Tg = a.t.tent + a.t.toff[g];
            const uint32_t tg = a.t.tri[g];
            const uint32_t* S = nb <= tg ? Tb : Tg;
            const uint32_t* L = nb <= tg ? Tg : Tb;
            const uint32_t ns = nb <= tg ? nb : tg, nl = nb <= tg ? tg : nb;
            uint32_t lo = 0;
            for (uint32_t s = 0; s < ns && lo < nl; ++s) {
              const uint32_t y = S[s];
              lo += lb32(L + lo, nl - lo, y);
              if (lo < nl && L[lo] == y && !bit(w.bm, y) && y != pa) ++tri3;
            }
          }
        }
        sum = warp_sum(sum) - warp_sum(tri3);
        if (lane == 0 && sum) {
          ull slot;
          if (KIND == kFastHouse) {  // (a, b)
            const ull ao = a.off[av];
            slot = ao + lb32(a.adj + ao, static_cast<uint32_t>(a.off[av + 1] - ao), bv);
          } else {  // (v0, v1) = (b, a)
            const ull bo = a.off[bv];
            slot = bo + lb32(a.adj + bo, static_cast<uint32_t>(a.off[bv + 1] - bo), av);
          }
          atomicAdd(&a.acc2[slot], sum);
        }
      }
      __syncwarp();
      const uint32_t nt = nt_sh[wib];
      for (uint32_t z = lane; z < nt; z += 32) {
        w.t0[w.touched[z]] = 0u;
        w.touched[z] = 0u;
      }
      for (uint32_t j = lane; j < na; j += 32) w.bm[Ta[j] >> 5] = 0u;
      __syncwarp();
    }
  }
}

// Rectangle (both plans): one CTA per centre c, its neighbours u in ascending
// order; the table holds the 2-hop scatter of N(c) & [0, u) when unit (c, u)
// is evaluated (then u's own list is added).  NAMED: units u > c (c = v1);
// motif: units u < c (c = v0).
template <bool NAMED, bool ARRAY>
__global__ void __launch_bounds__(kFastThreads) rect_kernel(const FastArgs a) {
  __shared__ ull center_sh;
  __shared__ ull red_sh[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* cnt = a.dense + static_cast<uint64_t>(blockIdx.x) * a.n;
  uint32_t* bm = a.scratch + static_cast<uint64_t>(blockIdx.x) * a.scratch_words;  // per CTA: bits over N(u)
  ull total = 0, units = 0;  // thread 0
  bool ovf = false;
  for (;;) {
    const ull c = next_center(a, &center_sh);
    if (c >= a.n) break;
    if (!ARRAY && !owns_center(a, c)) continue;  // shards split the centres
    const ull co = a.off[c];
    const uint32_t dc = static_cast<uint32_t>(a.off[c + 1] - co);
    // named: every neighbour is scattered, units are the u > c; motif: units
    // and scatters stop at the first u > c
    const uint32_t steps = NAMED ? dc : lb32(a.adj + co, dc, static_cast<uint32_t>(c));
    for (uint32_t k = 0; k < steps; ++k) {
      const uint32_t u = a.adj[co + k];
      // ARRAY: every unit's value goes to acc0[its slot (v0, v1)] (cached for
      // root-range calls); else the units in the root range are summed here
      const bool unit = (NAMED ? u > c : true) &&
                        (ARRAY || ((NAMED ? u : c) >= a.root_lo && (NAMED ? u : c) < a.root_hi));
      if (unit) {
        const ull uo = a.off[u];
        const uint32_t du = static_cast<uint32_t>(a.off[u + 1] - uo);
        const ull euc = a.t.rev[co + k];  // slot (u, c)
        const uint32_t* T = a.t.tent + a.t.toff[euc];
        const uint32_t nT = a.t.tri[euc];
        const uint32_t pc = static_cast<uint32_t>(euc - uo);  // position of c in N(u)
        const uint32_t iu = lb32(a.adj + uo, du, u);         // #N(u) below u
        for (uint32_t j = threadIdx.x; j < nT; j += blockDim.x) atomicOr(&bm[T[j] >> 5], 1u << (T[j] & 31));
        __syncthreads();
        ull s = 0;
        for (uint32_t x = threadIdx.x; x < pc; x += blockDim.x)
          if (!bit(bm, x)) s += cnt[a.adj[uo + x]];
        for (uint32_t j = wib; j < nT; j += nw) {  // t in T(u,c) & [0,u)
          const uint32_t q = T[j];
          if (q >= iu) break;
          const ull f = uo + q;
          const uint32_t* Tf = a.t.tent + a.t.toff[f];
          const uint32_t tf = lb32(Tf, a.t.tri[f], pc);  // x < c
          for (uint32_t r = lane; r < tf; r += 32)
            if (!bit(bm, Tf[r])) --s;  // mod 2^64; the unit total is >= 0
        }
        s = warp_sum(s);
        if (lane == 0) red_sh[wib] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
          ull v = 0;
          for (int w2 = 0; w2 < nw; ++w2) v += red_sh[w2];
          if (ARRAY) {
            a.acc0[NAMED ? euc : co + k] = v;  // the unit's slot (v0, v1)
          } else {
            checked_add(total, v, ovf);
            ++units;
          }
        }
        for (uint32_t j = threadIdx.x; j < nT; j += blockDim.x) bm[T[j] >> 5] = 0u;
      }
      // add u's list: cnt[z] += 1 for z in N(u)
      {
        const ull uo = a.off[u];
        const uint32_t du = static_cast<uint32_t>(a.off[u + 1] - uo);
        for (uint32_t z = threadIdx.x; z < du; z += blockDim.x) atomicAdd(&cnt[a.adj[uo + z]], 1u);
      }
      __syncthreads();
    }
    for (uint32_t k = 0; k < steps; ++k) {
      const uint32_t u = a.adj[co + k];
      const ull uo = a.off[u];
      const uint32_t du = static_cast<uint32_t>(a.off[u + 1] - uo);
      for (uint32_t z = threadIdx.x; z < du; z += blockDim.x) cnt[a.adj[uo + z]] = 0u;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (total) {
      const ull old = atomicAdd(a.count, total);
      if (old + total < old) ovf = true;
    }
    if (units) atomicAdd(a.units, units);
    if (ovf) atomicOr(a.overflow, 1u);
  }
}

// Per unit slot e = (v0, v1): house count = acc0 - acc1[e] - acc1[rev e] + acc2
// (v1 < v0 only); tailed diamond (b) = acc0 + acc2.
template <int KIND>
__global__ void __launch_bounds__(kFastThreads) combine_kernel(const FastArgs a) {
  const int lane = threadIdx.x & 31;
  ull cnt = 0, units = 0;
  bool ovf = false;
  uint64_t e0;
  while (grab_chunk(a, lane, e0)) {
    bool mine;
    const uint64_t e = unit_slot(a, e0 + lane, mine);  // walks (v0, v1) slots directly
    uint32_t v0 = 0, v1 = 0;
    if (mine) {
      v0 = a.src[e];
      v1 = a.adj[e];
      mine = v0 >= a.root_lo && v0 < a.root_hi && (KIND == kFastTailedDiamondB || v1 < v0);  // rect/path4/house: v1 < v0
    }
    units += __popc(__ballot_sync(kAll, mine));
    if (mine) {
      const ull c = KIND == kFastHouse ? a.acc0[e] - a.acc1[e] - a.acc1[a.t.rev[e]] + a.acc2[e]
                    : (KIND == kFastPath4 || KIND == kFastRectangle || KIND == kFastRectangleMotif) ? a.acc0[e]
                                         : a.acc0[e] + a.acc2[e];
      checked_add(cnt, c, ovf);
    }
  }
  flush(a, cnt, units, ovf, lane);
}

// Flattened pass over the entries of the index lists T(base + P[j]) for j in
// [0, np): the warp's lanes take consecutive entries of their concatenation
// (32 lists at a time, owner found by a shuffle search over the exclusive
// scan), so short lists do not leave lanes idle.  aux(j) is a per-list word
// carried to every entry; f(k, r, x, eidx, auxv): list j0 + k, entry r of it,
// its value x, its index in tent.  All 32 lanes must call it; after(j, k) runs
// on lane k for list j = j0 + k once its entries are done.
template <class AUX, class F, class AFTER>
__device__ __forceinline__ void flat_entries(const FastArgs& a, ull base, const uint32_t* P, uint32_t np, AUX aux,
                                             F f, AFTER after) {
  const int lane = threadIdx.x & 31;
  for (uint32_t j0 = 0; j0 < np; j0 += 32) {
    const uint32_t j = j0 + lane;
    uint32_t len = 0, av = 0;
    ull to = 0;
    if (j < np) {
      const ull fs = base + P[j];
      len = a.t.tri[fs];
      to = a.t.toff[fs];
      av = aux(j, fs, len, to);
    }
    uint32_t incl = len;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(kAll, incl, d);
      if (lane >= d) incl += v;
    }
    const uint32_t tot = __shfl_sync(kAll, incl, 31), excl = incl - len;
    for (uint32_t t0 = 0; t0 < tot; t0 += 32) {
      const uint32_t idx = t0 + lane;
      int k = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t ex = __shfl_sync(kAll, excl, k + step);
        if (ex <= idx) k += step;
      }
      const ull o_to = __shfl_sync(kAll, to, k);
      const uint32_t o_ex = __shfl_sync(kAll, excl, k);
      const uint32_t o_av = __shfl_sync(kAll, av, k);
      if (idx < tot) {
        const uint32_t r = idx - o_ex;
        f(k, r, a.t.tent[o_to + r], o_to + r, o_av);
      }
    }
    __syncwarp();
    if (j < np) after(j, lane);
    __syncwarp();
  }
}

// ------------------------------------------------------ full-count mode ---
// For the whole root range the per-unit terms whose evaluation needs K4-level
// merges are summed in closed form over the triangle index instead (checked
// against per-unit evaluation in tests/test_fast.py):
//   sum over units of S6 (tailed diamond a) = sum_entries C(k4, 2) - 60 K5
//   sum over units of T5 (tailed diamond b) = 1/2 sum_entries k4 (k4 - 1) - 60 K5
//   house: sum_units W = 1/2 [sum_{(t,a)} sum_{x not in N_L[a]} cl (cl - 1)
//                             - sum_entries k4 (k4 - 1) + 120 K5]
//          sum_units (H(v0,v1) + H(v1,v0)) = sum over all ordered slots of H
// (K5 = number of 5-cliques, counted by the engine's clique-local path).  The
// kernels below add each CTA's signed share to part[2 blockIdx] as 128 bits.
typedef __int128 i128;


__device__ __forceinline__ i128 warp_sum128(i128 v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    const ull lo = __shfl_xor_sync(kAll, static_cast<ull>(v), d);
    const ull hi = __shfl_xor_sync(kAll, static_cast<ull>(v >> 64), d);
    v += static_cast<i128>((static_cast<unsigned __int128>(hi) << 64) | lo);
  }
  return v;
}

// every thread calls it once, at the end; sums the block and stores its share
__device__ void store_partial(const FastArgs& a, i128 v, ull units) {
  __shared__ i128 red[32];  // up to 1024 threads per CTA
  __shared__ ull ured[32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  __syncthreads();  // a kernel may call it once per sum: the previous read of red[] is over
  v = warp_sum128(v);
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) units += __shfl_xor_sync(kAll, units, d);
  if (lane == 0) {
    red[wib] = v;
    ured[wib] = units;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = 0;
    ull u = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      t += red[w];
      u += ured[w];
    }
    a.part[2 * blockIdx.x] = static_cast<ull>(t);
    a.part[2 * blockIdx.x + 1] = static_cast<ull>(t >> 64);
    if (u) atomicAdd(a.units, u);
  }
}

// house, centre a (dense c_a): sum over slots (a, b) of [b < a] |T| E(a, b) - H(a, b)
__global__ void __launch_bounds__(kFastThreads) house_full_center_kernel(const FastArgs a) {
  __shared__ ull center_sh;
  __shared__ uint32_t nt_sh[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* cnt = a.dense + static_cast<uint64_t>(blockIdx.x) * a.n;
  const WarpScratch w = warp_scratch(a);
  i128 acc = 0;
  ull units = 0;
  for (;;) {
    const ull ca = next_center(a, &center_sh);
    if (ca >= a.n) break;
    const ull ao = a.off[ca];
    const uint32_t da = static_cast<uint32_t>(a.off[ca + 1] - ao);
    if (da == 0 || !owns_center(a, ca)) continue;
    dense_scatter(a, cnt, ao, da, false);
    __syncthreads();
    for (uint32_t bb = wib; bb < da; bb += nw) {
      const ull e = ao + bb;
      const uint32_t b = a.adj[e];
      const ull r = a.t.rev[e];
      const ull bo = a.off[b];
      const uint32_t db = static_cast<uint32_t>(a.off[b + 1] - bo);
      const uint32_t pa = static_cast<uint32_t>(r - bo);
      const uint32_t* Tba = a.t.tent + a.t.toff[r];
      const uint32_t nT = a.t.tri[r];
      const bool needE = b < ca;
      if (lane == 0) {
        nt_sh[wib] = 0;
        if (needE) ++units;
      }
      for (uint32_t j = lane; j < nT; j += 32) atomicOr(&w.bm[Tba[j] >> 5], 1u << (Tba[j] & 31));
      __syncwarp();
      flat_entries(
          a, bo, Tba, nT, [](uint32_t, ull, uint32_t, ull) { return 0u; },
          [&](int, uint32_t, uint32_t x, ull, uint32_t) {
            if (atomicAdd(&w.t0[x], 1u) == 0u) w.touched[atomicAdd(&nt_sh[wib], 1u)] = x;
          },
          [](uint32_t, int) {});
      __syncwarp();
      ull Esum = 0, sumA = 0, H = 0;
      if (needE)
        for (uint32_t x = lane; x < db; x += 32)
          if (!bit(w.bm, x) && x != pa) Esum += cnt[a.adj[bo + x]];
      const uint32_t nt = nt_sh[wib];
      for (uint32_t z = lane; z < nt; z += 32) {
        const uint32_t x = w.touched[z];
        w.touched[z] = 0u;
        const ull al = w.t0[x];
        w.t0[x] = 0u;
        if (!bit(w.bm, x) && x != pa) {
          sumA += al;
          H += al * (static_cast<ull>(cnt[a.adj[bo + x]]) - al - 1);
        }
      }
      __syncwarp();
      for (uint32_t j = lane; j < nT; j += 32) w.bm[Tba[j] >> 5] = 0u;
      Esum = warp_sum(Esum);
      sumA = warp_sum(sumA);
      H = warp_sum(H);
      __syncwarp();
      if (lane == 0) {
        if (needE) acc += static_cast<i128>(nT) * static_cast<i128>(Esum - sumA - static_cast<ull>(db - nT - 1));
        acc -= static_cast<i128>(H);
      }
    }
    __syncthreads();
    dense_scatter(a, cnt, ao, da, true);
  }
  store_partial(a, acc, units);
}

// tailed diamond (b), centre v1 (dense c_v1): sum over its units of T1 - T2 + T3
// (T1's |P & N(v2)| is the index's k4 of entry v1 in T(v0, v2)).
__global__ void __launch_bounds__(kFastThreads) tdb_full_center_kernel(const FastArgs a) {
  __shared__ ull center_sh;
  __shared__ uint32_t nt_sh[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* cnt = a.dense + static_cast<uint64_t>(blockIdx.x) * a.n;
  const WarpScratch w = warp_scratch(a);
  i128 acc = 0;
  ull units = 0;
  for (;;) {
    const ull v1 = next_center(a, &center_sh);
    if (v1 >= a.n) break;
    const ull o1 = a.off[v1];
    const uint32_t d1 = static_cast<uint32_t>(a.off[v1 + 1] - o1);
    if (d1 == 0 || !owns_center(a, v1)) continue;
    dense_scatter(a, cnt, o1, d1, false);
    __syncthreads();
    for (uint32_t bb = wib; bb < d1; bb += nw) {
      if (lane == 0) ++units;
      const uint32_t v0 = a.adj[o1 + bb];
      const ull e = a.t.rev[o1 + bb];
      const ull oo = a.off[v0];
      const uint32_t d0 = static_cast<uint32_t>(a.off[v0 + 1] - oo);
      const uint32_t p1 = static_cast<uint32_t>(e - oo);
      const uint32_t* P = a.t.tent + a.t.toff[e];
      const uint32_t np = a.t.tri[e];
      if (np == 0) continue;
      const uint32_t i0 = lb32(a.adj + oo, d0, v0);
      if (lane == 0) nt_sh[wib] = 0;
      for (uint32_t j = lane; j < np; j += 32) atomicOr(&w.bm[P[j] >> 5], 1u << (P[j] & 31));
      __syncwarp();
      ull T1 = 0;
      flat_entries(
          a, oo, P, np,
          [&](uint32_t j, ull f2, uint32_t t02, ull to2) -> uint32_t {
            if (P[j] >= i0) return 0u;  // v2 < v0 only
            const ull C = a.t.k4[to2 + lb32(a.t.tent + to2, t02, p1)];  // |T(v0,v2) & P|
            const uint32_t tri12 = a.t.tri[o1 + lb32(a.adj + o1, d1, a.adj[f2])];
            T1 += (t02 - C - 1) * (static_cast<ull>(d1) - np - tri12 + C);
            return 1u;
          },
          [&](int, uint32_t, uint32_t x, ull, uint32_t bounded) {
            if (!bit(w.bm, x) && x != p1) {
              if (atomicAdd(&w.t0[x], 1u) == 0u) w.touched[atomicAdd(&nt_sh[wib], 1u)] = x;
              if (bounded) atomicAdd(&w.t1[x], 1u);
            }
          },
          [](uint32_t, int) {});
      T1 = warp_sum(T1);
      __syncwarp();
      const uint32_t nt = nt_sh[wib];
      ull T2 = 0, T3 = 0;
      for (uint32_t z = lane; z < nt; z += 32) {
        const uint32_t x = w.touched[z];
        w.touched[z] = 0u;
        const ull A = w.t0[x], B = w.t1[x];
        w.t0[x] = 0u;
        w.t1[x] = 0u;
        T2 += B * cnt[a.adj[oo + x]];
        T3 += B * A;
      }
      __syncwarp();
      for (uint32_t j = lane; j < np; j += 32) w.bm[P[j] >> 5] = 0u;
      T2 = warp_sum(T2);
      T3 = warp_sum(T3);
      __syncwarp();
      if (lane == 0) acc += static_cast<i128>(T1) - static_cast<i128>(T2) + static_cast<i128>(T3);  // T1 summed above
    }
    __syncthreads();
    dense_scatter(a, cnt, o1, d1, true);
  }
  store_partial(a, acc, units);
}

// Ego-network pass, full mode, one warp per slot (t, a) of this shard:
//   house: sum_{x not in N_L[a]} cl(x) (cl(x) - 1)
//   tdb:   sum_{x not in N_L[a]} cl(x) cl2(x), cl2 from y in N_L(a) with y > t
template <int KIND>
__global__ void __launch_bounds__(kFastThreads) ego_full_kernel(const FastArgs a) {
  __shared__ uint32_t nt_sh[kFastThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const WarpScratch w = warp_scratch(a);
  i128 acc = 0;
  uint64_t e0;
  while (grab_chunk(a, lane, e0)) {
    const uint64_t me = e0 + lane;
    unsigned todo = __ballot_sync(kAll, me < a.e_hi && a.t.tri[me < a.e_hi ? me : 0] > 0);
    while (todo) {
      const int jl = __ffs(todo) - 1;
      todo &= todo - 1;
      const ull e = e0 + jl;
      const uint32_t t = a.src[e];
      const ull to = a.off[t];
      const uint32_t pa = static_cast<uint32_t>(e - to);
      const uint32_t* Ta = a.t.tent + a.t.toff[e];
      const uint32_t na = a.t.tri[e];
      const uint32_t it = KIND == kFastTailedDiamondB
                              ? lb32(a.adj + to, static_cast<uint32_t>(a.off[t + 1] - to), t) : 0u;
      if (lane == 0) nt_sh[wib] = 0;
      for (uint32_t j = lane; j < na; j += 32) atomicOr(&w.bm[Ta[j] >> 5], 1u << (Ta[j] & 31));
      __syncwarp();
      flat_entries(
          a, to, Ta, na,
          [&](uint32_t j, ull, uint32_t, ull) -> uint32_t {
            return (KIND == kFastTailedDiamondB && Ta[j] >= it) ? 1u : 0u;  // y > t
          },
          [&](int, uint32_t, uint32_t x, ull, uint32_t up) {
            if (atomicAdd(&w.t0[x], 1u) == 0u) w.touched[atomicAdd(&nt_sh[wib], 1u)] = x;
            if (up) atomicAdd(&w.t1[x], 1u);
          },
          [](uint32_t, int) {});
      __syncwarp();
      const uint32_t nt = nt_sh[wib];
      ull s = 0;
      for (uint32_t z = lane; z < nt; z += 32) {
        const uint32_t x = w.touched[z];
        w.touched[z] = 0u;
        const ull c = w.t0[x];
        w.t0[x] = 0u;
        ull c2 = 0;
        if (KIND == kFastTailedDiamondB) {
          c2 = w.t1[x];
          w.t1[x] = 0u;
        }
        if (!bit(w.bm, x) && x != pa) s += KIND == kFastHouse ? c * (c - 1) : c * c2;
      }
      __syncwarp();
      for (uint32_t j = lane; j < na; j += 32) w.bm[Ta[j] >> 5] = 0u;
      acc += static_cast<i128>(s);
      __syncwarp();
    }
  }
  store_partial(a, acc, 0);
}

// Tailed diamond (a), full mode: the per-unit terms except S6, one warp per
// unit, the (v2, x) pairs flattened over the lanes (flat_entries).
__global__ void __launch_bounds__(kFastThreads) tda_full_kernel(const FastArgs a) {
  __shared__ uint32_t ntouched[kFastThreads / 32];
  __shared__ uint32_t cnt_a[kFastThreads / 32][32], cnt_c[kFastThreads / 32][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const WarpScratch w = warp_scratch(a);
  cnt_a[wib][lane] = 0;
  cnt_c[wib][lane] = 0;
  ull cnt = 0, units = 0;
  bool ovf = false;
  uint64_t e0;
  while (grab_chunk(a, lane, e0)) {
    bool mine;
    const uint64_t e = unit_slot(a, e0 + lane, mine);
    units += __popc(__ballot_sync(kAll, mine));
    unsigned todo = __ballot_sync(kAll, mine && a.t.tri[mine ? e : 0] > 0);
    while (todo) {
      const int jl = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t ue = __shfl_sync(kAll, static_cast<ull>(e), jl);
      const uint32_t c = a.src[ue];
      const ull c0 = a.off[c];
      const uint32_t d1 = static_cast<uint32_t>(a.off[c + 1] - c0);
      const uint32_t i0 = static_cast<uint32_t>(ue - c0);
      const uint32_t* P = a.t.tent + a.t.toff[ue];
      const uint32_t np = a.t.tri[ue];
      if (lane == 0) ntouched[wib] = 0;
      for (uint32_t j = lane; j < np; j += 32) atomicOr(&w.bm[P[j] >> 5], 1u << (P[j] & 31));
      __syncwarp();
      ull S2 = 0, S5 = 0;
      flat_entries(
          a, c0, P, np,
          [&](uint32_t, ull, uint32_t t2, ull to2) -> uint32_t { return lb32(a.t.tent + to2, t2, i0); },
          [&](int k, uint32_t r, uint32_t x, ull eidx, uint32_t lb) {
            if (bit(w.bm, x)) {
              atomicAdd(&cnt_c[wib][k], 1u);
            } else if (r < lb) {
              atomicAdd(&cnt_a[wib][k], 1u);
              if (atomicAdd(&w.t0[x], 1u) == 0u) w.touched[atomicAdd(&ntouched[wib], 1u)] = x;
              S5 += a.t.k4[eidx];
            }
          },
          [&](uint32_t j, int k) {
            const uint32_t t2 = a.t.tri[c0 + P[j]];
            S2 += static_cast<ull>(cnt_a[wib][k]) * (t2 - cnt_c[wib][k]);
            cnt_a[wib][k] = 0;
            cnt_c[wib][k] = 0;
          });
      __syncwarp();
      const uint32_t nt = ntouched[wib];
      ull pairs = 0, S3 = 0, S4 = 0;
      for (uint32_t z = lane; z < nt; z += 32) {
        const uint32_t x = w.touched[z];
        w.touched[z] = 0u;
        const ull al = w.t0[x];
        w.t0[x] = 0u;
        pairs += al;
        S3 += static_cast<ull>(a.t.tri[c0 + x]) * al;
        S4 += al * al;
      }
      for (uint32_t j = lane; j < np; j += 32) w.bm[P[j] >> 5] = 0u;
      pairs = warp_sum(pairs);
      S2 = warp_sum(S2);
      S3 = warp_sum(S3);
      S4 = warp_sum(S4);
      S5 = warp_sum(S5);
      __syncwarp();
      if (lane == jl) checked_add(cnt, static_cast<ull>(d1 - np) * pairs - S2 - S3 + S4 + S5, ovf);  // + S6 >= 0
    }
  }
  flush(a, cnt, units, ovf, lane);
}

__global__ void k4_pairs_kernel(const uint32_t* __restrict__ k4, uint64_t entries, ull* out) {
  ull s = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < entries;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const ull k = k4[i];
    s += k * (k - (k ? 1 : 0));
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

int cuda_fail(cudaError_t e, const char* what, std::string* err) {
  if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
  return 1;
}

}  // namespace

void tindex_free(TIndex* t) {
  if (t->rev) cudaFree(t->rev);
  if (t->tri) cudaFree(t->tri);
  if (t->toff) cudaFree(t->toff);
  if (t->tent) cudaFree(t->tent);
  if (t->lowpref) cudaFree(t->lowpref);
  if (t->k4) cudaFree(t->k4);
  *t = TIndex();
}

#define TI_CUDA(call, what)                          \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) {                         \
      cudaFree(tmp);                                 \
      cudaFree(wide);                                \
      cudaFree(nxt);                                 \
      return cuda_fail(e_, what, err);               \
    }                                                \
  } while (0)

int tindex_build(TIndex* t, const ull* off, const uint32_t* adj, const uint32_t* src, uint64_t n, uint64_t slots,
                 int num_sms, cudaStream_t st, bool want_low, bool want_k4, std::string* err) {
  (void)n;
  void* tmp = nullptr;
  ull* wide = nullptr;
  ull* nxt = nullptr;
  const unsigned grid = static_cast<unsigned>(num_sms) * 8;
  const uint64_t s1 = std::max<uint64_t>(slots, 1);
  TI_CUDA(cudaMalloc(&nxt, sizeof(ull)), "tindex cursor");
  if (!t->tent) {
    t->slots = slots;
    TI_CUDA(cudaMalloc(&t->rev, s1 * sizeof(ull)), "tindex rev");
    TI_CUDA(cudaMalloc(&t->tri, s1 * sizeof(uint32_t)), "tindex tri");
    TI_CUDA(cudaMalloc(&t->toff, (slots + 1) * sizeof(ull)), "tindex offsets");
    TI_CUDA(cudaMalloc(&wide, (slots + 1) * sizeof(ull)), "tindex scan buffer");
    if (slots) {
      rev_kernel<<<grid, 256, 0, st>>>(off, adj, src, slots, t->rev);
      TI_CUDA(cudaGetLastError(), "rev_kernel");
      TI_CUDA(cudaMemsetAsync(nxt, 0, sizeof(ull), st), "memset");
      tri_kernel<false><<<grid, 256, 0, st>>>(off, adj, src, slots, t->tri, nullptr, nullptr, nullptr, nxt);
      TI_CUDA(cudaGetLastError(), "tri count");
      mirror_tri_kernel<<<grid, 256, 0, st>>>(src, adj, t->rev, slots, t->tri, wide);
      TI_CUDA(cudaGetLastError(), "tri mirror");
    }
    TI_CUDA(cudaMemsetAsync(wide + slots, 0, sizeof(ull), st), "memset");
    size_t tb = 0;
    TI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, wide, t->toff, slots + 1, st), "scan size");
    TI_CUDA(cudaMalloc(&tmp, std::max<size_t>(tb, 4)), "scan temp");
    TI_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, wide, t->toff, slots + 1, st), "scan");
    ull entries = 0;
    TI_CUDA(cudaMemcpyAsync(&entries, t->toff + slots, sizeof(ull), cudaMemcpyDeviceToHost, st), "D2H");
    TI_CUDA(cudaStreamSynchronize(st), "tindex count");
    t->entries = entries;
    TI_CUDA(cudaMalloc(&t->tent, std::max<ull>(entries, 1) * sizeof(uint32_t)), "tindex entries");
    if (slots) {
      TI_CUDA(cudaMemsetAsync(nxt, 0, sizeof(ull), st), "memset");
      tri_kernel<true><<<grid, 256, 0, st>>>(off, adj, src, slots, t->tri, t->toff, t->tent, t->rev, nxt);
      TI_CUDA(cudaGetLastError(), "tri write");
    }
    cudaFree(tmp);
    tmp = nullptr;
    cudaFree(wide);
    wide = nullptr;
  }
  if (want_low && !t->has_low) {
    TI_CUDA(cudaMalloc(&wide, (slots + 1) * sizeof(ull)), "lowtri");
    if (!t->lowpref) TI_CUDA(cudaMalloc(&t->lowpref, (slots + 1) * sizeof(ull)), "lowpref");
    if (slots) {
      low_kernel<<<grid, 256, 0, st>>>(off, src, t->tri, t->toff, t->tent, slots, wide);
      TI_CUDA(cudaGetLastError(), "low_kernel");
    }
    TI_CUDA(cudaMemsetAsync(wide + slots, 0, sizeof(ull), st), "memset");
    size_t tb = 0;
    TI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, wide, t->lowpref, slots + 1, st), "scan size");
    TI_CUDA(cudaMalloc(&tmp, std::max<size_t>(tb, 4)), "scan temp");
    TI_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, wide, t->lowpref, slots + 1, st), "scan");
    // lowpref <- per-list prefix: scan[e] - scan[first slot of src e] (wide reused as the scan copy)
    TI_CUDA(cudaMemcpyAsync(wide, t->lowpref, (slots + 1) * sizeof(ull), cudaMemcpyDeviceToDevice, st), "copy");
    if (slots) {
      lowpref_kernel<<<grid, 256, 0, st>>>(off, src, wide, slots, t->lowpref);
      TI_CUDA(cudaGetLastError(), "lowpref_kernel");
    }
    TI_CUDA(cudaStreamSynchronize(st), "lowpref");
    cudaFree(tmp);
    tmp = nullptr;
    cudaFree(wide);
    wide = nullptr;
    t->has_low = true;
  }
  if (want_k4 && !t->has_k4 && std::getenv("SMG_TRACE")) {
    TI_CUDA(cudaStreamSynchronize(st), "tindex");
    std::fprintf(stderr, "[smg trace] triangle lists built; computing k4 per entry\n");
  }
  if (want_k4 && !t->has_k4) {
    if (!t->k4) TI_CUDA(cudaMalloc(&t->k4, std::max<ull>(t->entries, 1) * sizeof(uint32_t)), "k4");
    if (slots) {
      TI_CUDA(cudaMemsetAsync(nxt, 0, sizeof(ull), st), "memset");
      k4_kernel<<<grid, 256, 0, st>>>(off, src, t->tri, t->toff, t->tent, slots, t->k4, nxt);
      TI_CUDA(cudaGetLastError(), "k4_kernel");
    }
    TI_CUDA(cudaStreamSynchronize(st), "k4");
    t->has_k4 = true;
  }
  TI_CUDA(cudaStreamSynchronize(st), "tindex");
  cudaFree(nxt);
  return 0;
}

int fast_kind(const smg_plan& p) {
  auto is = [&](int depth, const uint8_t* is_, const uint8_t* df, const int8_t* par) {
    if (p.depth != depth) return false;
    for (int i = 0; i < depth; ++i)
      if (p.isect_mask[i] != is_[i] || p.diff_mask[i] != df[i] || p.parent[i] != par[i]) return false;
    return true;
  };
  // motif_counts' star4 plan (canonical [1,0,2,3])
  static const uint8_t s_is[] = {0, 1, 2, 2}, s_df[] = {0, 0, 1, 5};
  static const int8_t s_par[] = {-1, -1, 0, 2};
  if (is(4, s_is, s_df, s_par)) return kFastStar4;
  // tailed diamond (a): L1 ([0]) L2 ([0,1]) L3 ([1,2]-[0], <v0) L4 ([1]-[0,2,3])
  static const uint8_t a_is[] = {0, 1, 3, 6, 2}, a_df[] = {0, 0, 0, 1, 13};
  static const int8_t a_par[] = {-1, -1, -1, 0, -1};
  if (is(5, a_is, a_df, a_par)) return kFastTailedDiamondA;
  // house (named pattern): L1 ([0],<v0) L2 ([0,1]) L3 ([1]-[0,2]) L4 ([0,3]-[1,2])
  static const uint8_t h_is[] = {0, 1, 3, 2, 9}, h_df[] = {0, 0, 0, 5, 6};
  static const int8_t h_par[] = {-1, 0, -1, -1, -1};
  if (is(5, h_is, h_df, h_par)) return kFastHouse;
  // tailed diamond (b): L1 ([0]) L2 ([0,1],<v0) L3 ([0,2]-[1]) L4 ([1]-[0,2,3])
  static const uint8_t b_is[] = {0, 1, 3, 5, 2}, b_df[] = {0, 0, 0, 2, 13};
  static const int8_t b_par[] = {-1, -1, 0, -1, -1};
  if (is(5, b_is, b_df, b_par)) return kFastTailedDiamondB;
  // motif_counts' tailed triangle, diamond and path4 plans
  static const uint8_t t_is[] = {0, 1, 3, 2}, t_df[] = {0, 0, 0, 5};
  static const int8_t t_par[] = {-1, -1, 0, -1};
  if (is(4, t_is, t_df, t_par)) return kFastTailedTriangle;
  static const uint8_t d_is[] = {0, 1, 3, 5}, d_df[] = {0, 0, 0, 2};
  static const int8_t d_par[] = {-1, -1, 0, 1};
  if (is(4, d_is, d_df, d_par)) return kFastDiamond;
  static const uint8_t p_is[] = {0, 1, 2, 1}, p_df[] = {0, 0, 1, 6};
  static const int8_t p_par[] = {-1, 0, -1, -1};
  if (is(4, p_is, p_df, p_par)) return kFastPath4;
  // rectangle: named (L2 ([0]-[1], <v1) L3 ([1,2]-[0], <v0)) and motif_counts' plan
  static const uint8_t r_is[] = {0, 1, 1, 6}, r_df[] = {0, 0, 2, 1};
  static const int8_t r_par[] = {-1, 0, 1, 0};
  if (is(4, r_is, r_df, r_par)) return kFastRectangle;
  static const uint8_t m_is[] = {0, 1, 2, 5}, m_df[] = {0, 0, 1, 2};
  static const int8_t m_par[] = {-1, 0, 0, 1};
  if (is(4, m_is, m_df, m_par)) return kFastRectangleMotif;
  return kFastNone;
}

uint64_t fast_scratch_words(int kind, uint64_t dmax) {
  if (kind == kFastTailedDiamondA) return 3 * dmax + (dmax + 31) / 32 + 32;  // WarpScratch layout
  if (kind == kFastHouse || kind == kFastTailedDiamondB || kind == kFastPath4) return 3 * dmax + (dmax + 31) / 32 + 32;
  if (kind == kFastRectangle || kind == kFastRectangleMotif) return (dmax + 31) / 32 + 32;  // per CTA (see fast_launch)
  return 0;
}

int fast_slot_arrays(int kind) {
  if (kind == kFastHouse) return 3;
  if (kind == kFastPath4 || kind == kFastRectangle || kind == kFastRectangleMotif) return 1;
  if (kind == kFastTailedDiamondB) return 2;
  return 0;
}

bool fast_dense(int kind) {
  return kind == kFastHouse || kind == kFastTailedDiamondB || kind == kFastPath4 || kind == kFastRectangle ||
         kind == kFastRectangleMotif;
}

// ------------------------------- 4-vertex plans, label-free full counts ---
// Every 4-vertex plan fast_kind() recognises counts each induced instance of
// its pattern exactly once (its restrictions leave one automorphic embedding),
// so the full count does not depend on the vertex labels and equals an integer
// combination of subgraph (non-induced) counts of the whole graph:
//     K4    = 4-cliques (generic executor, clique-local path)
//     D     = sum_{edges e} C(t_e, 2)            diamonds,   t_e = |N(u) & N(v)|
//     C4    = sum_c sum_{x > c} C(w_c(x), 2)     4-cycles,   w_c(x) = #{u in N(c) & N(x) : u > c}
//     PAW   = sum_v t_v (d_v - 2)                tailed triangles, t_v = triangles at v
//     P4    = sum_{(u,v) in E} (d_u - 1)(d_v - 1) - 3 T   3-edge paths, T = triangles
//     S     = sum_v C(d_v, 3)                    3-stars
//   induced diamond  = D - 6 K4
//   induced 4-cycle  = C4 - D + 3 K4
//   induced paw      = PAW - 4 D + 12 K4
//   induced path4    = P4 - 2 PAW + 6 D - 4 C4 - 12 K4
//   induced star4    = S - PAW + 2 D - 4 K4
// (a subgraph copy of X inside an induced Y, counted per Y: paw has 1 star and 2
// paths; C4 4 paths; diamond 2 stars, 4 paws, 1 C4, 6 paths; K4 4 stars, 12
// paws, 3 C4, 6 diamonds, 12 paths.)  The sums run on the degree-ordered copy
// of the CSR (orient_reindex: id 0 = highest degree; engine.cu keeps one per
// replica): the C4 pass walks only wedges c - u - x with u, x > c, sum_u d(u)
// d-(u) elements (d- = neighbours of higher degree) instead of sum_u d(u)^2.
// The kernels store the raw sums per CTA as 128 bits in regions of a.part
// (kM4* below); the host applies the weights of the kind (m4_weights).
__device__ __forceinline__ bool owns_vertex(const FastArgs& a, uint32_t v) {
  return a.num_shards <= 1 || v % a.num_shards == a.shard;
}

// C4: one CTA per centre c, dense per-CTA table w_c (n words, kept zero between
// centres).  Each touch adds atomicAdd's return value: the k-th increment of a
// word returns k - 1, and 0 + 1 + ... + (w - 1) = C(w, 2).
// One list of the scatter: x in N(u), x > c (c itself is in N(u): the suffix
// starts right after it).  Four touches in flight per lane.
constexpr int kC4Threads = 1024;
constexpr int kM4EdgeThreads = 512;

template <bool RESET>
__device__ __forceinline__ ull c4_list(const FastArgs& a, uint32_t* cnt, uint32_t c, uint32_t u, int lane) {
  const ull uo = a.off[u];
  const uint32_t du = static_cast<uint32_t>(a.off[u + 1] - uo);
  const uint32_t x0 = lb32(a.adj + uo, du, c + 1u);
  const uint32_t* X = a.adj + uo;
  ull s = 0;
  uint32_t k = x0 + lane;
  for (; k + 96 < du; k += 128) {
    const uint32_t xa = X[k], xb = X[k + 32], xc = X[k + 64], xd = X[k + 96];
    if (RESET) {
      cnt[xa] = 0u;
      cnt[xb] = 0u;
      cnt[xc] = 0u;
      cnt[xd] = 0u;
    } else {
      const uint32_t ra = atomicAdd(&cnt[xa], 1u), rb = atomicAdd(&cnt[xb], 1u);
      const uint32_t rc = atomicAdd(&cnt[xc], 1u), rd = atomicAdd(&cnt[xd], 1u);
      s += static_cast<ull>(ra) + rb + rc + rd;
    }
  }
  for (; k < du; k += 32) {
    if (RESET) cnt[X[k]] = 0u;
    else s += atomicAdd(&cnt[X[k]], 1u);
  }
  return s;
}

// kC4Threads per CTA (the tables allow two CTAs per SM: 32 warps each fill it).
__global__ void __launch_bounds__(kC4Threads) c4_kernel(const FastArgs a) {
  __shared__ ull center_sh;
  __shared__ i128 red[kC4Threads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* cnt = a.dense + static_cast<uint64_t>(blockIdx.x) * a.n;
  i128 acc = 0;
  for (;;) {
    const ull c = a.group_end + next_center(a, &center_sh);  // smaller ids: the hub and group tiers
    if (c >= a.n) break;
    if (!owns_vertex(a, static_cast<uint32_t>(c))) continue;
    const ull co = a.off[c];
    const uint32_t dc = static_cast<uint32_t>(a.off[c + 1] - co);
    const uint32_t k0 = lb32(a.adj + co, dc, static_cast<uint32_t>(c) + 1u);  // first u > c
    const uint32_t np = dc - k0;
    if (np < 2) continue;
    const uint32_t* U = a.adj + co + k0;
    ull s = 0;
    for (uint32_t j = wib; j < np; j += nw) s += c4_list<false>(a, cnt, static_cast<uint32_t>(c), U[j], lane);
    acc += static_cast<i128>(s);
    __syncthreads();
    for (uint32_t j = wib; j < np; j += nw) c4_list<true>(a, cnt, static_cast<uint32_t>(c), U[j], lane);
  }
  acc = warp_sum128(acc);
  if (lane == 0) red[wib] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = 0;
    for (int w = 0; w < nw; ++w) t += red[w];
    a.part[2 * blockIdx.x] = static_cast<ull>(t);
    a.part[2 * blockIdx.x + 1] = static_cast<ull>(t >> 64);
  }
}

// A hub centre (the first a.hub_count ids of the degree-ordered CSR): the
// whole grid scatters it into table 0, one launch for the scatter (the CTA's
// sum is added to its partial) and one for the reset, so the largest centres
// do not serialise on one CTA at the tail.
template <bool RESET>
__global__ void __launch_bounds__(kFastThreads) c4_hub_kernel(const FastArgs a, uint32_t c) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, tw = (gridDim.x * blockDim.x) >> 5;
  const ull co = a.off[c];
  const uint32_t dc = static_cast<uint32_t>(a.off[c + 1] - co);
  const uint32_t k0 = lb32(a.adj + co, dc, c + 1u);
  const uint32_t np = dc - k0;
  const uint32_t* U = a.adj + co + k0;
  ull s = 0;
  for (uint32_t j = gw; j < np; j += tw) s += c4_list<RESET>(a, a.dense, c, U[j], lane);
  if (RESET) return;
  __shared__ ull red[kFastThreads / 32];
  s = warp_sum(s);
  if (lane == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = static_cast<i128>((static_cast<unsigned __int128>(a.part[2 * blockIdx.x + 1]) << 64) |
                               a.part[2 * blockIdx.x]);
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += static_cast<i128>(red[w]);
    a.part[2 * blockIdx.x] = static_cast<ull>(t);
    a.part[2 * blockIdx.x + 1] = static_cast<ull>(t >> 64);
  }
}

// Group tier of the C4 pass: centres [hub_count, group_end) (degree from
// kM4GroupDegree up to the hub degree) carry ~95% of the table touches.  The
// grid splits into a.groups groups of CTAs; a group owns one table of 16-bit
// counters packed in pairs (n / 2 words; counts stay below the hub degree), so
// the a.groups tables together stay resident in the 126 MB L2 instead of
// streaming 32-byte DRAM sectors per 4-byte touch.  Group g takes centres
// hub_count + g, + groups, ... (degrees descend with the id: round-robin is
// largest-first); its CTAs split the centre's lists and meet at a group
// barrier after the scatter and after the reset.  Cooperative launch: every
// CTA is resident, so the spin barrier cannot starve.
__device__ __forceinline__ void group_barrier(ull* bar, ull& target, unsigned ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += ctas;
    __threadfence();
    atomicAdd(bar, 1ull);
    while (*reinterpret_cast<volatile ull*>(bar) < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

template <bool RESET>
__device__ __forceinline__ ull c4_list16(const FastArgs& a, uint32_t* tab, uint32_t c, uint32_t u, int lane) {
  const ull uo = a.off[u];
  const uint32_t du = static_cast<uint32_t>(a.off[u + 1] - uo);
  const uint32_t x0 = lb32(a.adj + uo, du, c + 1u);
  const uint32_t* X = a.adj + uo;
  ull s = 0;
  uint32_t k = x0 + lane;
  for (; k + 96 < du; k += 128) {
    const uint32_t xa = X[k], xb = X[k + 32], xc = X[k + 64], xd = X[k + 96];
    if (RESET) {
      tab[xa >> 1] = 0u;  // both halves end the reset phase at zero
      tab[xb >> 1] = 0u;
      tab[xc >> 1] = 0u;
      tab[xd >> 1] = 0u;
    } else {
      const uint32_t sa = (xa & 1u) << 4, sb = (xb & 1u) << 4, sc = (xc & 1u) << 4, sd = (xd & 1u) << 4;
      const uint32_t ra = atomicAdd(&tab[xa >> 1], 1u << sa), rb = atomicAdd(&tab[xb >> 1], 1u << sb);
      const uint32_t rc = atomicAdd(&tab[xc >> 1], 1u << sc), rd = atomicAdd(&tab[xd >> 1], 1u << sd);
      s += static_cast<ull>((ra >> sa) & 0xffffu) + ((rb >> sb) & 0xffffu) + ((rc >> sc) & 0xffffu) +
           ((rd >> sd) & 0xffffu);
    }
  }
  for (; k < du; k += 32) {
    const uint32_t x = X[k];
    if (RESET) {
      tab[x >> 1] = 0u;
    } else {
      const uint32_t sh = (x & 1u) << 4;
      s += (atomicAdd(&tab[x >> 1], 1u << sh) >> sh) & 0xffffu;
    }
  }
  return s;
}

__global__ void __launch_bounds__(kC4Threads, 2) c4_group_kernel(const FastArgs a) {
  __shared__ ull red[kC4Threads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned cpg = gridDim.x / a.groups;  // the launch makes gridDim.x = groups x cpg
  const unsigned g = blockIdx.x / cpg, rank = blockIdx.x % cpg;
  const uint64_t words = m4_group_table_words(a.n);  // a multiple of 4: tables stay 16-byte aligned
  uint32_t* tab = a.gtab + static_cast<uint64_t>(g) * words;
  ull* bar = a.gbar + g;
  ull target = 0, s = 0;
  // the shard's centres c = shard (mod num_shards) of the tier, dealt round-robin to the groups
  const uint64_t S = a.num_shards > 1 ? a.num_shards : 1;
  const uint64_t first = a.hub_count + (S + (a.num_shards > 1 ? a.shard : 0) - a.hub_count % S) % S;
  for (uint64_t c64 = first + g * S; c64 < a.group_end; c64 += a.groups * S) {
    const uint32_t c = static_cast<uint32_t>(c64);
    const ull co = a.off[c];
    const uint32_t dc = static_cast<uint32_t>(a.off[c + 1] - co);
    const uint32_t k0 = lb32(a.adj + co, dc, c + 1u);
    const uint32_t np = dc - k0;
    if (np < 2) continue;  // the same decision in every CTA of the group
    const uint32_t* U = a.adj + co + k0;
    for (uint32_t j = rank * nw + wib; j < np; j += cpg * nw) s += c4_list16<false>(a, tab, c, U[j], lane);
    group_barrier(bar, target, cpg);
    if (static_cast<uint64_t>(np) * 512 >= words) {
      // big centre: clearing the whole table (16-byte stores) beats walking the lists again
      uint4* t4 = reinterpret_cast<uint4*>(tab);
      const uint64_t n4 = words / 4;
      for (uint64_t i = static_cast<uint64_t>(rank) * blockDim.x + threadIdx.x; i < n4;
           i += static_cast<uint64_t>(cpg) * blockDim.x)
        t4[i] = make_uint4(0u, 0u, 0u, 0u);
      if (rank == 0)
        for (uint64_t i = n4 * 4 + threadIdx.x; i < words; i += blockDim.x) tab[i] = 0u;
    } else {
      for (uint32_t j = rank * nw + wib; j < np; j += cpg * nw) c4_list16<true>(a, tab, c, U[j], lane);
    }
    group_barrier(bar, target, cpg);
  }
  s = warp_sum(s);
  if (lane == 0) red[wib] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    i128 t = static_cast<i128>((static_cast<unsigned __int128>(a.part[2 * blockIdx.x + 1]) << 64) |
                               a.part[2 * blockIdx.x]);
    for (int w = 0; w < nw; ++w) t += static_cast<i128>(red[w]);
    a.part[2 * blockIdx.x] = static_cast<ull>(t);
    a.part[2 * blockIdx.x + 1] = static_cast<ull>(t >> 64);
  }
}

// Per undirected edge (slot e = (u, v), u < v; the shard that owns u):
// C(t, 2), t and (d_u - 1)(d_v - 1); and tv[x] += t at the owned endpoints
// (tv[x] = 2 t_x once every edge at x is in; only when a.acc0 is given).
__global__ void __launch_bounds__(kM4EdgeThreads, 2) m4_edge_kernel(const FastArgs a) {
  const int lane = threadIdx.x & 31;
  i128 acc_d = 0, acc_t3 = 0, acc_p4 = 0;
  ull units = 0;
  for (;;) {
    ull chunk = 0;
    if (lane == 0) chunk = atomicAdd(a.next_chunk, 1ull);
    chunk = __shfl_sync(kAll, chunk, 0);
    if (chunk * kSlotChunk >= a.slots) break;
    const uint64_t e = chunk * kSlotChunk + lane;
    bool mine = e < a.slots;
    uint32_t u = 0, v = 0;
    bool own_u = false, own_v = false;
    if (mine) {
      u = a.src[e];
      v = a.adj[e];
      own_u = owns_vertex(a, u);
      own_v = a.acc0 != nullptr && owns_vertex(a, v);
      mine = u < v && (own_u || own_v);
    }
    ull bu = 0, bv = 0;
    uint32_t du = 0, dv = 0;
    if (mine) {
      bu = a.off[u];
      du = static_cast<uint32_t>(a.off[u + 1] - bu);
      bv = a.off[v];
      dv = static_cast<uint32_t>(a.off[v + 1] - bv);
    }
    ull t = 0;
    const bool small = mine && min(du, dv) <= 8;
    if (small) t = isect_count(a.adj + bu, du, a.adj + bv, dv);
    unsigned big = __ballot_sync(kAll, mine && !small);
    while (big) {
      const int j = __ffs(big) - 1;
      big &= big - 1;
      const ull jbu = __shfl_sync(kAll, bu, j), jbv = __shfl_sync(kAll, bv, j);
      const uint32_t jdu = __shfl_sync(kAll, du, j), jdv = __shfl_sync(kAll, dv, j);
      const bool su = jdu <= jdv;
      const uint32_t* S = a.adj + (su ? jbu : jbv);
      const uint32_t* L = a.adj + (su ? jbv : jbu);
      const uint32_t ns = su ? jdu : jdv, nl = su ? jdv : jdu;
      ull tj = 0;
      for (uint32_t i = lane; i < ns; i += 32) {
        const uint32_t x = S[i];
        const uint32_t p = lb32(L, nl, x);
        tj += (p < nl && L[p] == x) ? 1u : 0u;
      }
      tj = warp_sum(tj);
      if (lane == j) t = tj;
    }
    if (mine) {
      if (own_u) {
        units += a.units_per_edge;
        acc_d += static_cast<i128>(t * (t - 1) / 2);
        acc_t3 += static_cast<i128>(t);
        acc_p4 += static_cast<i128>(static_cast<ull>(du - 1) * static_cast<ull>(dv - 1));
      }
      if (a.acc0 != nullptr && t) {
        if (own_u) atomicAdd(&a.acc0[u], t);
        if (own_v) atomicAdd(&a.acc0[v], t);
      }
    }
  }
  FastArgs w = a;
  const unsigned B = gridDim.x;
  w.part = a.part + 2 * B * kM4D;
  store_partial(w, acc_d, units);
  w.part = a.part + 2 * B * kM4T3;
  store_partial(w, acc_t3, 0);
  w.part = a.part + 2 * B * kM4P4E;
  store_partial(w, acc_p4, 0);
}

// The same sums from per-slot triangle counts the 4-clique kernels left behind
// (k4.cu, tcount: slot (u, v), v < u, holds t_e): a streaming pass, no
// intersections.  Single shard only (a shard's K4 roots see only part of t_e).
__global__ void __launch_bounds__(kFastThreads) m4_edge_counts_kernel(const FastArgs a) {
  i128 acc_d = 0, acc_t3 = 0, acc_p4 = 0;
  ull units = 0;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < a.slots;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t u = a.src[e], v = a.adj[e];
    if (v >= u) continue;
    const ull t = a.tcount[e];
    const ull du = a.off[u + 1] - a.off[u], dv = a.off[v + 1] - a.off[v];
    units += a.units_per_edge;
    acc_d += static_cast<i128>(t * (t - 1) / 2);
    acc_t3 += static_cast<i128>(t);
    acc_p4 += static_cast<i128>((du - 1) * (dv - 1));
    if (a.acc0 != nullptr && t) {
      atomicAdd(&a.acc0[u], t);
      atomicAdd(&a.acc0[v], t);
    }
  }
  FastArgs w = a;
  const unsigned B = gridDim.x;
  w.part = a.part + 2 * B * kM4D;
  store_partial(w, acc_d, units);
  w.part = a.part + 2 * B * kM4T3;
  store_partial(w, acc_t3, 0);
  w.part = a.part + 2 * B * kM4P4E;
  store_partial(w, acc_p4, 0);
}

// Per owned vertex v: (d_v - 2) t_v and C(d_v, 3), t_v = tv[v] / 2 (0 when
// a.acc0 is not given); tv is zeroed again.
__global__ void __launch_bounds__(kFastThreads) m4_vertex_kernel(const FastArgs a) {
  i128 acc_paw = 0, acc_star = 0;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < a.n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (!owns_vertex(a, static_cast<uint32_t>(v))) continue;
    const ull d = a.off[v + 1] - a.off[v];
    if (d >= 3) acc_star += static_cast<i128>(d * (d - 1) / 2) * static_cast<i128>(d - 2) / 3;
    if (a.acc0 != nullptr) {
      const ull tv = a.acc0[v] / 2;
      a.acc0[v] = 0ull;
      if (tv) acc_paw += static_cast<i128>(tv) * static_cast<i128>(d - 2);
    }
  }
  FastArgs w = a;
  const unsigned B = gridDim.x;
  w.part = a.part + 2 * B * kM4Paw;
  store_partial(w, acc_paw, 0);
  w.part = a.part + 2 * B * kM4Star;
  store_partial(w, acc_star, 0);
}

// need: bit r set = region r (kM4*) is wanted.  a.part: kM4Regions x blocks pairs.
// ev (may be null): 4 events recorded before the C4 pass, after it, after the
// edge pass and after the vertex pass (per-kernel device times).
int m4_launch(const FastArgs& a, unsigned need, unsigned blocks, cudaStream_t st, cudaEvent_t* ev) {
  if (cudaMemsetAsync(a.part, 0, 2 * kM4Regions * blocks * sizeof(ull), st) != cudaSuccess) return 1;
  if (ev) cudaEventRecord(ev[0], st);
  if (need & (1u << kM4C4)) {
    if (cudaMemsetAsync(a.next2, 0, sizeof(ull), st) != cudaSuccess) return 1;
    FastArgs w = a;
    w.part = a.part + 2 * blocks * kM4C4;
    c4_kernel<<<std::max(1u, std::min(blocks, a.c4_blocks)), kC4Threads, 0, st>>>(w);  // stores its partials; the others add
    for (uint32_t c = 0; c < a.hub_count; ++c) {
      if (a.num_shards > 1 && c % a.num_shards != a.shard) continue;
      c4_hub_kernel<false><<<blocks, kFastThreads, 0, st>>>(w, c);
      c4_hub_kernel<true><<<blocks, kFastThreads, 0, st>>>(w, c);
    }
    if (cudaGetLastError() != cudaSuccess) return 1;
    if (a.group_end > a.hub_count) {
      if (cudaMemsetAsync(a.gbar, 0, a.groups * sizeof(ull), st) != cudaSuccess) return 1;
      // every CTA must be resident (spin barriers): size the grid by occupancy
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c4_group_kernel, kC4Threads, 0);
      const unsigned fit = std::min<unsigned>(blocks, static_cast<unsigned>(std::max(1, per_sm) * sms));
      if (fit < a.groups) w.groups = fit;
      const unsigned grid = (fit / w.groups) * w.groups;
      void* params[] = {static_cast<void*>(&w)};
      if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(c4_group_kernel), dim3(grid), dim3(kC4Threads), params,
                                      0, st) != cudaSuccess)
        return 1;
    }
  }
  if (ev) cudaEventRecord(ev[1], st);
  FastArgs w = a;
  if (!(need & (1u << kM4Paw))) w.acc0 = nullptr;  // no per-vertex triangle counts needed
  if (a.tcount != nullptr && a.num_shards <= 1) m4_edge_counts_kernel<<<blocks, kFastThreads, 0, st>>>(w);
  else m4_edge_kernel<<<blocks, kM4EdgeThreads, 0, st>>>(w);
  if (cudaGetLastError() != cudaSuccess) return 1;
  if (ev) cudaEventRecord(ev[2], st);
  if (need & ((1u << kM4Paw) | (1u << kM4Star))) {
    m4_vertex_kernel<<<blocks, kFastThreads, 0, st>>>(w);
    if (cudaGetLastError() != cudaSuccess) return 1;
  }
  if (ev) cudaEventRecord(ev[3], st);
  return 0;
}

bool m4_weights(int kind, M4Weights* w) {
  *w = M4Weights{};
  switch (kind) {
    case kFastRectangle:
    case kFastRectangleMotif: w->w[kM4C4] = 1; w->w[kM4D] = -1; w->k4 = 3; return true;
    case kFastDiamond: w->w[kM4D] = 1; w->k4 = -6; return true;
    case kFastTailedTriangle: w->w[kM4Paw] = 1; w->w[kM4D] = -4; w->k4 = 12; return true;
    case kFastPath4:
      w->w[kM4P4E] = 1; w->w[kM4T3] = -1; w->w[kM4Paw] = -2; w->w[kM4D] = 6; w->w[kM4C4] = -4; w->k4 = -12;
      return true;
    case kFastStar4: w->w[kM4Star] = 1; w->w[kM4Paw] = -1; w->w[kM4D] = 2; w->k4 = -4; return true;
    case kFastClique4: w->k4 = 1; return true;
    default: return false;
  }
}

bool fast_has_full(int kind) {
  return kind == kFastHouse || kind == kFastTailedDiamondA || kind == kFastTailedDiamondB;
}

int fast_launch_full(int kind, const FastArgs& a, unsigned blocks, cudaStream_t st) {
  if (kind == kFastTailedDiamondA) {  // per-unit terms without S6, checked sum into count
    tda_full_kernel<<<blocks, kFastThreads, 0, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
  }
  if (kind != kFastHouse && kind != kFastTailedDiamondB) return 2;
  // centre pass -> part[0 .. blocks), ego pass -> part[blocks .. 2 blocks)
  if (cudaMemsetAsync(a.part, 0, 4 * blocks * sizeof(ull), st) != cudaSuccess) return 1;
  if (cudaMemsetAsync(a.next2, 0, sizeof(ull), st) != cudaSuccess) return 1;
  if (kind == kFastHouse) house_full_center_kernel<<<blocks, kFastThreads, 0, st>>>(a);
  else tdb_full_center_kernel<<<blocks, kFastThreads, 0, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return 1;
  FastArgs w = a;
  w.part = a.part + 2 * blocks;
  if (kind == kFastHouse) ego_full_kernel<kFastHouse><<<blocks, kFastThreads, 0, st>>>(w);
  else ego_full_kernel<kFastTailedDiamondB><<<blocks, kFastThreads, 0, st>>>(w);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int tindex_k4_pairs(const TIndex& t, int num_sms, cudaStream_t st, unsigned long long* out, std::string* err) {
  ull* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(ull));
  if (e == cudaSuccess) e = cudaMemsetAsync(d, 0, sizeof(ull), st);
  if (e == cudaSuccess && t.entries) {
    k4_pairs_kernel<<<num_sms * 8, 256, 0, st>>>(t.k4, t.entries, d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, sizeof(ull), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d);
  return e == cudaSuccess ? 0 : cuda_fail(e, "k4 pairs", err);
}

bool fast_center_v1(int kind) {
  return kind == kFastStar4 || kind == kFastTailedDiamondA || kind == kFastTailedTriangle;
}

int fast_launch(int kind, const FastArgs& a, unsigned blocks, cudaStream_t st, bool combine_only) {
  if (kind == kFastStar4) {
    star4_kernel<<<blocks, kFastThreads, 0, st>>>(a);
  } else if (kind == kFastTailedDiamondA) {
    tda_kernel<false><<<blocks, kFastThreads, 0, st>>>(a);
  } else if (kind == kFastTailedTriangle) {
    star_kernel<kFastTailedTriangle><<<blocks, kFastThreads, 0, st>>>(a);
  } else if (kind == kFastDiamond) {
    star_kernel<kFastDiamond><<<blocks, kFastThreads, 0, st>>>(a);
  } else if (kind == kFastRectangle || kind == kFastRectangleMotif) {
    const bool array = a.acc0 != nullptr;  // root-range call: per-unit values, cached, then combined
    if (!(array && combine_only)) {
      if (cudaMemsetAsync(a.next2, 0, sizeof(ull), st) != cudaSuccess) return 1;
      if (kind == kFastRectangle) {
        if (array) rect_kernel<true, true><<<blocks, kFastThreads, 0, st>>>(a);
        else rect_kernel<true, false><<<blocks, kFastThreads, 0, st>>>(a);
      } else {
        if (array) rect_kernel<false, true><<<blocks, kFastThreads, 0, st>>>(a);
        else rect_kernel<false, false><<<blocks, kFastThreads, 0, st>>>(a);
      }
      if (cudaGetLastError() != cudaSuccess) return 1;
    }
    if (array) {
      if (kind == kFastRectangle) combine_kernel<kFastRectangle><<<blocks, kFastThreads, 0, st>>>(a);
      else combine_kernel<kFastRectangleMotif><<<blocks, kFastThreads, 0, st>>>(a);
    }
  } else if (kind == kFastPath4) {
    if (!combine_only) {
      if (cudaMemsetAsync(a.next2, 0, sizeof(ull), st) != cudaSuccess) return 1;
      house_eh_kernel<true><<<blocks, kFastThreads, 0, st>>>(a);
      if (cudaGetLastError() != cudaSuccess) return 1;
    }
    combine_kernel<kFastPath4><<<blocks, kFastThreads, 0, st>>>(a);
  } else if (kind == kFastHouse || kind == kFastTailedDiamondB) {
    // (1) center-table pass, (2) ego-network pass, (3) combine; the queue
    // cursors are reset between passes on the stream
    if (combine_only) {
      if (kind == kFastHouse) combine_kernel<kFastHouse><<<blocks, kFastThreads, 0, st>>>(a);
      else combine_kernel<kFastTailedDiamondB><<<blocks, kFastThreads, 0, st>>>(a);
      return cudaGetLastError() == cudaSuccess ? 0 : 1;
    }
    if (cudaMemsetAsync(a.next2, 0, sizeof(ull), st) != cudaSuccess) return 1;
    if (cudaMemsetAsync(a.acc2, 0, a.slots * sizeof(ull), st) != cudaSuccess) return 1;
    if (kind == kFastHouse) house_eh_kernel<false><<<blocks, kFastThreads, 0, st>>>(a);
    else tdb_unit_kernel<<<blocks, kFastThreads, 0, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) return 1;
    FastArgs w = a;  // the ego pass walks every slot (no shard map, no root filter)
    w.num_shards = 1;
    w.e_lo = 0;
    w.e_hi = a.slots;
    w.via_rev = 0;
    w.next_chunk = a.next2;
    if (cudaMemsetAsync(a.next2, 0, sizeof(ull), st) != cudaSuccess) return 1;
    if (kind == kFastHouse) ego_w_kernel<kFastHouse><<<blocks, kFastThreads, 0, st>>>(w);
    else ego_w_kernel<kFastTailedDiamondB><<<blocks, kFastThreads, 0, st>>>(w);
    if (cudaGetLastError() != cudaSuccess) return 1;
    if (kind == kFastHouse) combine_kernel<kFastHouse><<<blocks, kFastThreads, 0, st>>>(a);
    else combine_kernel<kFastTailedDiamondB><<<blocks, kFastThreads, 0, st>>>(a);
  } else {
    return 2;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace smg

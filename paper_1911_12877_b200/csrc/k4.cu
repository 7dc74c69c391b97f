// k4.cu -- 4-cliques of a degree-ordered CSR on B200 (sm_100a).
//
// The closed forms of the 4-vertex plans (tindex.cu, m4_launch) and the
// 4-clique plan itself need K4, the number of 4-cliques of the whole graph.  A
// 4-clique plan counts it through the reference's nested merges
// (Executor::count_from, proj/src/engine.cpp:89-115: v0 > v1 > v2 > v3); the
// total does not depend on the vertex labels, so on the orient_reindex copy
// (graph.cpp:137-161: ids by descending degree) it is counted per root instead
// of per level-1 unit:
//
//   K4 = sum_d T(G[L_d]),  L_d = N-(d) = {u in N(d) : u < d}
//
// (every 4-clique at its largest vertex d; T = triangles of the graph induced
// on L_d).  |L_d| is at most ~sqrt(2m) on the ordered copy.  Per root the
// local adjacency is built once as bitmap rows over positions in L_d --
// row(i) = {j < i : L[j] ~ L[i]} -- and every local edge (i, j) contributes
// popc(row(i) & row(j)): the common neighbours below j.  The generic executor
// rebuilds the rows of U = N(v0) & N(v1) for every unit (v0, v1); here a root's
// rows serve all its units.
//
//  * k4_warp_kernel: roots with 3 <= |L| <= 32, one warp per root, one row per
//    lane (a register), adjacency by binary search of L[j] in N-(L[lane]).
//  * k4_cta_kernel: roots with |L| > 32, one CTA per root from a dynamic queue,
//    rows in shared memory (|L| <= kSmemL) or in the CTA's slice of a global
//    scratch (L2-resident), built by one warp per row (the shorter of N-(x) and
//    L[0..i) is searched into the other), counted by sub-warp groups that AND
//    the words of row(i) and row(j) for one local edge each.
#include <cstdio>

#include "k4.hpp"

namespace smg {

namespace {

typedef unsigned long long ull;
constexpr unsigned kAll = 0xffffffffu;
constexpr int kThreads = 512;
constexpr uint32_t kMaxL = 12288;   // list capacity of the CTA tier (48 KB of shared memory)
constexpr uint32_t kSmemL = 352;    // rows of lists up to this length live in shared memory (352 x 11 words)
constexpr uint32_t kSmemRowWords = 352 * 11;  // with the list and degrees: 112 KB per CTA, two CTAs per SM
// ctr layout
enum { kNextWarp = 0, kNextCta = 1, kCount = 2, kFlags = 3, kLmax = 4, kUnits = 5, kCtrWords = 8 };
constexpr uint32_t kRootsPerStep = 16;  // roots a CTA takes per queue step

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

__device__ __forceinline__ ull warp_sum(ull v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(kAll, v, d);
  return v;
}

__device__ __forceinline__ void add_count(ull* ctr, ull v) {
  if (!v) return;
  const ull old = atomicAdd(&ctr[kCount], v);
  if (old + v < old) atomicOr(&ctr[kFlags], 2ull);
}

__device__ __forceinline__ bool owns(uint32_t d, uint32_t shard, uint32_t num_shards) {
  return num_shards <= 1 || d % num_shards == shard;
}

// max_d |N-(d)|
__global__ void lmax_kernel(const ull* __restrict__ off, const uint32_t* __restrict__ adj, uint64_t n, ull* ctr) {
  uint32_t best = 0;
  for (uint64_t d = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; d < n;
       d += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const ull o = off[d];
    best = max(best, lb32(adj + o, static_cast<uint32_t>(off[d + 1] - o), static_cast<uint32_t>(d)));
  }
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) best = max(best, __shfl_xor_sync(kAll, best, s));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(&ctr[kLmax], static_cast<ull>(best));
}

template <int K>
__global__ void __launch_bounds__(kThreads) k4_warp_kernel(const ull* __restrict__ off,
                                                           const uint32_t* __restrict__ adj, uint64_t n,
                                                           uint32_t shard, uint32_t num_shards, ull* ctr,
                                                           uint32_t* __restrict__ tcount) {
  const int lane = threadIdx.x & 31;
  ull total = 0, units = 0;
  for (;;) {
    ull chunk = 0;
    if (lane == 0) chunk = atomicAdd(&ctr[kNextWarp], 1ull);
    chunk = __shfl_sync(kAll, chunk, 0);
    if (chunk * 32 >= n) break;
    const uint64_t mine = chunk * 32 + lane;
    uint32_t len = 0;
    ull base = 0;
    if (mine < n && owns(static_cast<uint32_t>(mine), shard, num_shards)) {
      base = off[mine];
      len = lb32(adj + base, static_cast<uint32_t>(off[mine + 1] - base), static_cast<uint32_t>(mine));
    }
    units += len;  // level-1 units (v1 < v0) of the owned roots
    // with tcount, lists of 2 matter too: their one possible local edge is a triangle
    unsigned todo = __ballot_sync(kAll, len >= (tcount ? 2u : static_cast<uint32_t>(K - 1)) && len <= 32);
    while (todo) {
      const int r = __ffs(todo) - 1;
      todo &= todo - 1;
      const ull rb = __shfl_sync(kAll, base, r);
      const uint32_t l = __shfl_sync(kAll, len, r);
      // lane i holds x = L[i] and searches the smaller L[j] in N-(x)
      uint32_t x = 0, xn = 0;
      const uint32_t* X = adj;
      if (lane < static_cast<int>(l)) {
        x = adj[rb + lane];
        const ull xo = off[x];
        X = adj + xo;
        xn = lb32(X, static_cast<uint32_t>(off[x + 1] - xo), x);
      }
      uint32_t row = 0;
      for (uint32_t j = 0; j + 1 < l; ++j) {
        const uint32_t u = __shfl_sync(kAll, x, j);
        if (lane > static_cast<int>(j) && lane < static_cast<int>(l) && xn) {
          const uint32_t p = lb32(X, xn, u);
          if (p < xn && X[p] == u) {
            row |= 1u << j;
            if (tcount) atomicAdd(&tcount[(X - adj) + p], 1u);  // triangle {u, x, root}: edge (x, u)
          }
        }
      }
      if (tcount) {
        // edges (root, L[lane]): the local degree of lane = its row plus the rows that name it
        uint32_t deg = __popc(row);
        for (uint32_t j = 1; j < l; ++j) {
          const uint32_t rj = __shfl_sync(kAll, row, j);
          if (lane < static_cast<int>(j)) deg += (rj >> lane) & 1u;
        }
        if (lane < static_cast<int>(l) && deg) atomicAdd(&tcount[rb + lane], deg);
      }
      uint32_t cnt = 0;
      for (uint32_t j = 0; j + 1 < l; ++j) {
        const uint32_t rj = __shfl_sync(kAll, row, j);
        const uint32_t mij = ((row >> j) & 1u) ? (row & rj) : 0u;  // common local neighbours below j
        if (K == 4) {
          cnt += __popc(mij);
        } else {  // K == 5: triangles (i, j, k) and their common neighbours below k
          for (uint32_t k = 0; k < j; ++k) {
            const uint32_t rk = __shfl_sync(kAll, row, k);
            if ((mij >> k) & 1u) cnt += __popc(mij & rk);
          }
        }
      }
      total += cnt;
    }
  }
  total = warp_sum(total);
  units = warp_sum(units);
  if (lane == 0) {
    add_count(ctr, total);
    if (units) atomicAdd(&ctr[kUnits], units);
  }
}

struct CtaShared {
  uint32_t L[kMaxL];
  uint32_t deg[kMaxL];  // local degrees (only with tcount)
  ull root;
};

template <int K>
__global__ void __launch_bounds__(kThreads) k4_cta_kernel(const ull* __restrict__ off,
                                                          const uint32_t* __restrict__ adj, uint64_t n,
                                                          uint32_t shard, uint32_t num_shards, ull* ctr,
                                                          uint32_t* __restrict__ scratch, uint64_t scratch_words,
                                                          uint32_t* __restrict__ tcount) {
  extern __shared__ uint32_t dyn[];
  CtaShared& sh = *reinterpret_cast<CtaShared*>(dyn);
  uint32_t* srows = dyn + (sizeof(CtaShared) + 3) / 4;
  uint32_t* grows = scratch + static_cast<uint64_t>(blockIdx.x) * scratch_words;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  ull total = 0;
  for (;;) {
    // next roots (kRootsPerStep per queue step); only lists longer than a warp's are taken here
    __syncthreads();
    if (threadIdx.x == 0) sh.root = atomicAdd(&ctr[kNextCta], 1ull);
    __syncthreads();
    const ull chunk = sh.root;
    if (chunk * kRootsPerStep >= n) break;
    for (uint32_t r = 0; r < kRootsPerStep; ++r) {
      const uint64_t d = chunk * kRootsPerStep + r;
      if (d >= n) break;
      if (!owns(static_cast<uint32_t>(d), shard, num_shards)) continue;
      const ull base = off[d];
      const uint32_t l = lb32(adj + base, static_cast<uint32_t>(off[d + 1] - base), static_cast<uint32_t>(d));
      if (l <= 32) continue;  // uniform across the CTA
      if (l > kMaxL) {
        if (threadIdx.x == 0) atomicOr(&ctr[kFlags], 1ull);
        continue;
      }
      const uint32_t stride = ((l + 31) >> 5) | 1u;  // odd: rows start in different banks
      uint32_t* rows = (l <= kSmemL) ? srows : grows;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < l; i += blockDim.x) {
        sh.L[i] = adj[base + i];
        sh.deg[i] = 0u;
      }
      for (uint64_t i = threadIdx.x; i < static_cast<uint64_t>(l) * stride; i += blockDim.x) rows[i] = 0u;
      __syncthreads();
      // rows: row(i) = {j < i : L[j] in N-(L[i])}
      for (uint32_t i = 1 + wib; i < l; i += nw) {
        const uint32_t x = sh.L[i];
        const ull xo = off[x];
        const uint32_t* X = adj + xo;
        const uint32_t xn = lb32(X, static_cast<uint32_t>(off[x + 1] - xo), x);
        uint32_t* row = rows + static_cast<uint64_t>(i) * stride;
        if (xn <= 4 * i) {
          // walk N-(x) (coalesced), find each element among L[0..i)
          const uint32_t lo = lb32(X, xn, sh.L[0]);
          for (uint32_t k = lo + lane; k < xn; k += 32) {
            const uint32_t u = X[k];
            const uint32_t p = lb32(sh.L, i, u);
            if (p < i && sh.L[p] == u) {
              atomicOr(&row[p >> 5], 1u << (p & 31));
              if (tcount) {  // triangle {u, x, root}: edge (x, u) here, edges (root, x), (root, u) below
                atomicAdd(&tcount[xo + k], 1u);
                atomicAdd(&sh.deg[p], 1u);
                atomicAdd(&sh.deg[i], 1u);
              }
            }
          }
        } else {
          // walk L[0..i), find each element in N-(x)
          for (uint32_t j0 = 0; j0 < i; j0 += 32) {
            const uint32_t j = j0 + lane;
            bool hit = false;
            if (j < i) {
              const uint32_t u = sh.L[j];
              const uint32_t p = lb32(X, xn, u);
              hit = p < xn && X[p] == u;
              if (hit && tcount) {
                atomicAdd(&tcount[xo + p], 1u);
                atomicAdd(&sh.deg[j], 1u);
              }
            }
            const unsigned m = __ballot_sync(kAll, hit);
            if (lane == 0 && m) {
              row[j0 >> 5] = m;
              if (tcount) atomicAdd(&sh.deg[i], static_cast<uint32_t>(__popc(m)));
            }
          }
        }
      }
      __syncthreads();
      if (tcount)
        for (uint32_t i = threadIdx.x; i < l; i += blockDim.x)
          if (sh.deg[i]) atomicAdd(&tcount[base + i], sh.deg[i]);
      if (K == 4) {
        // local edges (i, j), j < i: popc(row(i) & row(j)) over the words below j.
        // Sub-warp groups of G lanes take one edge each; G covers the row's words.
        uint32_t G = 1;
        while (G < 32 && G < stride) G <<= 1;
        const uint32_t gid = lane / G, gl = lane % G, ng = 32 / G;
        for (uint32_t i = 2 + wib; i < l; i += nw) {
          const uint32_t* ri = rows + static_cast<uint64_t>(i) * stride;
          const uint32_t wi = (i + 31) >> 5;  // words of row(i) that can be non-zero
          for (uint32_t w = 0; w < wi; ++w) {
            const uint32_t m = ri[w];
            const uint32_t c = __popc(m);
            for (uint32_t k0 = 0; k0 < c; k0 += ng) {
              const uint32_t k = k0 + gid;
              if (k < c) {
                const uint32_t j = (w << 5) + __fns(m, 0, k + 1);
                const uint32_t* rj = rows + static_cast<uint64_t>(j) * stride;
                const uint32_t wj = (j + 31) >> 5;
                uint32_t s = 0;
                for (uint32_t q = gl; q < wj; q += G) s += __popc(ri[q] & rj[q]);
                total += s;
              }
            }
          }
        }
      } else {
        // K == 5: local triangles (i, j, k), k < j < i, each adds
        // popc(row(i) & row(j) & row(k)).  A warp takes row i, compacts its set
        // bits 1,024 at a time into its list (the degree array's space: tcount
        // is never used with K == 5), and every lane walks one local edge (i, j).
        uint16_t* list = reinterpret_cast<uint16_t*>(sh.deg) + wib * 1024;
        for (uint32_t i = 3 + wib; i < l; i += nw) {
          const uint32_t* ri = rows + static_cast<uint64_t>(i) * stride;
          const uint32_t wi = (i + 31) >> 5;
          for (uint32_t w0 = 0; w0 < wi; w0 += 32) {
            const uint32_t wq = w0 + lane;
            uint32_t m = wq < wi ? ri[wq] : 0u;
            uint32_t pos = __popc(m);
            uint32_t incl = pos;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const uint32_t o = __shfl_up_sync(kAll, incl, d);
              if (lane >= d) incl += o;
            }
            const uint32_t cnt = __shfl_sync(kAll, incl, 31);
            pos = incl - pos;
            while (m) {
              const uint32_t b = __ffs(m) - 1;
              m &= m - 1;
              list[pos++] = static_cast<uint16_t>((wq << 5) + b);
            }
            __syncwarp();
            for (uint32_t e = lane; e < cnt; e += 32) {
              const uint32_t j = list[e];
              const uint32_t* rj = rows + static_cast<uint64_t>(j) * stride;
              const uint32_t wj = (j + 31) >> 5;
              ull s = 0;
              for (uint32_t q = 0; q < wj; ++q) {
                uint32_t mm = ri[q] & rj[q];
                while (mm) {
                  const uint32_t k = (q << 5) + (__ffs(mm) - 1);
                  mm &= mm - 1;
                  const uint32_t* rk = rows + static_cast<uint64_t>(k) * stride;
                  const uint32_t wk = (k + 31) >> 5;
                  uint32_t t = 0;
                  for (uint32_t q2 = 0; q2 < wk; ++q2) t += __popc(ri[q2] & rj[q2] & rk[q2]);
                  s += t;
                }
              }
              total += s;
            }
            __syncwarp();
          }
        }
      }
    }
  }
  __shared__ ull red[kThreads / 32];
  total = warp_sum(total);
  if (lane == 0) red[wib] = total;
  __syncthreads();
  if (threadIdx.x == 0) {
    ull t = 0;
    for (int w = 0; w < nw; ++w) t += red[w];
    add_count(ctr, t);
  }
}

int cuda_fail(cudaError_t e, const char* what, std::string* err) {
  if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
  return 1;
}

}  // namespace

void k4_free(K4Work* w) {
  if (w->ctr) cudaFree(w->ctr);
  if (w->host) cudaFreeHost(w->host);
  if (w->rows) cudaFree(w->rows);
  if (w->ev0) cudaEventDestroy(w->ev0);
  if (w->ev1) cudaEventDestroy(w->ev1);
  *w = K4Work();
}

int k4_count(const unsigned long long* off, const uint32_t* adj, uint64_t n, uint32_t shard, uint32_t num_shards,
             int num_sms, cudaStream_t st, K4Work* w, uint32_t* tcount, unsigned long long* count,
             unsigned long long* units, double* ms, std::string* err, int k) {
  cudaError_t e = cudaSuccess;
  if (k != 4 && k != 5) {
    if (err) *err = "clique size must be 4 or 5";
    return 1;
  }
  if (k == 5) tcount = nullptr;
  if (!w->ctr) {
    e = cudaMalloc(&w->ctr, kCtrWords * sizeof(ull));
    if (e == cudaSuccess) e = cudaMallocHost(&w->host, kCtrWords * sizeof(ull));
    if (e == cudaSuccess) e = cudaEventCreate(&w->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&w->ev1);
    if (e != cudaSuccess) return cuda_fail(e, "k4 buffers", err);
  }
  *count = 0;
  *units = 0;
  *ms = 0;
  if (n == 0) return 0;
  const unsigned blocks = static_cast<unsigned>(num_sms) * 2;
  const size_t smem = ((sizeof(CtaShared) + 3) / 4 + kSmemRowWords) * sizeof(uint32_t);
  e = cudaFuncSetAttribute(k4_cta_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k4_cta_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_fail(e, "k4 shared memory", err);
  e = cudaMemsetAsync(w->ctr, 0, kCtrWords * sizeof(ull), st);
  if (e != cudaSuccess) return cuda_fail(e, "k4 memset", err);
  if (!w->lmax) {
    lmax_kernel<<<num_sms * 8, 256, 0, st>>>(off, adj, n, w->ctr);
    e = cudaMemcpyAsync(w->host, w->ctr, kCtrWords * sizeof(ull), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "k4 list lengths", err);
    w->lmax = static_cast<uint32_t>(w->host[kLmax]) + 1;  // + 1: "known" even when every list is empty
  }
  const uint32_t lmax = w->lmax - 1;
  if (lmax > kMaxL) return 2;
  uint64_t scratch_words = 0;
  if (lmax > kSmemL) {
    scratch_words = static_cast<uint64_t>(lmax) * (((lmax + 31) >> 5) | 1u);
    const size_t need = static_cast<size_t>(blocks) * scratch_words * sizeof(uint32_t);
    if (need > w->rows_bytes) {
      if (w->rows) cudaFree(w->rows);
      w->rows = nullptr;
      w->rows_bytes = 0;
      e = cudaMalloc(&w->rows, need);
      if (e != cudaSuccess) return cuda_fail(e, "k4 row scratch", err);
      w->rows_bytes = need;
    }
  }
  cudaEventRecord(w->ev0, st);
  if (k == 4) {
    k4_cta_kernel<4><<<blocks, kThreads, smem, st>>>(off, adj, n, shard, num_shards, w->ctr, w->rows, scratch_words,
                                                     tcount);
    k4_warp_kernel<4><<<num_sms * 8, kThreads, 0, st>>>(off, adj, n, shard, num_shards, w->ctr, tcount);
  } else {
    k4_cta_kernel<5><<<blocks, kThreads, smem, st>>>(off, adj, n, shard, num_shards, w->ctr, w->rows, scratch_words,
                                                     nullptr);
    k4_warp_kernel<5><<<num_sms * 8, kThreads, 0, st>>>(off, adj, n, shard, num_shards, w->ctr, nullptr);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k4 launch", err);
  cudaEventRecord(w->ev1, st);
  e = cudaMemcpyAsync(w->host, w->ctr, kCtrWords * sizeof(ull), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "k4 kernels", err);
  float t = 0.f;
  cudaEventElapsedTime(&t, w->ev0, w->ev1);
  *ms = t;
  if (w->host[kFlags] & 1ull) return 2;
  if (w->host[kFlags] & 2ull) return 3;
  *count = w->host[kCount];
  *units = w->host[kUnits];
  return 0;
}

}  // namespace smg

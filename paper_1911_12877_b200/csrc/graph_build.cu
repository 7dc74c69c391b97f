// graph_build.cu -- device-side CSR construction.
//
//   device_from_edges : Graph::from_edges (proj/src/graph.cpp:13-47) -- drop self
//                       loops, symmetrise, sort, deduplicate, offsets -- as two
//                       64-bit radix sorts (CUB) over canonical (min,max) keys
//                       and the directed slot keys, a unique pass, a degree
//                       histogram and a scan.  The output is bit-identical to
//                       the reference layout (strictly ascending lists).
//   device_orient     : orient_reindex (proj/src/graph.cpp:137-161) -- new ids
//                       by (degree desc, old id asc) via one radix sort of
//                       (maxdeg - deg, id) keys, relabel every slot, re-sort.
//
// Both leave the CSR resident on the device (plus the per-slot source map the
// counting kernels use), so a graph can be built and counted without the
// host-side single-threaded sort (50-130 s at cfg4/cfg5 in the reference).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <mutex>
#include <string>
#include <vector>

#include "graph_build.hpp"

namespace smg {

namespace {

constexpr uint64_t kLoopKey = ~0ull;

__global__ void canon_kernel(const uint32_t* __restrict__ pairs, uint64_t m, uint64_t n,
                             unsigned long long* __restrict__ keys, unsigned long long* loops,
                             unsigned int* bad) {
  uint64_t local = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u >= n || v >= n) {
      atomicOr(bad, 1u);
      keys[i] = kLoopKey;
      continue;
    }
    if (u == v) {
      ++local;
      keys[i] = kLoopKey;
      continue;
    }
    keys[i] = u < v ? (static_cast<unsigned long long>(u) << 32) | v
                    : (static_cast<unsigned long long>(v) << 32) | u;
  }
  if (local) atomicAdd(loops, static_cast<unsigned long long>(local));
}

// directed[2i] = (u,v), directed[2i+1] = (v,u) for the mu unique undirected keys
__global__ void expand_kernel(const unsigned long long* __restrict__ uniq, uint64_t mu,
                              unsigned long long* __restrict__ directed) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < mu;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = uniq[i];
    directed[2 * i] = k;
    directed[2 * i + 1] = (k << 32) | (k >> 32);
  }
}

// adj/src from sorted directed keys.
__global__ void split_kernel(const unsigned long long* __restrict__ keys, uint64_t slots,
                             uint32_t* __restrict__ adj, uint32_t* __restrict__ src) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < slots;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = keys[i];
    adj[i] = static_cast<uint32_t>(k);
    src[i] = static_cast<uint32_t>(k >> 32);
  }
}

// off[v] = lower_bound(src, v) over the sorted source column; deg[v] = off[v+1]-off[v].
__global__ void offsets_kernel(const uint32_t* __restrict__ src, uint64_t slots, uint64_t n,
                               unsigned long long* __restrict__ off) {
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v <= n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = slots;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (src[mid] < v) lo = mid + 1; else hi = mid;
    }
    off[v] = lo;
  }
}

__global__ void degree_kernel(const unsigned long long* __restrict__ off, uint64_t n,
                              unsigned long long* __restrict__ deg) {
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    deg[v] = off[v + 1] - off[v];
}

__global__ void degree_key_kernel(const unsigned long long* __restrict__ off, uint64_t n,
                                  uint64_t maxd, unsigned long long* __restrict__ keys) {
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t d = off[v + 1] - off[v];
    keys[v] = ((maxd - d) << 32) | v;  // ascending = degree desc, then old id asc
  }
}

__global__ void invert_kernel(const unsigned long long* __restrict__ sorted, uint64_t n,
                              uint32_t* __restrict__ new_to_old, uint32_t* __restrict__ old_to_new) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t old = static_cast<uint32_t>(sorted[i]);
    new_to_old[i] = old;
    old_to_new[old] = static_cast<uint32_t>(i);
  }
}

__global__ void relabel_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ adj,
                               uint64_t slots, const uint32_t* __restrict__ old_to_new,
                               unsigned long long* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < slots;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[i] = (static_cast<unsigned long long>(old_to_new[src[i]]) << 32) | old_to_new[adj[i]];
}

int bits_for(uint64_t n) {
  int b = 1;
  while ((1ull << b) < n + 1) ++b;
  return b;
}

// Temporaries of one build, freed on every exit path.  Stream-ordered
// allocations from the device's default pool, whose release threshold is
// raised once so that the sort buffers of one call serve the next (a graph
// handle per call pays no cudaMalloc/cudaFree round trips for them).
struct Guard {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Guard(cudaStream_t s) : st(s) {
    static std::once_flag once[64];
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64)
      std::call_once(once[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          unsigned long long keep = 8ull << 30;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
      });
  }
  ~Guard() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <class T>
  cudaError_t alloc(T** p, size_t bytes) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), bytes ? bytes : 8, st);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
};

#define GB_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      *err = std::string(#call) + ": " + cudaGetErrorString(e_);                   \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

// Sort directed slot keys (2*mu or slots of them) into a CSR at `out`.
int keys_to_csr(cudaStream_t st, unsigned long long* keys, unsigned long long* tmp, uint64_t slots,
                uint64_t n, int num_sms, DevCSR* out, std::string* err) {
  Guard g(st);
  const int end_bit = 32 + bits_for(n);
  size_t tb = 0;
  GB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, tmp, slots, 0, end_bit, st));
  void* tstore = nullptr;
  GB_CUDA(g.alloc(&tstore, tb));
  GB_CUDA(cub::DeviceRadixSort::SortKeys(tstore, tb, keys, tmp, slots, 0, end_bit, st));
  unsigned long long* deg = nullptr;
  GB_CUDA(g.alloc(&deg, (n + 1) * sizeof(unsigned long long)));
  GB_CUDA(cudaMemsetAsync(deg, 0, (n + 1) * sizeof(unsigned long long), st));
  GB_CUDA(cudaMalloc(&out->off, (n + 1) * sizeof(unsigned long long)));
  GB_CUDA(cudaMalloc(&out->adj, (slots ? slots : 1) * sizeof(uint32_t)));
  GB_CUDA(cudaMalloc(&out->src, (slots ? slots : 1) * sizeof(uint32_t)));
  const unsigned grid = static_cast<unsigned>(num_sms * 8);
  if (slots) split_kernel<<<grid, 256, 0, st>>>(tmp, slots, out->adj, out->src);
  offsets_kernel<<<grid, 256, 0, st>>>(out->src, slots, n, out->off);
  if (n) degree_kernel<<<grid, 256, 0, st>>>(out->off, n, deg);
  GB_CUDA(cudaGetLastError());
  unsigned long long* dmax = nullptr;
  GB_CUDA(g.alloc(&dmax, sizeof(unsigned long long)));
  size_t rb = 0;
  GB_CUDA(cub::DeviceReduce::Max(nullptr, rb, deg, dmax, n + 1, st));
  void* rstore = nullptr;
  GB_CUDA(g.alloc(&rstore, rb));
  GB_CUDA(cub::DeviceReduce::Max(rstore, rb, deg, dmax, n + 1, st));
  unsigned long long maxd = 0;
  GB_CUDA(cudaMemcpyAsync(&maxd, dmax, sizeof(maxd), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  out->n = n;
  out->slots = slots;
  out->max_degree = maxd;
  return 0;
}

}  // namespace

int device_from_edges(int dev, cudaStream_t st, int num_sms, const uint32_t* h_pairs, uint64_t m,
                      uint64_t n, DevCSR* out, uint64_t* dups, uint64_t* loops, std::string* err) {
  GB_CUDA(cudaSetDevice(dev));
  Guard g(st);
  uint32_t* pairs = nullptr;
  unsigned long long *keys = nullptr, *sorted = nullptr, *counters = nullptr;
  unsigned int* bad = nullptr;
  GB_CUDA(g.alloc(&pairs, 2 * m * sizeof(uint32_t)));
  GB_CUDA(g.alloc(&keys, m * sizeof(unsigned long long)));
  GB_CUDA(g.alloc(&sorted, m * sizeof(unsigned long long)));
  GB_CUDA(g.alloc(&counters, 2 * sizeof(unsigned long long)));
  GB_CUDA(g.alloc(&bad, sizeof(unsigned int)));
  GB_CUDA(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), st));
  GB_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned int), st));
  if (m) GB_CUDA(cudaMemcpyAsync(pairs, h_pairs, 2 * m * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  const unsigned grid = static_cast<unsigned>(num_sms * 8);
  if (m) canon_kernel<<<grid, 256, 0, st>>>(pairs, m, n, keys, counters, bad);
  GB_CUDA(cudaGetLastError());
  // sort canonical keys (self loops = ~0 sort last), unique
  size_t tb = 0;
  GB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, m, 0, 64, st));
  void* tstore = nullptr;
  GB_CUDA(g.alloc(&tstore, tb));
  if (m) GB_CUDA(cub::DeviceRadixSort::SortKeys(tstore, tb, keys, sorted, m, 0, 64, st));
  size_t ub = 0;
  GB_CUDA(cub::DeviceSelect::Unique(nullptr, ub, sorted, keys, counters + 1, m, st));
  void* ustore = nullptr;
  GB_CUDA(g.alloc(&ustore, ub));
  if (m) GB_CUDA(cub::DeviceSelect::Unique(ustore, ub, sorted, keys, counters + 1, m, st));
  unsigned long long host_c[2] = {0, 0};
  unsigned int host_bad = 0;
  GB_CUDA(cudaMemcpyAsync(host_c, counters, sizeof(host_c), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaMemcpyAsync(&host_bad, bad, sizeof(host_bad), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  if (host_bad) {
    *err = "edge endpoint out of range";
    return 2;
  }
  const uint64_t nloops = host_c[0];
  const uint64_t nuniq = m ? host_c[1] : 0;
  const uint64_t mu = nuniq - (nloops ? 1 : 0);  // all loops collapse into one ~0 key
  *loops = nloops;
  *dups = (m - nloops) - mu;
  unsigned long long* directed = nullptr;
  unsigned long long* dsorted = nullptr;
  GB_CUDA(g.alloc(&directed, 2 * mu * sizeof(unsigned long long)));
  GB_CUDA(g.alloc(&dsorted, 2 * mu * sizeof(unsigned long long)));
  if (mu) expand_kernel<<<grid, 256, 0, st>>>(keys, mu, directed);
  GB_CUDA(cudaGetLastError());
  return keys_to_csr(st, directed, dsorted, 2 * mu, n, num_sms, out, err);
}

int device_orient(int dev, cudaStream_t st, int num_sms, const DevCSR& in, DevCSR* out,
                  uint32_t* h_new_to_old, std::string* err) {
  GB_CUDA(cudaSetDevice(dev));
  Guard g(st);
  const uint64_t n = in.n;
  unsigned long long *vkeys = nullptr, *vsorted = nullptr;
  uint32_t *n2o = nullptr, *o2n = nullptr;
  GB_CUDA(g.alloc(&vkeys, n * sizeof(unsigned long long)));
  GB_CUDA(g.alloc(&vsorted, n * sizeof(unsigned long long)));
  GB_CUDA(g.alloc(&n2o, n * sizeof(uint32_t)));
  GB_CUDA(g.alloc(&o2n, n * sizeof(uint32_t)));
  const unsigned grid = static_cast<unsigned>(num_sms * 8);
  if (n) degree_key_kernel<<<grid, 256, 0, st>>>(in.off, n, in.max_degree, vkeys);
  GB_CUDA(cudaGetLastError());
  size_t tb = 0;
  GB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, vkeys, vsorted, n, 0, 64, st));
  void* tstore = nullptr;
  GB_CUDA(g.alloc(&tstore, tb));
  if (n) GB_CUDA(cub::DeviceRadixSort::SortKeys(tstore, tb, vkeys, vsorted, n, 0, 64, st));
  if (n) invert_kernel<<<grid, 256, 0, st>>>(vsorted, n, n2o, o2n);
  GB_CUDA(cudaGetLastError());
  unsigned long long *keys = nullptr, *sorted = nullptr;
  GB_CUDA(g.alloc(&keys, in.slots * sizeof(unsigned long long)));
  GB_CUDA(g.alloc(&sorted, in.slots * sizeof(unsigned long long)));
  if (in.slots) relabel_kernel<<<grid, 256, 0, st>>>(in.src, in.adj, in.slots, o2n, keys);
  GB_CUDA(cudaGetLastError());
  if (h_new_to_old && n)
    GB_CUDA(cudaMemcpyAsync(h_new_to_old, n2o, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  return keys_to_csr(st, keys, sorted, in.slots, n, num_sms, out, err);
}

}  // namespace smg

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

// ---------------------------------------------------------------- device ---

struct Counters {
  unsigned long long next_chunk;
  unsigned long long count;
  unsigned long long elements;
  unsigned long long units;
  unsigned int overflow;
  unsigned int pad;
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

template <bool METER>
__global__ void __launch_bounds__(kThreads) count_kernel(const KernelArgs a) {
  __shared__ WarpState states[kWarpsPerBlock];
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
      for (int t = P.node_begin[0]; t < P.node_end[0]; ++t) build_node(c, P, t);
      for (int t = P.node_begin[1]; t < P.node_end[1]; ++t) build_node(c, P, t);
      if (P.depth == 3) {
        checked_acc(cnt, leaf_count(c, P), ovf);
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
        for (int t = P.node_begin[level]; t < P.node_end[level]; ++t) build_node(c, P, t);
        if (level == P.depth - 2) {
          checked_acc(cnt, leaf_count(c, P), ovf);
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
  acc = __reduce_add_sync(kFull, static_cast<uint32_t>(acc & 0xffffffffu)) +
        (static_cast<uint64_t>(__reduce_add_sync(kFull, static_cast<uint32_t>(acc >> 32))) << 32);
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
int enqueue(const smg_graph& g, Replica& r, const Program& prog, const Launch& L) {
  SMG_CUDA(cudaSetDevice(r.device));
  const uint64_t cap = std::max<uint64_t>(32, (g.max_degree + 31) / 32 * 32);
  int per_sm = 0;
  if (L.meter) {
    SMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_kernel<true>, kThreads, 0));
  } else {
    SMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, count_kernel<false>, kThreads, 0));
  }
  per_sm = std::max(1, per_sm);
  uint64_t blocks = static_cast<uint64_t>(r.num_sms) * per_sm;
  // Keep the per-warp scratch within a budget (sets are at most max_degree).
  const uint64_t per_block = static_cast<uint64_t>(prog.nslots) * cap * 4 * kWarpsPerBlock;
  const uint64_t budget = 24ull << 30;
  if (per_block > 0) blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, budget / per_block));
  int rc = ensure_scratch(r, per_block * blocks);
  if (rc) return rc;
  SMG_CUDA(cudaMemsetAsync(r.ctr, 0, sizeof(Counters), r.active()));
  SMG_CUDA(cudaEventRecord(r.ev0, r.active()));
  if (L.meter && L.meter_roots && L.root_hi > L.root_lo) {
    const uint32_t nr = L.root_hi - L.root_lo;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((nr + 255) / 256, 4096));
    meter_roots_kernel<<<grid, 256, 0, r.active()>>>(r.off, r.adj, L.root_lo, L.root_hi,
                                                   prog.unit_bound, r.ctr);
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
  a.prog = prog;
  if (L.unit_end > L.unit_begin) {
    if (L.meter) {
      count_kernel<true><<<static_cast<unsigned>(blocks), kThreads, 0, r.active()>>>(a);
    } else {
      count_kernel<false><<<static_cast<unsigned>(blocks), kThreads, 0, r.active()>>>(a);
    }
  }
  SMG_CUDA(cudaGetLastError());
  SMG_CUDA(cudaEventRecord(r.ev1, r.active()));
  SMG_CUDA(cudaMemcpyAsync(r.host_ctr, r.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, r.active()));
  return SMG_OK;
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
  s += "],\"leaf\":" + (pr.depth >= 3 ? node_json(pr.leaf) : std::string("null")) + "}";
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

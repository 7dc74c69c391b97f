// k4.hpp -- 4-clique count on the degree-ordered copy of the CSR (see k4.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace smg {

// Work buffers of k4_count, kept by the caller between calls (k4_free releases them).
struct K4Work {
  unsigned long long* ctr = nullptr;  // device: queue cursors, count, flags, max list length
  unsigned long long* host = nullptr;  // pinned copy
  uint32_t* rows = nullptr;            // per-CTA adjacency rows of roots too large for shared memory
  size_t rows_bytes = 0;
  uint32_t lmax = 0;                   // max_d |N-(d)| of the CSR the buffers were sized for (0: unknown)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

// Number of k-cliques (k = 4 or 5) of the CSR whose largest vertex d is
// owned by `shard` (d % num_shards == shard), into *count; *units = the edges
// (u, d), u < d, of the owned d (the level-1 units); *ms = device time.
// The CSR must be sorted; it is meant to be the orient_reindex copy (ids by
// descending degree), where N-(d) = {u in N(d) : u < d} is short for every d.
// tcount (may be null; num_shards == 1 only): one word per slot, zeroed by the
// caller; on return the word of slot (d, u), u < d, holds |N(u) & N(d)|, the
// triangles on that edge -- every triangle is met once, at its largest vertex,
// as a local edge of that root, and adds one to each of its three edges.
// Returns 0, 1 on a CUDA error (*err), 2 if a root's N-(d) exceeds the
// kernel's capacity (the caller falls back to the generic executor), 3 on
// 64-bit overflow.
int k4_count(const unsigned long long* off, const uint32_t* adj, uint64_t n, uint32_t shard, uint32_t num_shards,
             int num_sms, cudaStream_t st, K4Work* w, uint32_t* tcount, unsigned long long* count,
             unsigned long long* units, double* ms, std::string* err, int k = 4);
void k4_free(K4Work* w);

}  // namespace smg

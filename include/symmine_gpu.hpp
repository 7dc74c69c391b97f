// symmine_gpu.hpp -- header-only C++ adapter: the reference's engine API on B200.
//
//   symmine::gpu::count_instances(const Graph&, const Plan&, unsigned gpus)
//
// has the signature and semantics of symmine::count_instances
// (proj/include/symmine/engine.hpp:23, proj/src/engine.cpp:145-179) with
// `workers` read as the number of GPUs.  It is compiled against the
// reference's own headers (Graph, Plan, CountResult, the error types) and
// links against libsymmine_gpu.so; no reference source changes.
//
//  * The CSR is read zero-copy through Graph's public accessors
//    (graph.hpp:34-41): adjacency = neighbors(0).data() .. + 2*edge_count(),
//    offsets rebuilt as neighbors(v).data() - base (size_t -> uint64_t).
//  * The device replica is cached per Graph object (a Graph is immutable after
//    construction, graph.hpp:18-19); call release(g) to drop it.  A cached
//    entry is reused only if the Graph at that address still has the same
//    shape, adjacency base pointer and a sampled checksum of its offsets and
//    adjacency, so a new Graph that lands at a destroyed one's address is
//    re-uploaded instead of silently counted on stale device data.
//  * C-ABI status codes are rethrown as the reference's exceptions:
//    SMG_EINPUT -> InputError, SMG_EOVERFLOW -> CountOverflowError,
//    SMG_EIO -> IoError (error.hpp:10-22), exactly the CLI's exit-code classes
//    (tools/main.cpp:20-23).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "symmine/engine.hpp"
#include "symmine/error.hpp"
#include "symmine_gpu.h"

namespace symmine::gpu {

namespace detail {

inline void check(int rc) {
  if (rc == SMG_OK) return;
  const std::string msg = smg_last_error();
  if (rc == SMG_EINPUT) throw InputError(msg);
  if (rc == SMG_EOVERFLOW) throw CountOverflowError(msg);
  throw IoError(msg);
}

// plan.hpp:14-37 -> smg_plan
inline smg_plan lower(const Plan& plan) {
  smg_plan p;
  std::memset(&p, 0, sizeof(p));
  p.depth = static_cast<int32_t>(plan.levels.size());
  if (p.depth > SMG_MAX_LEVELS) throw InputError("plan has more than 8 levels");
  for (int i = 0; i < SMG_MAX_LEVELS; ++i) p.parent[i] = -1;
  for (int i = 0; i < p.depth; ++i) {
    const PlanLevel& lv = plan.levels[i];
    for (int j : lv.intersect_sources) p.isect_mask[i] |= static_cast<uint8_t>(1u << j);
    for (int j : lv.diff_sources) p.diff_mask[i] |= static_cast<uint8_t>(1u << j);
    p.parent[i] = static_cast<int8_t>(lv.restriction_parent);
  }
  p.flags = (plan.options.use_bounds ? SMG_PLAN_USE_BOUNDS : 0u) |
            (plan.options.use_restrictions ? SMG_PLAN_USE_RESTRICTIONS : 0u);
  return p;
}

// Identity of a Graph's contents, cheap to recompute per call: shape, the
// adjacency base pointer and a checksum over <= 2 x 65,536 evenly spaced
// offsets and adjacency entries.
struct Fingerprint {
  size_t n = 0, m = 0;
  const VertexId* base = nullptr;
  uint64_t sum = 0;
  bool operator==(const Fingerprint& o) const {
    return n == o.n && m == o.m && base == o.base && sum == o.sum;
  }
};

inline Fingerprint fingerprint(const Graph& g) {
  Fingerprint f;
  f.n = g.vertex_count();
  f.m = g.edge_count();
  f.base = f.n ? g.neighbors(0).data() : nullptr;
  uint64_t h = 0x9E3779B97F4A7C15ull ^ (f.n * 31 + f.m);
  auto mix = [&h](uint64_t x) {
    h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
  };
  constexpr size_t kSamples = 65536;
  if (f.n) {
    const size_t step = std::max<size_t>(1, f.n / kSamples);
    for (size_t v = 0; v < f.n; v += step) mix(g.degree(static_cast<VertexId>(v)) * 0x100000001ull + v);
    const size_t slots = 2 * f.m;
    const size_t astep = std::max<size_t>(1, slots / kSamples);
    for (size_t i = 0; i < slots; i += astep) mix(f.base[i] ^ (static_cast<uint64_t>(i) << 32));
  }
  f.sum = h;
  return f;
}

struct Entry {
  Fingerprint fp;
  smg_graph* handle = nullptr;
};

struct Cache {
  std::mutex mu;
  std::map<std::pair<const Graph*, unsigned>, Entry> replicas;
  ~Cache() {
    for (auto& kv : replicas) smg_graph_destroy(kv.second.handle);
  }
};

inline Cache& cache() {
  static Cache c;
  return c;
}

inline smg_graph* replica(const Graph& g, unsigned gpus) {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  const Fingerprint fp = fingerprint(g);
  auto it = c.replicas.find({&g, gpus});
  if (it != c.replicas.end()) {
    if (it->second.fp == fp) return it->second.handle;
    smg_graph_destroy(it->second.handle);  // a different Graph now lives at this address
    c.replicas.erase(it);
  }
  const size_t n = g.vertex_count();
  std::vector<uint64_t> offsets(n + 1, 0);
  const VertexId* base = n ? g.neighbors(0).data() : nullptr;
  for (size_t v = 0; v < n; ++v) {
    const auto nb = g.neighbors(static_cast<VertexId>(v));
    offsets[v] = static_cast<uint64_t>(nb.data() - base);
    offsets[v + 1] = offsets[v] + nb.size();
  }
  smg_graph* h = nullptr;
  check(smg_graph_create(offsets.data(), base, n, nullptr, static_cast<int>(gpus), &h));
  c.replicas[{&g, gpus}] = Entry{fp, h};
  return h;
}

}  // namespace detail

// Drop the cached device replicas of g (call before destroying g).
inline void release(const Graph& g) {
  detail::Cache& c = detail::cache();
  std::lock_guard<std::mutex> lock(c.mu);
  for (auto it = c.replicas.begin(); it != c.replicas.end();) {
    if (it->first.first == &g) {
      smg_graph_destroy(it->second.handle);
      it = c.replicas.erase(it);
    } else {
      ++it;
    }
  }
}

// count_instances on `gpus` B200s (gpus == 0 -> 1, like workers, engine.cpp:146).
inline CountResult count_instances(const Graph& g, const Plan& plan, unsigned gpus = 1) {
  if (gpus == 0) gpus = 1;
  const smg_plan p = detail::lower(plan);
  smg_result r;
  detail::check(smg_count(detail::replica(g, gpus), &p, gpus, 0, &r));
  CountResult out;
  out.count = r.count;
  out.per_worker.assign(r.per_gpu, r.per_gpu + gpus);
  out.wall_ms = r.wall_ms;
  return out;
}

// One count_instances per plan as one call (the loop of motif_counts,
// engine.cpp:193-205): work the plans share on the device is done once.
inline std::vector<CountResult> count_many(const Graph& g, const std::vector<Plan>& plans, unsigned gpus = 1) {
  if (gpus == 0) gpus = 1;
  std::vector<smg_plan> pods;
  pods.reserve(plans.size());
  for (const Plan& p : plans) pods.push_back(detail::lower(p));
  std::vector<smg_result> res(plans.size());
  if (!plans.empty())
    detail::check(smg_count_many(detail::replica(g, gpus), pods.data(), static_cast<uint32_t>(pods.size()), gpus, 0,
                                 res.data()));
  std::vector<CountResult> out(plans.size());
  for (size_t i = 0; i < plans.size(); ++i) {
    out[i].count = res[i].count;
    out[i].per_worker.assign(res[i].per_gpu, res[i].per_gpu + gpus);
    out[i].wall_ms = res[i].wall_ms;
  }
  return out;
}

}  // namespace symmine::gpu

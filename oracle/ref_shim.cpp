// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.  C entry points over the
// reference symmine library compiled from /root/reference/proj (never copied;
// see oracle/Makefile).  Only tests/, __graft_entry__.smoke() and bench.py's
// CPU-baseline leg may load the resulting oracle/_ref/libsymmine_ref.so.
//
// The reference's Executor lives in an anonymous namespace of engine.cpp, so
// this TU includes that source file to reach Executor::count_range
// (proj/src/engine.cpp:36-43) for root-range parity; the library build leaves
// engine.cpp out of its own object list so nothing is defined twice.
// Everything engine.cpp includes comes first, so that the access override
// below applies to engine.cpp's own Executor only: ref_count_units drives the
// reference's count_from(2) for single level-1 units (v0, v1) -- the same
// code path count_range runs for them (engine.cpp:36-43, 89-115).
#include <array>
#include <chrono>
#include <optional>
#include <span>
#include <thread>
#include <vector>

#include "symmine/engine.hpp"
#include "symmine/error.hpp"
#include "symmine/set_ops.hpp"
#define private public
#include SYMMINE_ENGINE_CPP
#undef private

#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>
#include <sstream>
#include <string>

#include "symmine/error.hpp"
#include "symmine/oracle.hpp"
#include "symmine/plan.hpp"

using namespace symmine;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InputError& e) {
    g_err = e.what();
    return 2;
  } catch (const CountOverflowError& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int put(const std::string& s, char* buf, size_t cap) {
  if (s.size() + 1 > cap) {
    g_err = "buffer too small";
    return -static_cast<int>(s.size() + 1);
  }
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

Pattern pattern_of(const char* name, int k, const char* text) {
  if (text && *text) return parse_pattern(text);
  return named_pattern(name, k);
}

nlohmann::ordered_json plan_record(const Pattern& p, int schedule_index, bool use_r, bool use_b) {
  Schedule schedule;
  RestrictionMap rm;
  size_t index = 0;
  if (schedule_index < 0) {  // python/module.cpp:40-53 parents_from_choice
    SelectedSchedule sel = select_schedule(p, {});
    schedule = sel.choice.schedule;
    rm = sel.choice.restrictions;
    index = sel.index;
  } else {
    auto all = analyze_schedules(p, {});
    if (static_cast<size_t>(schedule_index) >= all.size()) throw InputError("schedule index out of range");
    schedule = all[schedule_index].schedule;
    rm = all[schedule_index].restrictions;
    index = static_cast<size_t>(schedule_index);
  }
  const Plan plan = compile_plan(p, schedule, rm, {use_r, use_b});
  nlohmann::ordered_json j = plan_to_json(plan);
  j["schedule_index"] = index;
  j["automorphisms"] = automorphisms(p).multiplicity();
  return j;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_graph_from_edges(uint64_t n, const uint32_t* pairs, uint64_t m, uint64_t* dups,
                           uint64_t* loops) {
  Graph* out = nullptr;
  int rc = guarded([&] {
    std::vector<std::pair<VertexId, VertexId>> edges(m);
    for (uint64_t i = 0; i < m; ++i) edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
    LoadStats st;
    out = new Graph(Graph::from_edges(n, edges, &st));
    if (dups) *dups = st.duplicate_edges;
    if (loops) *loops = st.self_loops;
  });
  return rc ? nullptr : out;
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

void ref_graph_shape(void* gp, uint64_t* n, uint64_t* slots, uint64_t* maxd) {
  const Graph& g = *static_cast<Graph*>(gp);
  *n = g.vertex_count();
  *slots = 2 * g.edge_count();
  *maxd = g.max_degree();
}

void ref_graph_csr(void* gp, uint64_t* off, uint32_t* adj) {
  const Graph& g = *static_cast<Graph*>(gp);
  uint64_t pos = 0;
  off[0] = 0;
  for (VertexId v = 0; v < g.vertex_count(); ++v) {
    for (VertexId x : g.neighbors(v)) adj[pos++] = x;
    off[v + 1] = pos;
  }
}

void* ref_graph_orient(void* gp, uint32_t* new_to_old) {
  OrientResult r = orient_reindex(*static_cast<Graph*>(gp));
  if (new_to_old) std::memcpy(new_to_old, r.new_to_old.data(), r.new_to_old.size() * sizeof(uint32_t));
  return new Graph(std::move(r.graph));
}

// Plan JSON (plan_to_json, plan.cpp:31-50) plus schedule_index/automorphisms.
int ref_plan_json(const char* name, int k, const char* pattern_text, int schedule_index,
                  int use_restrictions, int use_bounds, char* buf, size_t cap) {
  std::string s;
  int rc = guarded([&] {
    s = plan_record(pattern_of(name, k, pattern_text), schedule_index, use_restrictions != 0,
                    use_bounds != 0).dump();
  });
  return rc ? rc : put(s, buf, cap);
}

// motif_counts' plans (engine.cpp:193-205): one record per connected k-pattern.
int ref_motif_plans_json(int k, char* buf, size_t cap) {
  std::string s;
  int rc = guarded([&] {
    nlohmann::ordered_json arr = nlohmann::ordered_json::array();
    for (Pattern& p : connected_patterns(k)) {
      nlohmann::ordered_json j = plan_record(p, -1, true, true);
      j["key"] = canonical_key(p);
      j["bits"] = adjacency_bits(p);
      j["name"] = pattern_display_name(p);
      arr.push_back(std::move(j));
    }
    s = arr.dump();
  });
  return rc ? rc : put(s, buf, cap);
}

void* ref_plan_from_json(const char* text) {
  Plan* out = nullptr;
  int rc = guarded([&] { out = new Plan(plan_from_json(nlohmann::json::parse(text))); });
  return rc ? nullptr : out;
}

void ref_plan_free(void* p) { delete static_cast<Plan*>(p); }

int ref_count(void* g, void* plan, unsigned workers, uint64_t* count, double* wall_ms) {
  return guarded([&] {
    CountResult r = count_instances(*static_cast<Graph*>(g), *static_cast<Plan*>(plan), workers);
    *count = r.count;
    if (wall_ms) *wall_ms = r.wall_ms;
  });
}

// Executor(g, plan).count_range(lo, hi): the reference's own per-root counts.
int ref_count_range(void* g, void* plan, uint32_t lo, uint32_t hi, uint64_t* count) {
  return guarded([&] {
    Executor exec(*static_cast<Graph*>(g), *static_cast<Plan*>(plan));
    *count = exec.count_range(lo, hi);
  });
}

int ref_enumerate(void* g, void* plan, int has_limit, uint64_t limit, uint32_t* out,
                  uint64_t cap_tuples, uint64_t* n_out) {
  return guarded([&] {
    const Plan& p = *static_cast<Plan*>(plan);
    std::optional<uint64_t> lim;
    if (has_limit) lim = limit;
    auto emb = enumerate_instances(*static_cast<Graph*>(g), p, lim);
    const size_t depth = p.levels.size();
    uint64_t w = 0;
    for (const auto& e : emb) {
      if (w >= cap_tuples) break;
      for (size_t i = 0; i < depth; ++i) out[w * depth + i] = e[i];
      ++w;
    }
    *n_out = emb.size();
  });
}

int ref_oracle_induced(void* g, const char* name, int k, const char* pattern_text, uint64_t* count) {
  return guarded([&] { *count = oracle::induced_count(*static_cast<Graph*>(g), pattern_of(name, k, pattern_text)); });
}

// Dynamic root queue over all host threads with one Executor per thread (the
// reference's count_instances uses static root blocks, engine.cpp:157-158,
// whose slowest block sets the wall time).  Chunk c covers roots
// [starts[c], starts[c+1]); chunks are claimed in `order`, skipping those with
// done[c] != 0, and each finished chunk stores its count and sets done[c] = 1
// (the caller may snapshot both arrays while this runs: checkpoint/resume).
int ref_count_chunks(void* g, void* plan, unsigned workers, const uint32_t* starts, uint64_t nchunks,
                     const uint64_t* order, uint64_t* counts, volatile uint8_t* done) {
  std::atomic<uint64_t> next{0};
  std::atomic<int> status{0};
  auto work = [&] {
    int rc = guarded([&] {
      Executor exec(*static_cast<Graph*>(g), *static_cast<Plan*>(plan));
      for (;;) {
        if (status.load()) return;
        const uint64_t i = next.fetch_add(1);
        if (i >= nchunks) return;
        const uint64_t c = order[i];
        if (done[c]) continue;
        counts[c] = exec.count_range(starts[c], starts[c + 1]);
        std::atomic_thread_fence(std::memory_order_release);
        done[c] = 1;
      }
    });
    if (rc) status.store(rc);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < std::max(1u, workers); ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  return status.load();
}

// Per-root counts with the per-root CPU time (ns) of each, one Executor per
// thread, dynamic queue: the CPU baseline's sampler and hub-root goldens.
int ref_count_roots(void* g, void* plan, unsigned workers, const uint32_t* roots, uint64_t nroots,
                    uint64_t* counts, uint64_t* ns) {
  std::atomic<uint64_t> next{0};
  std::atomic<int> status{0};
  auto work = [&] {
    int rc = guarded([&] {
      Executor exec(*static_cast<Graph*>(g), *static_cast<Plan*>(plan));
      for (;;) {
        if (status.load()) return;
        const uint64_t i = next.fetch_add(1);
        if (i >= nroots) return;
        const auto t0 = std::chrono::steady_clock::now();
        counts[i] = exec.count_range(roots[i], roots[i] + 1);
        if (ns)
          ns[i] = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
      }
    });
    if (rc) status.store(rc);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < std::max(1u, workers); ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  return status.load();
}

// Per-unit counts of level-1 units (v0, v1) = directed edge slots, with the
// per-unit CPU time (ns): the reference's own count_from(2) after fixing
// values_[0..1] -- exactly what count_range does for that v1 inside root v0's
// level-1 loop (engine.cpp:106-113), including the level-1 parent check.
// Dynamic queue, one Executor per thread.  Used for edge-slot sampling (the
// CPU baseline) and per-unit goldens.
// budget_s > 0: stop claiming units once that much wall time has passed;
// *processed = the number of units counted (always a prefix of the list).
int ref_count_units(void* gp, void* pp, unsigned workers, const uint32_t* v0s, const uint32_t* v1s,
                    uint64_t nunits, uint64_t* counts, uint64_t* ns, double budget_s, uint64_t* processed) {
  const Graph& g = *static_cast<Graph*>(gp);
  const Plan& plan = *static_cast<Plan*>(pp);
  if (plan.levels.size() < 2) {
    g_err = "unit counts need a plan of depth >= 2";
    return 2;
  }
  const int par1 = plan.levels[1].restriction_parent;
  std::atomic<uint64_t> next{0};
  std::atomic<int> status{0};
  const auto start = std::chrono::steady_clock::now();
  auto work = [&] {
    int rc = guarded([&] {
      Executor exec(g, plan);
      for (;;) {
        if (status.load()) return;
        if (budget_s > 0 && std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count() > budget_s)
          return;
        const uint64_t i = next.fetch_add(1);
        if (i >= nunits) return;
        const auto t0 = std::chrono::steady_clock::now();
        uint64_t c = 0;
        if (!(par1 == 0 && v1s[i] >= v0s[i])) {
          exec.values_[0] = v0s[i];
          exec.values_[1] = v1s[i];
          c = plan.levels.size() == 2 ? 1 : exec.count_from(2);
        }
        counts[i] = c;
        if (ns)
          ns[i] = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
      }
    });
    if (rc) status.store(rc);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < std::max(1u, workers); ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (processed) *processed = std::min<uint64_t>(next.load(), nunits);
  return status.load();
}

}  // extern "C"

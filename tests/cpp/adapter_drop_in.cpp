// Drop-in check of include/symmine_gpu.hpp against the reference, written the
// way a reference maintainer would use it: the reference's own front end
// (named_pattern -> select_schedule -> compile_plan) and Graph::from_edges,
// then symmine::count_instances (CPU, reference engine) vs
// symmine::gpu::count_instances (B200).  Built by `make -C oracle adapter`
// against /root/reference headers; run by tests/test_gpu.py.
#include <cstdio>
#include <optional>
#include <random>

#include "symmine/cost_model.hpp"
#include "symmine/pattern.hpp"
#include "symmine/engine.hpp"
#include "symmine/error.hpp"
#include "symmine_gpu.hpp"

using namespace symmine;

int main() {
  std::mt19937 gen(7);
  std::vector<std::pair<VertexId, VertexId>> edges;
  const size_t n = 300;
  for (VertexId i = 0; i < n; ++i)
    for (VertexId j = i + 1; j < n; ++j)
      if (gen() % 100 < 6) edges.emplace_back(i, j);
  const Graph g = Graph::from_edges(n, edges);
  int bad = 0;
  const char* names[] = {"triangle", "rectangle", "pentagon", "house", "tailed_triangle", "hourglass"};
  for (const char* name : names) {
    const Pattern p = named_pattern(name);
    const SelectedSchedule sel = select_schedule(p, {});
    for (int opt = 0; opt < 3; ++opt) {
      PlanOptions o{opt != 1, opt != 2};
      const Plan plan = compile_plan(p, sel.choice.schedule, sel.choice.restrictions, o);
      const uint64_t cpu = count_instances(g, plan, 4).count;
      const CountResult r = gpu::count_instances(g, plan, 1);
      std::printf("%-16s restrictions=%d bounds=%d cpu=%llu gpu=%llu per_worker[0]=%llu\n", name,
                  o.use_restrictions, o.use_bounds, (unsigned long long)cpu,
                  (unsigned long long)r.count, (unsigned long long)r.per_worker.at(0));
      if (cpu != r.count) ++bad;
    }
  }
  // the motif loop (engine.cpp:193-205) as one batched call
  {
    std::vector<Plan> plans;
    std::vector<uint64_t> cpu;
    for (Pattern& p : connected_patterns(4)) {
      const SelectedSchedule sel = select_schedule(p, {});
      plans.push_back(compile_plan(p, sel.choice.schedule, sel.choice.restrictions));
      cpu.push_back(count_instances(g, plans.back(), 4).count);
    }
    const std::vector<CountResult> many = gpu::count_many(g, plans, 1);
    for (size_t i = 0; i < plans.size(); ++i) {
      std::printf("motif4[%zu] cpu=%llu gpu(count_many)=%llu\n", i, (unsigned long long)cpu[i],
                  (unsigned long long)many[i].count);
      if (cpu[i] != many[i].count) ++bad;
    }
  }
  // errors cross the ABI as the reference's exception types
  Plan broken = compile_plan(named_pattern("triangle"), {0, 1, 2}, {-1, 0, 1});
  broken.levels[2].restriction_parent = 2;
  try {
    gpu::count_instances(g, broken, 1);
    ++bad;
  } catch (const InputError& e) {
    std::printf("InputError as expected: %s\n", e.what());
  }
  gpu::release(g);

  // A loop-scoped Graph that lands where a released one lived must not reuse
  // the stale device replica (the cache checks a content fingerprint).
  {
    std::optional<Graph> slot;
    const Plan tri = compile_plan(named_pattern("triangle"), {0, 1, 2}, {-1, 0, 1});
    for (int round = 0; round < 3; ++round) {
      std::vector<std::pair<VertexId, VertexId>> es;
      const VertexId k = 20 + 5 * round;  // K_k: C(k,3) triangles
      for (VertexId i = 0; i < k; ++i)
        for (VertexId j = i + 1; j < k; ++j) es.emplace_back(i, j);
      slot.emplace(Graph::from_edges(k, es));
      const uint64_t want = uint64_t(k) * (k - 1) * (k - 2) / 6;
      const uint64_t got = gpu::count_instances(*slot, tri, 1).count;
      std::printf("K_%u triangles: gpu=%llu want=%llu\n", k, (unsigned long long)got, (unsigned long long)want);
      if (got != want) ++bad;
      slot.reset();  // destroyed without release(): the next Graph may reuse the address
    }
  }

  // A real device overflow: induced 3-stars (motif star4 plan, as motif_counts
  // compiles it, engine.cpp:193-205) in a star with 5,000,000 leaves number
  // C(5e6, 3) > 2^64 -> CountOverflowError, like checked_add (engine.cpp:13-19).
  {
    const VertexId leaves = 5000000;
    std::vector<std::pair<VertexId, VertexId>> es;
    es.reserve(leaves);
    for (VertexId i = 1; i <= leaves; ++i) es.emplace_back(0, i);
    const Graph star = Graph::from_edges(leaves + 1, es);
    for (Pattern& p : connected_patterns(4)) {
      if (pattern_display_name(p) != "star4") continue;
      const SelectedSchedule ss = select_schedule(p, {});
      const Plan plan = compile_plan(p, ss.choice.schedule, ss.choice.restrictions);
      try {
        const CountResult r = gpu::count_instances(star, plan, 1);
        std::printf("star4 on the 5M-leaf star: no overflow (count %llu)\n", (unsigned long long)r.count);
        ++bad;
      } catch (const CountOverflowError& e) {
        std::printf("CountOverflowError as expected: %s\n", e.what());
      }
    }
    gpu::release(star);
  }
  std::printf(bad ? "FAILED\n" : "OK\n");
  return bad ? 1 : 0;
}

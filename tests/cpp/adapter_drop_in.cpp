// Drop-in check of include/symmine_gpu.hpp against the reference, written the
// way a reference maintainer would use it: the reference's own front end
// (named_pattern -> select_schedule -> compile_plan) and Graph::from_edges,
// then symmine::count_instances (CPU, reference engine) vs
// symmine::gpu::count_instances (B200).  Built by `make -C oracle adapter`
// against /root/reference headers; run by tests/test_gpu.py.
#include <cstdio>
#include <random>

#include "symmine/cost_model.hpp"
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
  std::printf(bad ? "FAILED\n" : "OK\n");
  return bad ? 1 : 0;
}

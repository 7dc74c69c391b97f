/*
 * symmine_gpu.h -- C ABI of the B200 subgraph-counting engine.
 *
 * This is the drop-in boundary for the reference's matching step:
 *
 *   CountResult symmine::count_instances(const Graph& g, const Plan& plan,
 *                                        unsigned workers = 1);
 *     reference: proj/include/symmine/engine.hpp:23, proj/src/engine.cpp:145-179
 *
 * The host front end (pattern -> automorphisms -> schedules -> restrictions ->
 * compile_plan) stays in the reference's C++ and is unchanged.  A caller
 * uploads the sorted CSR once (smg_graph_create), lowers a compiled Plan to
 * the POD smg_plan (one entry per PlanLevel, proj/include/symmine/plan.hpp:14-18)
 * and calls smg_count.  No C++ exceptions and no torch types cross this ABI;
 * status codes mirror the reference CLI's exit codes (tools/main.cpp:20-23):
 *
 *   SMG_OK        0  success
 *   SMG_EIO       1  CUDA / device / allocation failure   (IoError, error.hpp:15-17)
 *   SMG_EINPUT    2  malformed plan or graph              (InputError, error.hpp:10-12)
 *   SMG_EOVERFLOW 3  count does not fit in 64 bits         (CountOverflowError,
 *                                                           error.hpp:19-22, engine.cpp:13-19)
 *
 * The C++ adapter in symmine_gpu.hpp rethrows these as the reference's
 * exception types.  See INTEGRATION.md for the reference-side binding.
 */
#ifndef SYMMINE_GPU_H_
#define SYMMINE_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMG_OK 0
#define SMG_EIO 1
#define SMG_EINPUT 2
#define SMG_EOVERFLOW 3

/* kMaxPatternVertices, proj/include/symmine/pattern.hpp:12 */
#define SMG_MAX_LEVELS 8
#define SMG_MAX_GPUS 8

/* smg_plan.flags */
#define SMG_PLAN_USE_BOUNDS 1u       /* PlanOptions::use_bounds (plan.hpp:20-23)       */
#define SMG_PLAN_USE_RESTRICTIONS 2u /* PlanOptions::use_restrictions (informational)  */

/* flags argument of the count calls */
#define SMG_METER 1u /* also compute E, the intersected-element count */
/* Run the generic plan executor, on the caller's vertex labels, even where a
 * folded closed-form kernel exists for the plan or its full count is
 * label-free (clique plans and the 4-vertex closed forms otherwise run on a
 * degree-ordered copy of the CSR).  The folded kernels never meter E:
 * SMG_METER also selects this path.  For A/B parity checks. */
#define SMG_GENERIC 2u
/* Root-range calls (smg_count_range) of the two-centre folded kinds (house,
 * tailed diamond b, path4, rectangle) run the generic executor unless this
 * flag asks for the folded per-unit passes (they sweep the whole graph once,
 * then serve later ranges from cached per-unit values). */
#define SMG_FOLDED_RANGE 4u

/*
 * One compiled plan, the POD image of symmine::Plan (plan.hpp:25-37) as
 * produced by compile_plan (plan.cpp:9-29).  Level 0 iterates every vertex;
 * level i >= 1 is
 *   C_i = { c : c in N(v_j) for every j in isect_mask[i],
 *               c not in N(v_j) for every j in diff_mask[i],
 *               c not in {v_0..v_{i-1}},
 *               c < v_parent[i]            when parent[i] >= 0 }
 * Bit j of isect_mask[i] / diff_mask[i] is earlier level j
 * (PlanLevel::intersect_sources / diff_sources); parent[i] is
 * PlanLevel::restriction_parent (-1 = kNoParent).  use_bounds only moves
 * where the bound is checked (engine.cpp:60-63 vs :95-96); counts are equal.
 */
typedef struct smg_plan {
  int32_t depth; /* number of levels = pattern vertex count, 2..8 */
  uint8_t isect_mask[SMG_MAX_LEVELS];
  uint8_t diff_mask[SMG_MAX_LEVELS];
  int8_t parent[SMG_MAX_LEVELS];
  uint32_t flags; /* SMG_PLAN_* */
} smg_plan;

/* CountResult (engine.hpp:11-15) plus device-side counters. */
typedef struct smg_result {
  uint64_t count;                  /* exact embedding count                         */
  uint64_t per_gpu[SMG_MAX_GPUS];  /* per-device partial counts (per_worker)        */
  uint64_t elements;               /* E (only with SMG_METER, else 0)               */
  uint64_t units;                  /* level-1 partial embeddings (v0,v1) processed  */
  double wall_ms;                  /* host wall time of the call                    */
  double kernel_ms;                /* device time of the counting kernels (max/GPU) */
  /* High 64 bits (two's complement) of a shard's signed partial: the folded
   * full-count kernels (house, tailed diamonds) split closed-form terms so a
   * single shard's share may fall outside [0, 2^64); the shares still sum
   * exactly to the count.  Always 0 for smg_count / smg_count_range and for
   * every other plan. */
  int64_t count_hi;
} smg_result;

typedef struct smg_graph smg_graph;

/*
 * Upload a sorted, symmetric CSR (the layout Graph::from_edges builds,
 * graph.cpp:13-47: offsets[n+1] as size_t, adjacency[offsets[n]] uint32,
 * each slice strictly ascending, no self loops) and replicate it on
 * devices[0..num_devices).  devices == NULL means devices 0..num_devices-1.
 * The host arrays are only read during the call.
 */
int smg_graph_create(const uint64_t* offsets, const uint32_t* adjacency, uint64_t n_vertices,
                     const int* devices, int num_devices, smg_graph** out);
void smg_graph_destroy(smg_graph* g);

/*
 * Graph::from_edges (graph.cpp:13-47) on the device: pairs[2i], pairs[2i+1]
 * is edge i over vertices 0..n-1; self loops and duplicates are dropped and
 * counted (LoadStats, graph.hpp:13-16); the sorted symmetric CSR is built on
 * devices[0] (radix sorts) and replicated on the others.  The result is
 * structurally equal (Graph::operator==, graph.hpp:50-52) to the host build.
 */
int smg_graph_from_edges(const uint32_t* pairs, uint64_t num_edges, uint64_t n_vertices,
                         const int* devices, int num_devices, smg_graph** out,
                         uint64_t* duplicate_edges, uint64_t* self_loops);

/*
 * orient_reindex (graph.cpp:137-161) on replica `replica`'s device: new ids by
 * (degree desc, old id asc); new_to_old (n entries, host) may be NULL.  The new
 * graph has one replica on that device.
 */
int smg_graph_orient(const smg_graph* g, int replica, smg_graph** out, uint32_t* new_to_old);

/* Copy replica `replica`'s CSR to the host (offsets: n+1, adjacency: slots). */
int smg_graph_download(const smg_graph* g, int replica, uint64_t* offsets, uint32_t* adjacency);
int smg_graph_info(const smg_graph* g, uint64_t* n_vertices, uint64_t* n_slots,
                   uint64_t* max_degree, int* num_devices);

/*
 * Launch replica `replica`'s work on the caller's CUDA stream (a
 * cudaStream_t of that replica's device; NULL restores the library's own
 * stream).  Calls still return only after their results are on the host.
 */
int smg_graph_set_stream(smg_graph* g, int replica, void* stream);

/* Check an smg_plan against the PlanLevel invariants of compile_plan. */
int smg_plan_validate(const smg_plan* plan);

/*
 * The device set program the plan lowers to (hoisted, shared prefix sets),
 * as JSON into buf.  Host-only; for inspection and tests.  Returns SMG_OK,
 * or SMG_EINPUT for a bad plan / too small a buffer.
 */
int smg_plan_describe(const smg_plan* plan, char* buf, size_t cap);

/*
 * count_instances(g, plan, workers) with workers -> GPUs: the level-1 edge
 * units are sharded over the first num_gpus replicas of g, each device runs
 * its shard, and the partial counts are summed with overflow detection
 * (checked_add, engine.cpp:13-19, :172-174).
 */
int smg_count(const smg_graph* g, const smg_plan* plan, unsigned num_gpus, uint32_t flags,
              smg_result* out);

/*
 * motif_counts' loop over plans (engine.cpp:193-205: one count_instances per
 * connected pattern) as one call: out[i] is what smg_count(g, &plans[i],
 * num_gpus, flags, &out[i]) returns.  Work the plans share is done once per
 * call: the 4-vertex plans that have a closed form over subgraph counts of the
 * whole graph (star, path, cycle, tailed triangle, diamond) share one 4-clique
 * count, one triangle-per-edge pass and one 4-cycle pass, and a fully
 * restricted 4-clique plan in the batch takes its count from the same K4.
 */
int smg_count_many(const smg_graph* g, const smg_plan* plans, uint32_t num_plans, unsigned num_gpus,
                   uint32_t flags, smg_result* out);
/* The same for one shard on one replica (one process per GPU): out[i] is what
 * smg_count_shard(g, &plans[i], replica, shard, num_shards, flags, &out[i]) returns. */
int smg_count_many_shard(const smg_graph* g, const smg_plan* plans, uint32_t num_plans, int replica,
                         uint32_t shard, uint32_t num_shards, uint32_t flags, smg_result* out);

/*
 * Device times (CUDA events on the launching stream, ms) of the kernels of the
 * last closed-form 4-vertex count on a replica: ms[0] the 4-clique count
 * (k4_cta_kernel + k4_warp_kernel, or the generic count_kernel), ms[1] the
 * 4-cycle pass (c4_group_kernel, c4_hub_kernel launches, c4_kernel), ms[2] the
 * edge pass, ms[3] m4_vertex_kernel.  For measurement (bench.py's roofline).
 */
int smg_phase_times(const smg_graph* g, int replica, double* ms);

/*
 * One shard of the level-1 units on replica `replica` of g (one process per
 * GPU: shard = rank, num_shards = world size).  Shards of any num_shards
 * partition the units exactly, so the sum over shards equals smg_count.
 */
int smg_count_shard(const smg_graph* g, const smg_plan* plan, int replica, uint32_t shard,
                    uint32_t num_shards, uint32_t flags, smg_result* out);

/*
 * The shard map smg_count / smg_count_shard use for num_shards > 1 (replaces
 * the reference's static root blocks, engine.cpp:157-158): the level-1 unit
 * slots are cut into chunks of 32; chunk k costs sum over its slots (v0, v1)
 * of 1 + min(deg v0, deg v1) (only slots with v1 < v0 when unit_bound); the
 * chunks are split into J = num_shards * 64 super-chunks of equal cost
 * (bounds[j] = first chunk k whose exclusive cost prefix P[k] satisfies
 * P[k] * J >= j * total; bounds[J] = #chunks), and super-chunk j belongs to
 * shard j % num_shards, which runs a dynamic queue over its super-chunks.
 * Writes the J + 1 bounds (host array).
 */
int smg_shard_bounds(const smg_graph* g, int replica, uint32_t num_shards, int unit_bound,
                     uint64_t* bounds);

/* Roots [lo, hi) only, like Executor::count_range (engine.cpp:36-43). */
int smg_count_range(const smg_graph* g, const smg_plan* plan, int replica, uint32_t lo,
                    uint32_t hi, uint32_t flags, smg_result* out);

/*
 * enumerate_instances(g, plan, limit) (engine.hpp:34-37, engine.cpp:181-191):
 * the completed embeddings as per-level vertex tuples in the reference's
 * order (level-0 ascending, then lexicographic), truncated at `limit` when
 * has_limit (limit 0 -> none).  Writes min(total, cap_tuples) tuples of
 * plan->depth uint32 each to out; *n_out = total (after truncation).
 */
int smg_enumerate(const smg_graph* g, const smg_plan* plan, int replica, int has_limit,
                  uint64_t limit, uint32_t* out, uint64_t cap_tuples, uint64_t* n_out);

/* Last error message of the calling thread ("" if none). */
const char* smg_last_error(void);

/* Number of visible CUDA devices (0 when there is no GPU). */
int smg_device_count(void);

/* ABI version, bumped on any change to the structs above. */
int smg_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SYMMINE_GPU_H_ */

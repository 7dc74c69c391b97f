/*
 * symmine_graph.h -- host-side CSR toolkit of the B200 engine (C ABI).
 *
 * Builds the sorted, symmetric, deduplicated uint32 CSR that the reference's
 * Graph::from_edges produces (proj/src/graph.cpp:13-47) and the seeded
 * synthetic graphs of the five BASELINE configs:
 *   ER (uniform pairs, first m distinct), RMAT (a,b,c,d quadrant recursion,
 *   ids permuted), Chung-Lu (power-law expected degrees, capped, first m
 *   distinct, ids permuted).
 * All randomness is a counter-based splitmix64 stream keyed by the seed, so
 * every generator is deterministic and independent of the thread count.
 * Status codes as in symmine_gpu.h.
 */
#ifndef SYMMINE_GRAPH_H_
#define SYMMINE_GRAPH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct smg_csr smg_csr;

/* Graph::from_edges: pairs[2*i], pairs[2*i+1] is edge i.  Self loops and
 * duplicates are dropped and counted (LoadStats, graph.hpp:13-16). */
int smg_csr_from_edges(uint64_t n, const uint32_t* pairs, uint64_t num_edges, smg_csr** out,
                       uint64_t* duplicate_edges, uint64_t* self_loops);

int smg_gen_er(uint64_t n, uint64_t m, uint64_t seed, smg_csr** out);
int smg_gen_rmat(int scale, uint64_t edge_factor, double a, double b, double c, uint64_t seed,
                 smg_csr** out);
int smg_gen_chung_lu(uint64_t n, uint64_t m, double gamma, double w_max, uint64_t seed,
                     smg_csr** out);

/* Relabel by (degree desc, id asc), orient_reindex (graph.cpp:137-161). */
int smg_csr_orient(const smg_csr* g, smg_csr** out, uint32_t* new_to_old /* n, may be NULL */);

int smg_csr_info(const smg_csr* g, uint64_t* n, uint64_t* slots, uint64_t* max_degree);
const uint64_t* smg_csr_offsets(const smg_csr* g);
const uint32_t* smg_csr_adjacency(const smg_csr* g);
void smg_csr_free(smg_csr* g);
const char* smg_graph_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SYMMINE_GRAPH_H_ */

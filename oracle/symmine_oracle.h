/* symmine_oracle.h -- TEST INFRASTRUCTURE ONLY (see symmine_oracle.c). */
#ifndef SYMMINE_ORACLE_H_
#define SYMMINE_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/symmine_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

size_t oracle_intersect(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int has_bound,
                        uint32_t bound, uint32_t* out);
size_t oracle_difference(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int has_bound,
                         uint32_t bound, uint32_t* out);

int oracle_count_range(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                       uint32_t lo, uint32_t hi, uint64_t* count, uint64_t* elements);
int oracle_count(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                 int threads, uint64_t* count, uint64_t* elements);
int oracle_count_edges(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                       const uint64_t* slots, uint64_t num_slots, uint64_t* count,
                       uint64_t* elements);
int oracle_enumerate(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                     uint64_t limit, uint32_t* out, uint64_t* n_out);
int oracle_from_edges(uint64_t n, const uint32_t* pairs, uint64_t m, uint64_t* off, uint32_t* adj,
                      uint64_t* slots, uint64_t* dups, uint64_t* loops);
int oracle_orient(const uint64_t* off, const uint32_t* adj, uint64_t n, uint64_t* off_out,
                  uint32_t* adj_out, uint32_t* new_to_old);

#ifdef __cplusplus
}
#endif

#endif

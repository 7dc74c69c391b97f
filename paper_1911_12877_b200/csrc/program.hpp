// program.hpp -- lowering of an smg_plan to the device set program.
//
// The reference builds every level's candidate set from scratch
// (Executor::build_level, proj/src/engine.cpp:58-80): for level i it re-reads
// the neighbour lists of all earlier levels for every partial embedding.  The
// set each level needs is
//
//   C_i = (AND_{j in I_i} N(v_j)) - (OR_{j in D_i} N[v_j]),  c < v_{p_i}
//
// (closed neighbourhoods N[v] = N(v) + {v} implement the `taken` test,
// engine.cpp:82-87, because every earlier level is in I_i or D_i and there
// are no self loops).  Evaluated left to right over the sources in level
// order, the prefix over sources 0..k depends only on v_0..v_k, so it can be
// built once when v_k is fixed and reused for every later sibling: this is
// loop-invariant hoisting of the plan's set expressions.  Prefixes that are
// equal (same sources split the same way, same bound) are shared between
// levels, e.g. for clique-k the prefix of C_{i+1} over 0..i-1 *is* C_i.
//
// Bounds: a prefix built at loop k for level i can only apply a bound whose
// value is known at k.  Restrictions form chains v_a < v_{parent(a)}, so the
// tightest usable bound is the nearest ancestor of p_i in that chain with
// index <= k; the final set applies p_i itself.  All sets are sorted, so a
// bound is a prefix truncation and results are identical to the reference.
#pragma once

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/symmine_gpu.h"

namespace smg {

constexpr int kMaxLevels = SMG_MAX_LEVELS;
constexpr int kMaxNodes = 32;
constexpr int kMaxOps = 8;

enum : int8_t { kOpIsect = 0, kOpDiff = 1 };

struct Op {
  int8_t level;  // earlier level whose neighbour list is used
  int8_t mode;   // kOpIsect: keep x in N(v); kOpDiff: keep x not in N[v]
};

// One set in the program.  Built at loop level k (right after v_k is fixed)
// from `src` (a node built at an earlier loop level) or, when src < 0, from
// the raw CSR slice N(v_list); then filtered by ops and bounded by v_bound.
struct Node {
  int8_t k;
  int8_t src;
  int8_t list;
  int8_t bound;  // level index, -1 = none
  int8_t nops;
  int8_t raw;    // no ops on a raw list: a (bounded) CSR slice, nothing stored
  int8_t slot;   // scratch slot when materialized, -1 otherwise
  int8_t pad;
  Op ops[kMaxOps];
};

struct Program {
  int32_t depth;
  int32_t nnodes;
  int32_t nslots;        // materialized scratch slots per warp
  int8_t parent[kMaxLevels];
  uint8_t isect[kMaxLevels];
  uint8_t diff[kMaxLevels];
  int8_t cand[kMaxLevels];        // node holding C_i, 2 <= i <= depth-2
  int8_t node_begin[kMaxLevels];  // nodes built at loop k: [node_begin[k], node_end[k])
  int8_t node_end[kMaxLevels];
  int8_t unit_bound;              // level 1 requires v1 < v0
  // Leaf batching: when the leaf is `src (op) N(v_{n-2})`, the counts of all
  // siblings v_{n-2} in C_{n-2} are one edge count between two sets,
  //   sum_{x in C_{n-2}} |B & N(x)|,  B = the leaf's source set,
  // evaluated at loop n-3 (engine.cu, leaf_batch).
  int8_t batch;                   // 1 if the leaf can be batched
  int8_t batch_diff;              // leaf op is -N[x] (else & N(x))
  int8_t batch_yltx;              // leaf bound is x itself (y < x)
  int8_t batch_fixed_bound;       // leaf bound level < n-2 (fixed over siblings), -1 none
  // Clique plans (every source an intersection, depth >= 5): every level >= 2
  // lives inside U = N(v0) & N(v1), so a unit is counted on the local graph
  // of U as bitmaps (engine.cu, clique-local).
  int8_t clique;
  int8_t pad[2];
  Node leaf;                      // C_{depth-1}, counted not stored (depth >= 3)
  Node nodes[kMaxNodes];
};

// Returns "" on success, else a message (the plan violates compile_plan's
// invariants, plan.cpp:9-29).
inline std::string validate_plan(const smg_plan& p) {
  if (p.depth < 2 || p.depth > kMaxLevels) return "plan depth must be in 2..8";
  if (p.isect_mask[0] || p.diff_mask[0] || p.parent[0] != -1)
    return "level 0 must have no sources and no parent";
  for (int i = 1; i < p.depth; ++i) {
    const unsigned all = (1u << i) - 1u;
    if (p.isect_mask[i] & p.diff_mask[i]) return "level " + std::to_string(i) + ": source in both sets";
    if ((p.isect_mask[i] | p.diff_mask[i]) != all)
      return "level " + std::to_string(i) + ": sources must cover every earlier level";
    if (p.isect_mask[i] == 0) return "level " + std::to_string(i) + ": needs an intersect source";
    if (p.parent[i] < -1 || p.parent[i] >= i)
      return "level " + std::to_string(i) + ": restriction parent must be an earlier level";
  }
  return "";
}

// Effective bound of level i's prefix at loop k: nearest ancestor of p_i in the
// restriction chain with index <= k (v_{p} < v_{parent(p)} < ...).
inline int effective_bound(const smg_plan& p, int i, int k) {
  int q = p.parent[i];
  while (q > k) q = p.parent[q];
  return q;  // -1 if the chain ends before reaching <= k
}

inline bool same_node(const Node& a, const Node& b) {
  if (a.k != b.k || a.src != b.src || a.list != b.list || a.bound != b.bound || a.nops != b.nops)
    return false;
  for (int o = 0; o < a.nops; ++o)
    if (a.ops[o].level != b.ops[o].level || a.ops[o].mode != b.ops[o].mode) return false;
  return true;
}

inline std::string compile_program(const smg_plan& p, Program* out) {
  std::string err = validate_plan(p);
  if (!err.empty()) return err;
  Program pr;
  std::memset(&pr, 0, sizeof(pr));
  pr.depth = p.depth;
  for (int i = 0; i < kMaxLevels; ++i) {
    pr.parent[i] = i < p.depth ? p.parent[i] : -1;
    pr.isect[i] = i < p.depth ? p.isect_mask[i] : 0;
    pr.diff[i] = i < p.depth ? p.diff_mask[i] : 0;
    pr.cand[i] = -1;
  }
  pr.unit_bound = (p.depth >= 2 && p.parent[1] == 0) ? 1 : 0;
  pr.leaf.k = -1;
  const int n = p.depth;

  // Build each level's chain of prefix nodes, sharing identical ones.
  // Nodes are appended in increasing k within each chain; a final stable sort
  // by k keeps every node after its source.
  Node tmp[kMaxNodes];
  int nt = 0;
  for (int i = 2; i < n; ++i) {
    int j0 = 0;
    while (!((p.isect_mask[i] >> j0) & 1)) ++j0;
    int prev = -1;
    for (int k = j0; k <= i - 1; ++k) {
      Node nd;
      std::memset(&nd, 0, sizeof(nd));
      nd.k = static_cast<int8_t>(k);
      nd.bound = static_cast<int8_t>(effective_bound(p, i, k));
      nd.slot = -1;
      if (k == j0) {
        nd.src = -1;
        nd.list = static_cast<int8_t>(j0);
        for (int d = 0; d < j0; ++d) {  // all earlier sources are differences
          nd.ops[nd.nops].level = static_cast<int8_t>(d);
          nd.ops[nd.nops].mode = kOpDiff;
          ++nd.nops;
        }
      } else {
        nd.src = static_cast<int8_t>(prev);
        nd.list = -1;
        nd.ops[0].level = static_cast<int8_t>(k);
        nd.ops[0].mode = ((p.isect_mask[i] >> k) & 1) ? kOpIsect : kOpDiff;
        nd.nops = 1;
      }
      nd.raw = (nd.src < 0 && nd.nops == 0) ? 1 : 0;
      if (i == n - 1 && k == i - 1) {  // the leaf: counted, never stored
        pr.leaf = nd;
        break;
      }
      int id = -1;
      for (int t = 0; t < nt; ++t)
        if (same_node(tmp[t], nd)) id = t;
      if (id < 0) {
        if (nt == kMaxNodes) return "plan needs too many intermediate sets";
        tmp[nt] = nd;
        id = nt++;
      }
      prev = id;
      if (k == i - 1) pr.cand[i] = static_cast<int8_t>(id);
    }
  }
  // Order nodes by k (stable); remap ids.
  int order[kMaxNodes], remap[kMaxNodes];
  int no = 0;
  for (int k = 0; k < n; ++k) {
    pr.node_begin[k] = static_cast<int8_t>(no);
    for (int t = 0; t < nt; ++t)
      if (tmp[t].k == k) order[no++] = t;
    pr.node_end[k] = static_cast<int8_t>(no);
  }
  for (int t = 0; t < nt; ++t) remap[order[t]] = t;
  int slots = 0;
  for (int t = 0; t < nt; ++t) {
    Node nd = tmp[order[t]];
    if (nd.src >= 0) nd.src = static_cast<int8_t>(remap[nd.src]);
    nd.slot = nd.raw ? -1 : static_cast<int8_t>(slots++);
    pr.nodes[t] = nd;
  }
  if (pr.leaf.src >= 0) pr.leaf.src = static_cast<int8_t>(remap[pr.leaf.src]);
  for (int i = 0; i < kMaxLevels; ++i)
    if (pr.cand[i] >= 0) pr.cand[i] = static_cast<int8_t>(remap[pr.cand[i]]);
  pr.nnodes = nt;
  pr.nslots = slots;
  pr.batch_fixed_bound = -1;
  pr.clique = n >= 5 ? 1 : 0;
  for (int i = 1; i < n; ++i)
    if (p.diff_mask[i]) pr.clique = 0;
  if (n >= 4 && pr.leaf.src >= 0 && pr.leaf.nops == 1 && pr.leaf.ops[0].level == n - 2) {
    pr.batch = 1;
    pr.batch_diff = pr.leaf.ops[0].mode == kOpDiff ? 1 : 0;
    pr.batch_yltx = pr.leaf.bound == n - 2 ? 1 : 0;
    if (pr.leaf.bound >= 0 && pr.leaf.bound < n - 2) pr.batch_fixed_bound = pr.leaf.bound;
  }
  *out = pr;
  return "";
}

}  // namespace smg

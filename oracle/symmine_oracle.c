/*
 * symmine_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's matching path, used as the checker
 * for the CUDA engine.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product never does.
 * Pinned against the reference itself (oracle/_ref, compiled from
 * /root/reference) and the SPEC examples by tests/test_oracle.py and the
 * fixtures in tests/golden/.
 *
 *   intersect_into / difference_into   proj/include/symmine/set_ops.hpp:18-57
 *   build_level                        proj/src/engine.cpp:58-80
 *   taken                              proj/src/engine.cpp:82-87
 *   count_from / count_range           proj/src/engine.cpp:36-43, 89-115
 *   enumerate_from                     proj/src/engine.cpp:117-134
 *   checked_add                        proj/src/engine.cpp:13-19
 *   Graph::from_edges                  proj/src/graph.cpp:13-47
 *   orient_reindex                     proj/src/graph.cpp:137-161
 *
 * It also meters E: for every level build, the number of
 * elements below the level's bound in each source list.
 */
#include "symmine_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define LIMIT_NONE (((uint64_t)1) << 32)

/* set_ops.hpp:18-38 */
static size_t isect_into(const uint32_t* a, size_t na, const uint32_t* b, size_t nb,
                         uint64_t limit, uint32_t* out) {
  size_t i = 0, j = 0, k = 0;
  while (i < na && j < nb) {
    const uint32_t x = a[i];
    if ((uint64_t)x >= limit) break;
    const uint32_t y = b[j];
    if (x < y) {
      ++i;
    } else if (y < x) {
      ++j;
    } else {
      out[k++] = x;
      ++i;
      ++j;
    }
  }
  return k;
}

/* set_ops.hpp:40-57 */
static size_t diff_into(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, uint64_t limit,
                        uint32_t* out) {
  size_t i = 0, j = 0, k = 0;
  while (i < na) {
    const uint32_t x = a[i];
    if ((uint64_t)x >= limit) break;
    while (j < nb && b[j] < x) ++j;
    if (j < nb && b[j] == x) {
      ++i;
      continue;
    }
    out[k++] = x;
    ++i;
  }
  return k;
}

size_t oracle_intersect(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int has_bound,
                        uint32_t bound, uint32_t* out) {
  return isect_into(a, na, b, nb, has_bound ? (uint64_t)bound : LIMIT_NONE, out);
}

size_t oracle_difference(const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int has_bound,
                         uint32_t bound, uint32_t* out) {
  return diff_into(a, na, b, nb, has_bound ? (uint64_t)bound : LIMIT_NONE, out);
}

static size_t lower_bound_u32(const uint32_t* a, size_t n, uint64_t x) {
  size_t lo = 0, hi = n;
  while (lo < hi) {
    const size_t mid = lo + (hi - lo) / 2;
    if ((uint64_t)a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

typedef struct {
  const uint64_t* off;
  const uint32_t* adj;
  const smg_plan* plan;
  int depth;
  int use_bounds;
  int isrc[SMG_MAX_LEVELS][SMG_MAX_LEVELS];
  int nisrc[SMG_MAX_LEVELS];
  int dsrc[SMG_MAX_LEVELS][SMG_MAX_LEVELS];
  int ndsrc[SMG_MAX_LEVELS];
  uint32_t values[SMG_MAX_LEVELS];
  uint32_t* buffers[SMG_MAX_LEVELS];
  uint64_t elements;
  int overflow;
  /* enumeration */
  uint64_t limit, emitted;
  uint32_t* emit_out;
} Exec;

static void nbrs(const Exec* x, uint32_t v, const uint32_t** p, size_t* len) {
  *p = x->adj + x->off[v];
  *len = (size_t)(x->off[v + 1] - x->off[v]);
}

static int checked_add(Exec* x, uint64_t* acc, uint64_t add) {
  const uint64_t r = *acc + add;
  if (r < *acc) {
    x->overflow = 1;
    return 0;
  }
  *acc = r;
  return 1;
}

static int exec_init(Exec* x, const uint64_t* off, const uint32_t* adj, uint64_t n,
                     const smg_plan* plan) {
  memset(x, 0, sizeof(*x));
  x->off = off;
  x->adj = adj;
  x->plan = plan;
  x->depth = plan->depth;
  x->use_bounds = (plan->flags & SMG_PLAN_USE_BOUNDS) != 0;
  uint64_t maxd = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t d = off[v + 1] - off[v];
    if (d > maxd) maxd = d;
  }
  for (int i = 1; i < x->depth; ++i) {
    for (int j = 0; j < i; ++j) { /* compile_plan pushes sources in level order (plan.cpp:15-21) */
      if ((plan->isect_mask[i] >> j) & 1) x->isrc[i][x->nisrc[i]++] = j;
      if ((plan->diff_mask[i] >> j) & 1) x->dsrc[i][x->ndsrc[i]++] = j;
    }
    x->buffers[i] = (uint32_t*)malloc((maxd ? maxd : 1) * sizeof(uint32_t));
    if (!x->buffers[i]) return -1;
  }
  return 0;
}

static void exec_free(Exec* x) {
  for (int i = 1; i < SMG_MAX_LEVELS; ++i) free(x->buffers[i]);
}

/* engine.cpp:58-80, plus E metering */
static size_t build_level(Exec* x, int level) {
  const int par = x->plan->parent[level];
  uint64_t limit = LIMIT_NONE;
  if (x->use_bounds && par >= 0) limit = x->values[par];
  {
    const uint64_t beta = par >= 0 ? (uint64_t)x->values[par] : LIMIT_NONE;
    for (int j = 0; j < level; ++j) {
      const uint32_t* p;
      size_t len;
      nbrs(x, x->values[j], &p, &len);
      x->elements += lower_bound_u32(p, len, beta);
    }
  }
  uint32_t* out = x->buffers[level];
  const uint32_t *first, *second;
  size_t nfirst, nsecond, len;
  nbrs(x, x->values[x->isrc[level][0]], &first, &nfirst);
  if (x->nisrc[level] == 1) {
    len = diff_into(first, nfirst, NULL, 0, limit, out); /* bounded copy */
  } else {
    nbrs(x, x->values[x->isrc[level][1]], &second, &nsecond);
    len = isect_into(first, nfirst, second, nsecond, limit, out);
    for (int k = 2; k < x->nisrc[level]; ++k) {
      nbrs(x, x->values[x->isrc[level][k]], &second, &nsecond);
      len = isect_into(out, len, second, nsecond, LIMIT_NONE, out);
    }
  }
  for (int k = 0; k < x->ndsrc[level]; ++k) {
    nbrs(x, x->values[x->dsrc[level][k]], &second, &nsecond);
    len = diff_into(out, len, second, nsecond, LIMIT_NONE, out);
  }
  return len;
}

/* engine.cpp:82-87 */
static int taken(const Exec* x, uint32_t c, int level) {
  for (int j = 0; j < level; ++j)
    if (x->values[j] == c) return 1;
  return 0;
}

/* engine.cpp:89-115 */
static uint64_t count_from(Exec* x, int level) {
  if (level <= 0 || level >= SMG_MAX_LEVELS) return 0;
  const size_t len = build_level(x, level);
  const uint32_t* cands = x->buffers[level];
  const int par = x->plan->parent[level];
  const int check_parent = !x->use_bounds && par >= 0;
  const uint32_t parent_value = check_parent ? x->values[par] : 0;
  if (level == x->depth - 1) {
    uint64_t leaf = 0;
    for (size_t i = 0; i < len; ++i) {
      const uint32_t c = cands[i];
      if (check_parent && c >= parent_value) break;
      if (!taken(x, c, level)) ++leaf;
    }
    return leaf;
  }
  uint64_t total = 0;
  for (size_t i = 0; i < len; ++i) {
    const uint32_t c = cands[i];
    if (check_parent && c >= parent_value) break;
    if (taken(x, c, level)) continue;
    x->values[level] = c;
    if (!checked_add(x, &total, count_from(x, level + 1))) return total;
  }
  return total;
}

int oracle_count_range(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                       uint32_t lo, uint32_t hi, uint64_t* count, uint64_t* elements) {
  Exec x;
  if (exec_init(&x, off, adj, n, plan)) {
    exec_free(&x);
    return SMG_EIO;
  }
  uint64_t total = 0;
  for (uint64_t v = lo; v < hi && !x.overflow; ++v) { /* engine.cpp:36-43 */
    x.values[0] = (uint32_t)v;
    checked_add(&x, &total, count_from(&x, 1));
  }
  *count = total;
  if (elements) *elements = x.elements;
  const int ovf = x.overflow;
  exec_free(&x);
  return ovf ? SMG_EOVERFLOW : SMG_OK;
}

/* Level-1 units (v0, v1) given as CSR slot indices: the sum over a slot
 * sample of count_from(2) -- used for edge-sampled parity and CPU timing. */
int oracle_count_edges(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                       const uint64_t* slots, uint64_t num_slots, uint64_t* count,
                       uint64_t* elements) {
  Exec x;
  if (plan->depth < 3 || exec_init(&x, off, adj, n, plan)) return SMG_EINPUT;
  uint64_t total = 0;
  for (uint64_t s = 0; s < num_slots && !x.overflow; ++s) {
    const uint64_t e = slots[s];
    uint64_t lo = 0, hi = n; /* source vertex of slot e */
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) / 2;
      if (off[mid] <= e) lo = mid; else hi = mid;
    }
    x.values[0] = (uint32_t)lo;
    x.values[1] = adj[e];
    if (plan->parent[1] == 0 && !(x.values[1] < x.values[0])) continue;
    checked_add(&x, &total, count_from(&x, 2));
  }
  *count = total;
  if (elements) *elements = x.elements;
  const int ovf = x.overflow;
  exec_free(&x);
  return ovf ? SMG_EOVERFLOW : SMG_OK;
}

typedef struct {
  const uint64_t* off;
  const uint32_t* adj;
  uint64_t n;
  const smg_plan* plan;
  uint64_t next; /* atomic root cursor */
  uint64_t count;
  uint64_t elements;
  int status;
  pthread_mutex_t mu;
} Pool;

static void* worker(void* arg) {
  Pool* p = (Pool*)arg;
  Exec x;
  if (exec_init(&x, p->off, p->adj, p->n, p->plan)) {
    exec_free(&x);
    pthread_mutex_lock(&p->mu);
    p->status = SMG_EIO;
    pthread_mutex_unlock(&p->mu);
    return NULL;
  }
  uint64_t total = 0;
  const uint64_t chunk = 64;
  for (;;) {
    const uint64_t lo = __atomic_fetch_add(&p->next, chunk, __ATOMIC_RELAXED);
    if (lo >= p->n || x.overflow) break;
    const uint64_t hi = lo + chunk < p->n ? lo + chunk : p->n;
    for (uint64_t v = lo; v < hi && !x.overflow; ++v) {
      x.values[0] = (uint32_t)v;
      checked_add(&x, &total, count_from(&x, 1));
    }
  }
  pthread_mutex_lock(&p->mu);
  const uint64_t s = p->count + total;
  if (x.overflow || s < p->count) p->status = SMG_EOVERFLOW;
  p->count = s;
  p->elements += x.elements;
  pthread_mutex_unlock(&p->mu);
  exec_free(&x);
  return NULL;
}

/* Whole-graph count with `threads` workers pulling root chunks dynamically. */
int oracle_count(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                 int threads, uint64_t* count, uint64_t* elements) {
  if (threads < 1) threads = 1;
  Pool p;
  memset(&p, 0, sizeof(p));
  p.off = off;
  p.adj = adj;
  p.n = n;
  p.plan = plan;
  pthread_mutex_init(&p.mu, NULL);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, &p);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&p.mu);
  *count = p.count;
  if (elements) *elements = p.elements;
  return p.status;
}

/* engine.cpp:117-134 */
static int enumerate_from(Exec* x, int level) {
  const int depth = x->depth;
  if (level == depth) {
    if (x->emit_out)
      for (int i = 0; i < depth; ++i) x->emit_out[x->emitted * (uint64_t)depth + (uint64_t)i] = x->values[i];
    ++x->emitted;
    return !(x->limit && x->emitted >= x->limit);
  }
  if (level <= 0 || level >= SMG_MAX_LEVELS) return 0;
  const size_t len = build_level(x, level);
  const int par = x->plan->parent[level];
  const int check_parent = !x->use_bounds && par >= 0;
  const uint32_t parent_value = check_parent ? x->values[par] : 0;
  for (size_t i = 0; i < len; ++i) {
    const uint32_t c = x->buffers[level][i];
    if (check_parent && c >= parent_value) break;
    if (taken(x, c, level)) continue;
    x->values[level] = c;
    if (!enumerate_from(x, level + 1)) return 0;
  }
  return 1;
}

/* enumerate_instances (engine.cpp:181-191); limit 0 = unlimited here. */
int oracle_enumerate(const uint64_t* off, const uint32_t* adj, uint64_t n, const smg_plan* plan,
                     uint64_t limit, uint32_t* out, uint64_t* n_out) {
  Exec x;
  if (exec_init(&x, off, adj, n, plan)) {
    exec_free(&x);
    return SMG_EIO;
  }
  x.limit = limit;
  x.emit_out = out;
  for (uint64_t v = 0; v < n; ++v) {
    x.values[0] = (uint32_t)v;
    if (!enumerate_from(&x, 1)) break;
  }
  *n_out = x.emitted;
  exec_free(&x);
  return SMG_OK;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* graph.cpp:13-47.  adj must hold 2*m entries. */
int oracle_from_edges(uint64_t n, const uint32_t* pairs, uint64_t m, uint64_t* off, uint32_t* adj,
                      uint64_t* slots, uint64_t* dups, uint64_t* loops) {
  uint64_t* directed = (uint64_t*)malloc(sizeof(uint64_t) * (2 * m + 1));
  uint64_t nd = 0, nloops = 0;
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u >= n || v >= n) {
      free(directed);
      return SMG_EINPUT;
    }
    if (u == v) {
      ++nloops;
      continue;
    }
    directed[nd++] = ((uint64_t)u << 32) | v;
    directed[nd++] = ((uint64_t)v << 32) | u;
  }
  qsort(directed, nd, sizeof(uint64_t), cmp_u64);
  uint64_t w = 0;
  for (uint64_t i = 0; i < nd; ++i)
    if (i == 0 || directed[i] != directed[i - 1]) directed[w++] = directed[i];
  if (dups) *dups = (nd - w) / 2;
  if (loops) *loops = nloops;
  memset(off, 0, sizeof(uint64_t) * (n + 1));
  for (uint64_t i = 0; i < w; ++i) {
    ++off[(directed[i] >> 32) + 1];
    adj[i] = (uint32_t)directed[i];
  }
  for (uint64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  *slots = w;
  free(directed);
  return SMG_OK;
}

static const uint64_t* g_sort_off;
static int cmp_orient(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  const uint64_t dx = g_sort_off[x + 1] - g_sort_off[x], dy = g_sort_off[y + 1] - g_sort_off[y];
  if (dx != dy) return dx > dy ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* graph.cpp:137-161 (not thread-safe: qsort comparator uses a global). */
int oracle_orient(const uint64_t* off, const uint32_t* adj, uint64_t n, uint64_t* off_out,
                  uint32_t* adj_out, uint32_t* new_to_old) {
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
  uint32_t* old_to_new = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
  for (uint64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
  g_sort_off = off;
  qsort(order, n, sizeof(uint32_t), cmp_orient);
  for (uint64_t i = 0; i < n; ++i) old_to_new[order[i]] = (uint32_t)i;
  const uint64_t slots = off[n];
  uint32_t* pairs = (uint32_t*)malloc(sizeof(uint32_t) * (slots + 2));
  uint64_t m = 0;
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t i = off[u]; i < off[u + 1]; ++i)
      if (u < adj[i]) {
        pairs[2 * m] = old_to_new[u];
        pairs[2 * m + 1] = old_to_new[adj[i]];
        ++m;
      }
  uint64_t s2 = 0;
  const int rc = oracle_from_edges(n, pairs, m, off_out, adj_out, &s2, NULL, NULL);
  if (new_to_old) memcpy(new_to_old, order, sizeof(uint32_t) * n);
  free(pairs);
  free(order);
  free(old_to_new);
  return rc;
}

// graphgen.cpp -- host CSR toolkit: Graph::from_edges layout and the seeded
// BASELINE generators (see include/symmine_graph.h).  Parallel with OpenMP;
// results do not depend on the thread count.
#include <omp.h>
#include <parallel/algorithm>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/symmine_graph.h"

struct smg_csr {
  uint64_t n = 0;
  uint64_t max_degree = 0;
  std::vector<uint64_t> off;
  std::vector<uint32_t> adj;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}

inline uint64_t fmix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// i-th output of a splitmix64 stream whose state starts at key.
inline uint64_t rnd(uint64_t key, uint64_t i) { return fmix(key + (i + 1) * 0x9E3779B97F4A7C15ull); }
inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return fmix(seed * 0xD1B54A32D192ED03ull + stream * 0xA24BAED4963EE407ull + 0x632BE59BD9B4E019ull);
}
inline double unit01(uint64_t r) { return static_cast<double>(r >> 11) * 0x1.0p-53; }
inline uint32_t below32(uint32_t r, uint64_t n) {  // uniform in [0, n), n <= 2^32
  return static_cast<uint32_t>((static_cast<uint64_t>(r) * n) >> 32);
}

inline uint64_t canon(uint32_t u, uint32_t v) {
  return u < v ? (static_cast<uint64_t>(u) << 32) | v : (static_cast<uint64_t>(v) << 32) | u;
}

// CSR from sorted unique canonical keys (u < v).
smg_csr* csr_from_canonical(uint64_t n, const std::vector<uint64_t>& keys) {
  smg_csr* g = new smg_csr;
  g->n = n;
  g->off.assign(n + 1, 0);
  std::vector<uint64_t> deg(n, 0);
  for (uint64_t k : keys) {
    ++deg[k >> 32];
    ++deg[k & 0xffffffffu];
  }
  for (uint64_t v = 0; v < n; ++v) {
    g->off[v + 1] = g->off[v] + deg[v];
    g->max_degree = std::max(g->max_degree, deg[v]);
  }
  g->adj.resize(g->off[n]);
  // keys are sorted by (u, v): the forward halves arrive in order per u; the
  // backward halves (v -> u) arrive in increasing u per v.  Two passes keep
  // each list sorted without a per-list sort: first every backward neighbour
  // u < v, then every forward neighbour w > v.
  std::vector<uint64_t> fill(g->off.begin(), g->off.end() - 1);
  for (uint64_t k : keys) {
    const uint32_t u = static_cast<uint32_t>(k >> 32), v = static_cast<uint32_t>(k);
    g->adj[fill[v]++] = u;
  }
  for (uint64_t k : keys) {
    const uint32_t u = static_cast<uint32_t>(k >> 32), v = static_cast<uint32_t>(k);
    g->adj[fill[u]++] = v;
  }
  return g;
}

void sort_unique(std::vector<uint64_t>& keys) {
  __gnu_parallel::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
}

struct KeyIdx {
  uint64_t key;
  uint64_t idx;
  bool operator<(const KeyIdx& o) const { return key < o.key || (key == o.key && idx < o.idx); }
};

// The first m distinct keys of the draw stream i = 0,1,2,... (draws that
// return ~0 are rejected, e.g. self loops), exactly as a sequential
// reject-until-m loop would keep them.  Returned sorted by key.
template <class Draw>
int first_distinct(uint64_t m, double slack, Draw draw, std::vector<uint64_t>* out) {
  uint64_t total = static_cast<uint64_t>(static_cast<double>(m) * slack) + 1024;
  for (int attempt = 0; attempt < 12; ++attempt) {
    std::vector<KeyIdx> d(total);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < static_cast<int64_t>(total); ++i) d[i] = KeyIdx{draw(static_cast<uint64_t>(i)), static_cast<uint64_t>(i)};
    __gnu_parallel::sort(d.begin(), d.end());
    // keep the first occurrence of each key
    std::vector<KeyIdx> firsts;
    firsts.reserve(std::min<uint64_t>(total, m * 2));
    for (uint64_t i = 0; i < total; ++i) {
      if (d[i].key == ~0ull) break;
      if (i == 0 || d[i].key != d[i - 1].key) firsts.push_back(d[i]);
    }
    if (firsts.size() >= m) {
      std::nth_element(firsts.begin(), firsts.begin() + (m - 1), firsts.end(),
                       [](const KeyIdx& a, const KeyIdx& b) { return a.idx < b.idx; });
      out->resize(m);
      for (uint64_t i = 0; i < m; ++i) (*out)[i] = firsts[i].key;
      __gnu_parallel::sort(out->begin(), out->end());
      return 0;
    }
    total = total + total / 2;
  }
  return fail(2, "generator could not reach the requested distinct edge count");
}

// Seeded uniform permutation (Fisher-Yates); perm[old] = new.
std::vector<uint32_t> random_permutation(uint64_t n, uint64_t seed) {
  std::vector<uint32_t> p(n);
  std::iota(p.begin(), p.end(), 0u);
  const uint64_t key = stream_key(seed, 7);
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t r = rnd(key, n - i);
    const uint64_t j = static_cast<uint64_t>((static_cast<unsigned __int128>(r) * i) >> 64);
    std::swap(p[i - 1], p[j]);
  }
  return p;
}

void apply_permutation(std::vector<uint64_t>& keys, const std::vector<uint32_t>& perm) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(keys.size()); ++i) {
    const uint64_t k = keys[i];
    keys[i] = canon(perm[k >> 32], perm[k & 0xffffffffu]);
  }
  __gnu_parallel::sort(keys.begin(), keys.end());
}

}  // namespace

extern "C" {

const char* smg_graph_last_error(void) { return g_err.c_str(); }

int smg_csr_from_edges(uint64_t n, const uint32_t* pairs, uint64_t num_edges, smg_csr** out,
                       uint64_t* dups, uint64_t* loops) {
  if (!out) return fail(2, "null output");
  *out = nullptr;
  if (n >= (1ull << 32)) return fail(2, "vertex ids must fit in 32 bits");
  if (num_edges && !pairs) return fail(2, "null edge array");
  std::vector<uint64_t> keys;
  keys.reserve(num_edges);
  uint64_t nloops = 0;
  for (uint64_t i = 0; i < num_edges; ++i) {
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u >= n || v >= n) return fail(2, "edge endpoint out of range");  // graph.cpp:19
    if (u == v) {
      ++nloops;
      continue;
    }
    keys.push_back(canon(u, v));
  }
  const uint64_t before = keys.size();
  sort_unique(keys);
  if (dups) *dups = before - keys.size();
  if (loops) *loops = nloops;
  *out = csr_from_canonical(n, keys);
  return 0;
}

int smg_gen_er(uint64_t n, uint64_t m, uint64_t seed, smg_csr** out) {
  if (!out) return fail(2, "null output");
  *out = nullptr;
  if (n < 2 || n >= (1ull << 32)) return fail(2, "ER: n must be in 2..2^32-1");
  if (m > n * (n - 1) / 2) return fail(2, "ER: more edges than vertex pairs");
  const uint64_t key = stream_key(seed, 1);
  std::vector<uint64_t> keys;
  int rc = first_distinct(m, 1.02, [&](uint64_t i) -> uint64_t {
    const uint64_t r = rnd(key, i);
    const uint32_t u = below32(static_cast<uint32_t>(r >> 32), n);
    const uint32_t v = below32(static_cast<uint32_t>(r), n);
    return u == v ? ~0ull : canon(u, v);
  }, &keys);
  if (rc) return rc;
  *out = csr_from_canonical(n, keys);
  return 0;
}

int smg_gen_rmat(int scale, uint64_t edge_factor, double a, double b, double c, uint64_t seed,
                 smg_csr** out) {
  if (!out) return fail(2, "null output");
  *out = nullptr;
  if (scale < 1 || scale > 31) return fail(2, "RMAT: scale must be in 1..31");
  if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0) return fail(2, "RMAT: bad quadrant probabilities");
  const uint64_t n = 1ull << scale;
  const uint64_t draws = edge_factor * n;
  const uint64_t key = stream_key(seed, 2);
  const double ab = a + b, abc = a + b + c;
  std::vector<uint64_t> keys(draws);
#pragma omp parallel for schedule(static)
  for (int64_t d = 0; d < static_cast<int64_t>(draws); ++d) {
    uint32_t u = 0, v = 0;
    for (int bit = 0; bit < scale; ++bit) {
      const double r = unit01(rnd(key, static_cast<uint64_t>(d) * scale + bit));
      const uint32_t ub = r >= ab ? 1u : 0u;                       // quadrants c, d
      const uint32_t vb = (r >= a && r < ab) || r >= abc ? 1u : 0u;  // quadrants b, d
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    keys[d] = u == v ? ~0ull : canon(u, v);
  }
  sort_unique(keys);
  if (!keys.empty() && keys.back() == ~0ull) keys.pop_back();
  apply_permutation(keys, random_permutation(n, seed));
  *out = csr_from_canonical(n, keys);
  return 0;
}

int smg_gen_chung_lu(uint64_t n, uint64_t m, double gamma, double w_max, uint64_t seed,
                     smg_csr** out) {
  if (!out) return fail(2, "null output");
  *out = nullptr;
  if (n < 2 || n >= (1ull << 32)) return fail(2, "Chung-Lu: n must be in 2..2^32-1");
  if (gamma <= 1.0 || w_max <= 0) return fail(2, "Chung-Lu: need gamma > 1 and w_max > 0");
  if (m > n * (n - 1) / 2) return fail(2, "Chung-Lu: more edges than vertex pairs");
  // Expected degrees w_i = min(s * (i+1)^(-1/(gamma-1)), w_max) with the scale s
  // bisected so the mean equals 2m/n.
  const double alpha = 1.0 / (gamma - 1.0);
  std::vector<double> base(n);
  for (uint64_t i = 0; i < n; ++i) base[i] = std::pow(static_cast<double>(i + 1), -alpha);
  const double target = 2.0 * static_cast<double>(m) / static_cast<double>(n);
  auto mean_at = [&](double s) {
    double sum = 0;
    for (uint64_t i = 0; i < n; ++i) sum += std::min(s * base[i], w_max);
    return sum / static_cast<double>(n);
  };
  if (w_max < target) return fail(2, "Chung-Lu: w_max below the target mean degree");
  double lo = 0, hi = 1;
  while (mean_at(hi) < target) hi *= 2;
  for (int it = 0; it < 100; ++it) {
    const double mid = 0.5 * (lo + hi);
    (mean_at(mid) < target ? lo : hi) = mid;
  }
  std::vector<double> w(n);
  double total = 0;
  for (uint64_t i = 0; i < n; ++i) {
    w[i] = std::min(hi * base[i], w_max);
    total += w[i];
  }
  // Vose alias table for endpoint sampling proportional to w.
  std::vector<double> prob(n);
  std::vector<uint32_t> alias(n);
  {
    std::vector<double> scaled(n);
    std::vector<uint32_t> small, large;
    for (uint64_t i = 0; i < n; ++i) {
      scaled[i] = w[i] * static_cast<double>(n) / total;
      (scaled[i] < 1.0 ? small : large).push_back(static_cast<uint32_t>(i));
    }
    while (!small.empty() && !large.empty()) {
      const uint32_t s = small.back(), l = large.back();
      small.pop_back();
      prob[s] = scaled[s];
      alias[s] = l;
      scaled[l] = (scaled[l] + scaled[s]) - 1.0;
      if (scaled[l] < 1.0) {
        large.pop_back();
        small.push_back(l);
      }
    }
    for (uint32_t i : large) prob[i] = 1.0, alias[i] = i;
    for (uint32_t i : small) prob[i] = 1.0, alias[i] = i;
  }
  const uint64_t key = stream_key(seed, 3);
  auto endpoint = [&](uint64_t r) -> uint32_t {
    const uint32_t col = below32(static_cast<uint32_t>(r >> 32), n);
    const double coin = static_cast<double>(static_cast<uint32_t>(r)) * 0x1.0p-32;
    return coin < prob[col] ? col : alias[col];
  };
  std::vector<uint64_t> keys;
  int rc = first_distinct(m, 1.08, [&](uint64_t i) -> uint64_t {
    const uint32_t u = endpoint(rnd(key, 2 * i));
    const uint32_t v = endpoint(rnd(key, 2 * i + 1));
    return u == v ? ~0ull : canon(u, v);
  }, &keys);
  if (rc) return rc;
  apply_permutation(keys, random_permutation(n, seed));
  *out = csr_from_canonical(n, keys);
  return 0;
}

int smg_csr_orient(const smg_csr* g, smg_csr** out, uint32_t* new_to_old) {
  if (!g || !out) return fail(2, "null argument");
  const uint64_t n = g->n;
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    const uint64_t da = g->off[a + 1] - g->off[a], db = g->off[b + 1] - g->off[b];
    return da > db;  // stable: ties keep ascending old id (graph.cpp:141-144)
  });
  std::vector<uint32_t> old_to_new(n);
  for (uint64_t i = 0; i < n; ++i) old_to_new[order[i]] = static_cast<uint32_t>(i);
  std::vector<uint64_t> keys;
  keys.reserve(g->adj.size() / 2);
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i)
      if (u < g->adj[i]) keys.push_back(canon(old_to_new[u], old_to_new[g->adj[i]]));
  __gnu_parallel::sort(keys.begin(), keys.end());
  *out = csr_from_canonical(n, keys);
  if (new_to_old) std::memcpy(new_to_old, order.data(), n * sizeof(uint32_t));
  return 0;
}

int smg_csr_info(const smg_csr* g, uint64_t* n, uint64_t* slots, uint64_t* maxd) {
  if (!g) return fail(2, "null graph");
  if (n) *n = g->n;
  if (slots) *slots = g->adj.size();
  if (maxd) *maxd = g->max_degree;
  return 0;
}

const uint64_t* smg_csr_offsets(const smg_csr* g) { return g ? g->off.data() : nullptr; }
const uint32_t* smg_csr_adjacency(const smg_csr* g) { return g ? g->adj.data() : nullptr; }
void smg_csr_free(smg_csr* g) { delete g; }

}  // extern "C"

/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this; the product library never does.
 *
 * A plain-C restatement of the reference's ground-truth path (arXiv 1602.04478
 * artifact, /root/reference/proj):
 *   - splitmix64 / derive_seed / uniform_below ...... include/motif/rng.hpp:9-31
 *   - mt19937_64 (std::mt19937_64, the reference's engine; standard MT19937-64)
 *   - random_coloring ............................... src/graph.cpp:142-151
 *   - DataGraph::from_edges normalisation ........... src/graph.cpp:14-44
 *   - degree_rank ................................... src/graph.cpp:123-134
 *   - brute_matches / brute_colorful backtracker .... src/oracle.cpp:11-105
 *   - automorphism_count ............................ src/estimate.cpp:14-45
 *   - normalization_factor (k^k/k!) ................. src/estimate.cpp:47-79
 *   - coefficient_of_variation ...................... src/estimate.cpp:81-94
 *
 * Pinned by tests/test_oracle.py against (a) the known answers in the
 * reference's own tests (tests/test_oracle.cpp, test_engine.cpp, test_graph.cpp,
 * test_estimator.cpp) and (b) the compiled reference (oracle/_ref) on seeded
 * random inputs, plus the committed fixtures in tests/golden/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

uint64_t or_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t or_derive_seed(uint64_t master, uint64_t stream) {
  return or_splitmix64(master ^ or_splitmix64(stream + 0x632be59bd9b4e019ULL));
}

/* MT19937-64 exactly as std::mt19937_64 (w=64,n=312,m=156,r=31). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static uint64_t uniform_below(mt64* s, uint64_t bound) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t x;
  do {
    x = mt64_next(s);
  } while (x >= limit);
  return x % bound;
}

/* First `count` raw outputs (used to pin the generator against std::mt19937_64). */
void or_mt64_stream(uint64_t seed, uint64_t count, uint64_t* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = mt64_next(&s);
}

/* random_coloring: colours 1..k, i.i.d., vertex order 0..n-1. Returns -1 if k out of range. */
int or_random_coloring(uint32_t n, int k, uint64_t seed, uint8_t* chi) {
  if (k < 1 || k > 32) return -1;
  mt64 s;
  mt64_seed(&s, seed);
  for (uint32_t v = 0; v < n; ++v) chi[v] = (uint8_t)(1 + uniform_below(&s, (uint64_t)k));
  return 0;
}

/* ------------------------------------------------------------- graph.cpp */

static int cmp_pair(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* Normalise an edge list (orient, sort, dedupe, drop loops) into CSR.
 * offsets must hold n+1 entries, adj 2*m entries.  Returns the number of
 * undirected edges kept. */
uint64_t or_build_csr(uint32_t n, const uint32_t* eu, const uint32_t* ev, uint64_t m,
                      uint64_t* offsets, uint32_t* adj) {
  uint64_t* pk = (uint64_t*)malloc((m ? m : 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    uint32_t a = eu[i], b = ev[i];
    if (a > b) { uint32_t t = a; a = b; b = t; }
    pk[i] = ((uint64_t)a << 32) | b;
  }
  qsort(pk, m, sizeof(uint64_t), cmp_pair);
  uint64_t kept = 0;
  for (uint64_t i = 0; i < m; ++i) {
    if (i > 0 && pk[i] == pk[i - 1]) continue;
    if ((uint32_t)(pk[i] >> 32) == (uint32_t)pk[i]) continue;
    pk[kept++] = pk[i];
  }
  memset(offsets, 0, (size_t)(n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < kept; ++i) {
    offsets[(pk[i] >> 32) + 1]++;
    offsets[(uint32_t)pk[i] + 1]++;
  }
  for (uint32_t v = 0; v < n; ++v) offsets[v + 1] += offsets[v];
  uint64_t* cur = (uint64_t*)malloc((size_t)(n ? n : 1) * sizeof(uint64_t));
  memcpy(cur, offsets, (size_t)n * sizeof(uint64_t));
  for (uint64_t i = 0; i < kept; ++i) {
    uint32_t a = (uint32_t)(pk[i] >> 32), b = (uint32_t)pk[i];
    adj[cur[a]++] = b;
    adj[cur[b]++] = a;
  }
  for (uint32_t v = 0; v < n; ++v)
    qsort(adj + offsets[v], offsets[v + 1] - offsets[v], sizeof(uint32_t), cmp_u32);
  free(cur);
  free(pk);
  return kept;
}

/* degree_rank: position in the sort by (degree asc, id asc). */
static const uint64_t* g_rank_off;
static int cmp_by_degree(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  const uint64_t dx = g_rank_off[x + 1] - g_rank_off[x], dy = g_rank_off[y + 1] - g_rank_off[y];
  if (dx != dy) return dx < dy ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

void or_degree_rank(uint32_t n, const uint64_t* offsets, uint32_t* rank) {
  uint32_t* order = (uint32_t*)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
  for (uint32_t v = 0; v < n; ++v) order[v] = v;
  g_rank_off = offsets;
  qsort(order, n, sizeof(uint32_t), cmp_by_degree);
  for (uint32_t p = 0; p < n; ++p) rank[order[p]] = p;
  free(order);
}

/* ------------------------------------------------------------ oracle.cpp */

typedef struct {
  uint32_t n;
  const uint64_t* off;
  const uint32_t* adj;
  const uint8_t* chi; /* NULL: colours ignored */
  int k;
  int order[32];
  int nplaced[32];
  int placed[32][32];
  uint32_t image[32];
  uint8_t* used;
  uint32_t used_colors;
  uint64_t steps, limit, count;
  int over_budget;
} bt_state;

static int has_edge(const bt_state* s, uint32_t u, uint32_t v) {
  uint64_t lo = s->off[u], hi = s->off[u + 1];
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (s->adj[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo < s->off[u + 1] && s->adj[lo] == v;
}

static void bt_run(bt_state* s, int slot) {
  if (s->over_budget) return;
  if (slot == s->k) { s->count++; return; }
  for (uint32_t v = 0; v < s->n; ++v) {
    if (++s->steps > s->limit) { s->over_budget = 1; return; }
    if (s->used[v]) continue;
    uint32_t bit = 0;
    if (s->chi) {
      bit = 1u << (s->chi[v] - 1);
      if (s->used_colors & bit) continue;
    }
    int ok = 1;
    for (int i = 0; i < s->nplaced[slot] && ok; ++i)
      if (!has_edge(s, s->image[s->placed[slot][i]], v)) ok = 0;
    if (!ok) continue;
    s->image[slot] = v;
    s->used[v] = 1;
    s->used_colors |= bit;
    bt_run(s, slot + 1);
    s->used[v] = 0;
    s->used_colors &= ~bit;
    if (s->over_budget) return;
  }
}

/* Number of (colourful if chi != NULL) injective edge-preserving maps of the
 * query (k nodes, qm edges as pairs) into the CSR graph.  Returns 0 on success,
 * 5 on budget exhaustion (the reference's BudgetError exit code). */
int or_brute_count(uint32_t n, const uint64_t* off, const uint32_t* adj, const uint8_t* chi, int k,
                   const int32_t* qedges, int qm, uint64_t budget, uint64_t* out) {
  bt_state s;
  memset(&s, 0, sizeof(s));
  s.n = n; s.off = off; s.adj = adj; s.chi = chi; s.k = k; s.limit = budget;
  /* query adjacency (sorted neighbour lists, as QueryGraph::neighbors) */
  int nb[32][32], deg[32];
  memset(deg, 0, sizeof(deg));
  for (int i = 0; i < qm; ++i) {
    int a = qedges[2 * i], b = qedges[2 * i + 1];
    nb[a][deg[a]++] = b;
    nb[b][deg[b]++] = a;
  }
  for (int v = 0; v < k; ++v)
    qsort(nb[v], deg[v], sizeof(int), cmp_u32);
  /* DFS assignment order (stack-based, as oracle.cpp:240-257) */
  int seen[32] = {0}, stack[64], sp = 0, no = 0;
  for (int st = 0; st < k; ++st) {
    if (seen[st]) continue;
    stack[sp++] = st;
    seen[st] = 1;
    while (sp) {
      int v = stack[--sp];
      s.order[no++] = v;
      for (int i = 0; i < deg[v]; ++i) {
        int w = nb[v][i];
        if (!seen[w]) { seen[w] = 1; stack[sp++] = w; }
      }
    }
  }
  int slot_of[32];
  for (int i = 0; i < k; ++i) slot_of[s.order[i]] = i;
  for (int i = 0; i < k; ++i) {
    int v = s.order[i];
    for (int j = 0; j < deg[v]; ++j)
      if (slot_of[nb[v][j]] < i) s.placed[i][s.nplaced[i]++] = slot_of[nb[v][j]];
  }
  s.used = (uint8_t*)calloc(n ? n : 1, 1);
  bt_run(&s, 0);
  free(s.used);
  *out = s.count;
  return s.over_budget ? 5 : 0;
}

/* ---------------------------------------------------------- estimate.cpp */

static int q_adjacent(const uint32_t* qadj, int a, int b) { return (qadj[a] >> b) & 1u; }

static void aut_rec(const uint32_t* qadj, int k, int* perm, uint32_t used, int depth, uint64_t* c) {
  if (depth == k) { (*c)++; return; }
  for (int img = 0; img < k; ++img) {
    if ((used >> img) & 1u) continue;
    int ok = 1;
    for (int j = 0; j < depth && ok; ++j)
      if (q_adjacent(qadj, depth, j) != q_adjacent(qadj, img, perm[j])) ok = 0;
    if (!ok) continue;
    perm[depth] = img;
    aut_rec(qadj, k, perm, used | (1u << img), depth + 1, c);
  }
}

/* Returns 0 and the automorphism count, or 8 (SpecError) for k > 10. */
int or_automorphism_count(int k, const int32_t* qedges, int qm, uint64_t* out) {
  if (k > 10) return 8;
  uint32_t qadj[32] = {0};
  for (int i = 0; i < qm; ++i) {
    qadj[qedges[2 * i]] |= 1u << qedges[2 * i + 1];
    qadj[qedges[2 * i + 1]] |= 1u << qedges[2 * i];
  }
  int perm[32];
  *out = 0;
  aut_rec(qadj, k, perm, 0, 0, out);
  return 0;
}

/* k^k/k! — exact reduced rational in 128-bit while it fits, else long double. */
double or_normalization_factor(int k) {
  unsigned __int128 num = 1, den = 1;
  int exact = 1;
  for (int i = 1; i <= k && exact; ++i) {
    unsigned __int128 a = (unsigned)k, b = (unsigned)i, x, y, t;
    x = a; y = den; while (y) { t = x % y; x = y; y = t; }
    a /= x; den /= x;
    x = num; y = b; while (y) { t = x % y; x = y; y = t; }
    num /= x; b /= x;
    if (num > (~(unsigned __int128)0) / a) { exact = 0; break; }
    num *= a;
    den *= b;
  }
  if (exact) return (double)num / (double)den;
  long double f = 1.0L;
  for (int i = 1; i <= k; ++i) f *= (long double)k / i;
  return (double)f;
}

/* population variance / mean; 0 for <= 1 sample or an all-zero sample. */
double or_coefficient_of_variation(const uint64_t* c, uint64_t n) {
  if (n <= 1) return 0.0;
  long double sum = 0, sq = 0;
  for (uint64_t i = 0; i < n; ++i) {
    long double x = (long double)c[i];
    sum += x;
    sq += x * x;
  }
  if (sum == 0) return 0.0;
  long double mean = sum / (long double)n;
  return (double)((sq / (long double)n - mean * mean) / mean);
}

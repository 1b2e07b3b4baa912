#include "graph.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <fstream>
#include <numeric>
#include <random>
#include <sstream>
#include <thread>
#include <unordered_set>

#include "errors.hpp"

namespace mb {

namespace {

int host_threads() {
  unsigned t = std::thread::hardware_concurrency();
  return t == 0 ? 1 : static_cast<int>(std::min(t, 64u));
}

// Static block split of [0, count) over the host threads.
template <class F>
void parallel_blocks(uint64_t count, F&& fn) {
  const int nt = static_cast<int>(std::min<uint64_t>(host_threads(), std::max<uint64_t>(count, 1)));
  if (nt <= 1 || count < 4096) {
    fn(0, count, 0);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 0; t < nt; ++t) {
    const uint64_t lo = count * t / nt, hi = count * (t + 1) / nt;
    ts.emplace_back([&, lo, hi, t] { fn(lo, hi, t); });
  }
  for (auto& th : ts) th.join();
}

}  // namespace

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t derive_seed(uint64_t master, uint64_t stream) {
  return splitmix64(master ^ splitmix64(stream + 0x632be59bd9b4e019ULL));
}

// Bucket the oriented pairs by their smaller endpoint (counting sort), sort
// each bucket, drop duplicates and loops, then scatter both orientations.
// Because buckets are visited in increasing order, every row comes out
// already sorted: row v receives its smaller neighbours first (from earlier
// buckets) and then its own bucket in ascending order.
CsrGraph CsrGraph::from_edges(uint32_t n, std::vector<std::pair<uint32_t, uint32_t>>& edges,
                              LoadStats* st) {
  const uint64_t m_in = edges.size();
  std::vector<uint64_t> start(static_cast<size_t>(n) + 1, 0);
  uint64_t loops = 0;
  for (auto& e : edges) {
    if (e.first > e.second) std::swap(e.first, e.second);
    if (e.second >= n) fail(kSpec, "edge endpoint out of range");
    if (e.first == e.second) {
      ++loops;
      continue;
    }
    start[e.first + 1]++;
  }
  for (uint32_t v = 0; v < n; ++v) start[v + 1] += start[v];
  std::vector<uint32_t> bucket(start[n]);
  {
    std::vector<uint64_t> cur(start.begin(), start.end() - 1);
    for (const auto& e : edges)
      if (e.first != e.second) bucket[cur[e.first]++] = e.second;
  }
  edges.clear();
  edges.shrink_to_fit();
  std::vector<uint64_t> kept(static_cast<size_t>(n) + 1, 0);
  parallel_blocks(n, [&](uint64_t lo, uint64_t hi, int) {
    for (uint64_t v = lo; v < hi; ++v) {
      auto b = bucket.begin() + start[v], e = bucket.begin() + start[v + 1];
      std::sort(b, e);
      kept[v + 1] = static_cast<uint64_t>(std::unique(b, e) - b);
    }
  });
  CsrGraph g;
  g.n = n;
  std::vector<uint64_t> deg(n, 0);
  for (uint32_t a = 0; a < n; ++a) {
    deg[a] += kept[a + 1];
    for (uint64_t i = 0; i < kept[a + 1]; ++i) deg[bucket[start[a] + i]]++;
    g.m += kept[a + 1];
  }
  g.offsets.assign(static_cast<size_t>(n) + 1, 0);
  for (uint32_t v = 0; v < n; ++v) g.offsets[v + 1] = g.offsets[v] + deg[v];
  g.adj.resize(2 * g.m);
  std::vector<uint64_t> cur(g.offsets.begin(), g.offsets.end() - 1);
  for (uint32_t a = 0; a < n; ++a) {
    for (uint64_t i = 0; i < kept[a + 1]; ++i) {
      const uint32_t b = bucket[start[a] + i];
      g.adj[cur[a]++] = b;
      g.adj[cur[b]++] = a;
    }
  }
  if (st) {
    st->self_loops_dropped = loops;
    st->duplicates_dropped = m_in - loops - g.m;
  }
  return g;
}

CsrGraph CsrGraph::from_arrays(uint32_t n, const uint32_t* eu, const uint32_t* ev, uint64_t m,
                               LoadStats* st) {
  std::vector<std::pair<uint32_t, uint32_t>> e(m);
  for (uint64_t i = 0; i < m; ++i) e[i] = {eu[i], ev[i]};
  return from_edges(n, e, st);
}

bool CsrGraph::has_edge(uint32_t u, uint32_t v) const {
  auto b = adj.begin() + offsets[u], e = adj.begin() + offsets[u + 1];
  return std::binary_search(b, e, v);
}

void CsrGraph::validate() const {
  uint64_t deg_sum = 0;
  for (uint32_t v = 0; v < n; ++v) {
    for (uint64_t i = offsets[v]; i < offsets[v + 1]; ++i) {
      const uint32_t w = adj[i];
      if (w == v) fail(kSpec, "self loop survived normalization");
      if (i > offsets[v] && w <= adj[i - 1]) fail(kSpec, "neighbor list not strictly sorted");
      if (!has_edge(w, v)) fail(kSpec, "adjacency not symmetric");
    }
    deg_sum += offsets[v + 1] - offsets[v];
  }
  if (deg_sum != 2 * m) fail(kSpec, "degree sum != 2m");
}

// Same grammar and error text as the reference loader (graph.cpp:65-111).
CsrGraph load_edge_list(std::istream& in, LoadStats* st) {
  std::vector<std::pair<uint32_t, uint32_t>> edges;
  uint32_t max_id = 0;
  bool any = false;
  std::string line;
  uint64_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    std::istringstream ls(line);
    long long u, v;
    if (!(ls >> u)) continue;
    if (!(ls >> v)) fail(kParse, "line " + std::to_string(line_no) + ": expected \"u v\" pair");
    std::string extra;
    if (ls >> extra)
      fail(kParse, "line " + std::to_string(line_no) + ": trailing token '" + extra + "'");
    if (u < 0 || v < 0) fail(kParse, "line " + std::to_string(line_no) + ": negative vertex id");
    if (u > 0xFFFFFFFELL || v > 0xFFFFFFFELL)
      fail(kParse, "line " + std::to_string(line_no) + ": vertex id exceeds 32 bits");
    max_id = std::max({max_id, static_cast<uint32_t>(u), static_cast<uint32_t>(v)});
    any = true;
    edges.emplace_back(static_cast<uint32_t>(u), static_cast<uint32_t>(v));
  }
  if (in.bad()) fail(kParse, "I/O error while reading edge list");
  return CsrGraph::from_edges(any ? max_id + 1 : 0, edges, st);
}

CsrGraph load_edge_list_file(const std::string& path, LoadStats* st) {
  std::ifstream f(path);
  if (!f) fail(kParse, "cannot open graph file: " + path);
  return load_edge_list(f, st);
}

std::string serialize_edge_list(const CsrGraph& g) {
  std::ostringstream out;
  for (uint32_t u = 0; u < g.n; ++u)
    for (uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i)
      if (u < g.adj[i]) out << u << ' ' << g.adj[i] << '\n';
  return out.str();
}

std::vector<uint32_t> degree_rank(const CsrGraph& g) {
  // Counting sort by degree; ids ascend inside each degree class, so the
  // position is exactly the (degree, id) lexicographic rank.
  uint32_t maxd = 0;
  for (uint32_t v = 0; v < g.n; ++v) maxd = std::max(maxd, g.degree(v));
  std::vector<uint64_t> cnt(static_cast<size_t>(maxd) + 2, 0);
  for (uint32_t v = 0; v < g.n; ++v) cnt[g.degree(v) + 1]++;
  for (size_t d = 1; d < cnt.size(); ++d) cnt[d] += cnt[d - 1];
  std::vector<uint32_t> rank(g.n);
  for (uint32_t v = 0; v < g.n; ++v) rank[v] = static_cast<uint32_t>(cnt[g.degree(v)]++);
  return rank;
}

std::vector<uint8_t> random_coloring(uint32_t n, int k, uint64_t seed) {
  if (k < 1) fail(kSpec, "color count must be >= 1");
  if (k > 32) fail(kSpec, "color count > 32 unsupported (32-bit signatures)");
  std::vector<uint8_t> chi(n);
  std::mt19937_64 rng(seed);
  const uint64_t bound = static_cast<uint64_t>(k);
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  for (uint32_t v = 0; v < n; ++v) {
    uint64_t x;
    do {
      x = rng();
    } while (x >= limit);
    chi[v] = static_cast<uint8_t>(1 + x % bound);
  }
  return chi;
}

// ---------------------------------------------------------------- generators

namespace {

struct Stream {  // counter-based splitmix64 stream
  uint64_t s;
  uint64_t next() { return splitmix64(s++); }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// Seeded Fisher-Yates relabelling of vertex ids.
std::vector<uint32_t> seeded_permutation(uint32_t n, uint64_t seed) {
  std::vector<uint32_t> p(n);
  std::iota(p.begin(), p.end(), 0);
  Stream r{derive_seed(seed, 0x5eed)};
  for (uint32_t i = n; i > 1; --i) {
    const uint32_t j = static_cast<uint32_t>(r.next() % i);
    std::swap(p[i - 1], p[j]);
  }
  return p;
}

}  // namespace

CsrGraph gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed) {
  if (n < 2) fail(kSpec, "G(n,m) needs n >= 2");
  const uint64_t pairs = static_cast<uint64_t>(n) * (n - 1) / 2;
  if (m > pairs) fail(kSpec, "G(n,m): m exceeds the number of vertex pairs");
  std::unordered_set<uint64_t> seen;
  seen.reserve(m * 2);
  std::vector<std::pair<uint32_t, uint32_t>> edges;
  edges.reserve(m);
  Stream r{derive_seed(seed, 1)};
  while (edges.size() < m) {
    uint32_t u = static_cast<uint32_t>(r.next() % n), v = static_cast<uint32_t>(r.next() % n);
    if (u == v) continue;
    if (u > v) std::swap(u, v);
    if (seen.insert((static_cast<uint64_t>(u) << 32) | v).second) edges.emplace_back(u, v);
  }
  return CsrGraph::from_edges(n, edges);
}

CsrGraph gen_chung_lu(uint32_t n, double gamma, double avg_degree, double max_w, uint64_t seed) {
  if (n < 2 || !(gamma > 1.0) || !(avg_degree > 0)) fail(kSpec, "bad Chung-Lu parameters");
  if (max_w <= 0) max_w = std::sqrt(static_cast<double>(n) * avg_degree);
  const double expo = -1.0 / (gamma - 1.0);
  std::vector<double> raw(n);
  for (uint32_t i = 0; i < n; ++i) raw[i] = std::pow(static_cast<double>(i) + 1.0, expo);
  auto capped_mean = [&](double c) {
    long double s = 0;
    for (uint32_t i = 0; i < n; ++i) s += std::min(c * raw[i], max_w);
    return static_cast<double>(s / n);
  };
  double lo = 0, hi = 1;
  while (capped_mean(hi) < avg_degree) {
    hi *= 2;
    if (hi > 1e300) fail(kSpec, "Chung-Lu: average degree unreachable under the cap");
  }
  for (int it = 0; it < 100; ++it) {
    const double mid = 0.5 * (lo + hi);
    (capped_mean(mid) < avg_degree ? lo : hi) = mid;
  }
  std::vector<double> w(n);  // non-increasing in i
  long double W = 0;
  for (uint32_t i = 0; i < n; ++i) {
    w[i] = std::min(hi * raw[i], max_w);
    W += w[i];
  }
  const double Wd = static_cast<double>(W);
  // Exact independent-edge sampling by geometric skipping over the
  // weight-sorted sequence (each row its own counter-based stream).
  const int nt = host_threads();
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> part(nt);
  std::atomic<uint32_t> next_row{0};
  std::vector<std::thread> ts;
  for (int t = 0; t < nt; ++t) {
    ts.emplace_back([&, t] {
      auto& out = part[t];
      for (;;) {
        const uint32_t u0 = next_row.fetch_add(256);
        if (u0 >= n) break;
        const uint32_t u1 = std::min<uint32_t>(n, u0 + 256);
        for (uint32_t u = u0; u < u1; ++u) {
          Stream r{derive_seed(seed, u)};
          uint64_t v = static_cast<uint64_t>(u) + 1;
          double p = v < n ? std::min(1.0, w[u] * w[v] / Wd) : 0.0;
          while (v < n && p > 0) {
            if (p < 1.0) {
              const double x = r.unit();
              const double skip = std::floor(std::log1p(-x) / std::log1p(-p));
              if (!(skip < static_cast<double>(n))) break;
              v += static_cast<uint64_t>(skip);
            }
            if (v >= n) break;
            const double q = std::min(1.0, w[u] * w[v] / Wd);
            if (r.unit() < q / p) out.emplace_back(u, static_cast<uint32_t>(v));
            p = q;
            ++v;
          }
        }
      }
    });
  }
  for (auto& th : ts) th.join();
  const auto perm = seeded_permutation(n, seed);
  std::vector<std::pair<uint32_t, uint32_t>> edges;
  size_t total = 0;
  for (auto& p : part) total += p.size();
  edges.reserve(total);
  for (auto& p : part) {
    for (auto& e : p) edges.emplace_back(perm[e.first], perm[e.second]);
    p.clear();
    p.shrink_to_fit();
  }
  return CsrGraph::from_edges(n, edges);
}

CsrGraph gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed) {
  if (scale < 1 || scale > 31 || edge_factor < 1) fail(kSpec, "bad R-MAT parameters");
  const uint32_t n = 1u << scale;
  const uint64_t m = static_cast<uint64_t>(edge_factor) << scale;
  // thresholds on 32-bit draws for quadrants a | b | c | d
  const double ab = a + b, abc = a + b + c;
  if (!(a >= 0 && b >= 0 && c >= 0 && abc <= 1.0)) fail(kSpec, "bad R-MAT probabilities");
  const uint64_t ta = static_cast<uint64_t>(a * 4294967296.0);
  const uint64_t tab = static_cast<uint64_t>(ab * 4294967296.0);
  const uint64_t tabc = static_cast<uint64_t>(abc * 4294967296.0);
  std::vector<std::pair<uint32_t, uint32_t>> edges(m);
  parallel_blocks(m, [&](uint64_t lo, uint64_t hi, int) {
    for (uint64_t e = lo; e < hi; ++e) {
      uint64_t ctr = derive_seed(seed, e);
      uint32_t u = 0, v = 0;
      for (int l = 0; l < scale; l += 2) {
        const uint64_t x = splitmix64(ctr++);
        for (int h = 0; h < 2 && l + h < scale; ++h) {
          const uint64_t d = (x >> (32 * h)) & 0xFFFFFFFFULL;
          const uint32_t bit = 1u << (scale - 1 - (l + h));
          if (d < ta) {
          } else if (d < tab) {
            v |= bit;
          } else if (d < tabc) {
            u |= bit;
          } else {
            u |= bit;
            v |= bit;
          }
        }
      }
      edges[e] = {u, v};
    }
  });
  return CsrGraph::from_edges(n, edges);
}

}  // namespace mb

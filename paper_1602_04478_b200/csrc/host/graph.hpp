// Host-side data graph for the B200 colour-coding engine.
//
// Mirrors the reference interface (include/motif/graph.hpp):
//   DataGraph::from_edges  (graph.hpp:20)  -> CsrGraph::from_edges
//   load_edge_list         (graph.hpp:47)  -> load_edge_list
//   serialize_edge_list    (graph.hpp:51)  -> serialize_edge_list
//   degree_rank            (graph.hpp:68)  -> degree_rank
//   random_coloring        (graph.hpp:85)  -> random_coloring
// The layout is what the device wants: 64-bit row offsets (graphs beyond
// 2^32 half-edges fit), 32-bit sorted neighbour ids, and a per-vertex rank
// array that is uploaded once and shared by every colouring.
#pragma once

#include <cstdint>
#include <istream>
#include <string>
#include <vector>

namespace mb {

struct LoadStats {
  uint64_t self_loops_dropped = 0;
  uint64_t duplicates_dropped = 0;
};

struct CsrGraph {
  uint32_t n = 0;
  uint64_t m = 0;                 // undirected edges, each once
  std::vector<uint64_t> offsets;  // n + 1
  std::vector<uint32_t> adj;      // 2m, sorted per row

  // Orients, sorts, dedupes and drops self loops (graph.cpp:14-44 semantics).
  // `edges` holds (u,v) pairs; it is consumed.
  static CsrGraph from_edges(uint32_t n, std::vector<std::pair<uint32_t, uint32_t>>& edges,
                             LoadStats* st = nullptr);
  static CsrGraph from_arrays(uint32_t n, const uint32_t* eu, const uint32_t* ev, uint64_t m,
                              LoadStats* st = nullptr);

  uint32_t degree(uint32_t v) const { return static_cast<uint32_t>(offsets[v + 1] - offsets[v]); }
  bool has_edge(uint32_t u, uint32_t v) const;
  void validate() const;  // throws SpecError
};

CsrGraph load_edge_list(std::istream& in, LoadStats* st = nullptr);
CsrGraph load_edge_list_file(const std::string& path, LoadStats* st = nullptr);
std::string serialize_edge_list(const CsrGraph& g);

// rank[v] = position in the sort by (degree asc, id asc).
std::vector<uint32_t> degree_rank(const CsrGraph& g);

// chi[v] in 1..k, std::mt19937_64(seed) + rejection draw (rng.hpp:111),
// bit-identical to the reference's random_coloring.
std::vector<uint8_t> random_coloring(uint32_t n, int k, uint64_t seed);

uint64_t splitmix64(uint64_t x);
uint64_t derive_seed(uint64_t master, uint64_t stream);

// ---- seeded synthetic inputs (BASELINE.json configs) -----------------------
// Erdos-Renyi G(n, m): exactly m distinct undirected non-loop edges.
CsrGraph gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed);
// Chung-Lu with power-law expected degrees w_i ~ (i+1)^(-1/(gamma-1)), scaled so
// the mean expected degree is `avg_degree` after capping at `max_w`
// (max_w <= 0: sqrt(n * avg_degree) = sqrt(2m)); exact independent-edge
// sampling (p = min(1, w_u w_v / W)) by geometric skipping; ids shuffled by seed.
CsrGraph gen_chung_lu(uint32_t n, double gamma, double avg_degree, double max_w, uint64_t seed);
// R-MAT with 2^scale vertices and edge_factor * 2^scale generated edges,
// symmetrised and deduplicated, self loops dropped.
CsrGraph gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed);

}  // namespace mb

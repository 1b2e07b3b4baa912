// Query graphs and treewidth-2 decomposition plans.
//
// Mirrors the reference planner (include/motif/query.hpp):
//   QueryGraph::from_edges / parse_query     query.hpp:25,36
//   Block (LeafEdge | Cycle)                  query.hpp:43-62
//   DecompositionTree (+ canonical)           query.hpp:64-80
//   find_blocks / contract_block              query.hpp:85,89   (paper §4.1)
//   enumerate_trees / plan_score / select_plan query.hpp:94-108 (paper §6)
// Plans are tiny (k <= 32 nodes); this is host-only code.  The canonical
// serialisation is byte-identical to the reference's so plans can be
// compared across implementations (tests/golden/plans.json).
#pragma once

#include <cstdint>
#include <istream>
#include <string>
#include <vector>

namespace mb {

struct QEdge {
  int a = -1, b = -1;  // a < b
  int child = -1;      // annotating block, -1 for an original query edge
  bool child_fwd = true;
};

struct Query {
  int k = 0;
  std::vector<QEdge> edges;
  uint32_t live = 0;            // bitmask of nodes still present
  std::vector<int> node_child;  // per node, -1 if none

  static Query from_edges(int k, const std::vector<std::pair<int, int>>& e);
  bool alive(int v) const { return (live >> v) & 1u; }
  int alive_count() const { return __builtin_popcount(live); }
  int edge_index(int a, int b) const;
  std::vector<int> nbrs(int v) const;  // sorted
  bool connected() const;
};

Query parse_query(std::istream& in);
Query load_query_file(const std::string& path);

enum class BlockKind { Leaf, Cycle };

struct Block {
  int id = -1;
  BlockKind kind = BlockKind::Cycle;
  std::vector<int> nodes;     // cycle order; leaf: {boundary, leaf}
  std::vector<int> boundary;  // key order, 0..2 nodes
  std::vector<int> node_child;
  std::vector<int> edge_child;
  std::vector<char> edge_fwd;

  int size() const { return static_cast<int>(nodes.size()); }
  int edge_count() const { return kind == BlockKind::Cycle ? size() : 1; }
  int pos(int node) const;
  std::string canonical() const;
};

struct Plan {
  int k = 0;
  std::vector<Block> blocks;
  int root = -1;
  bool singleton_root = false;
  int singleton_node = -1;
  std::vector<int> parent;

  std::vector<int> bottom_up() const;
  std::string canonical() const;
  uint32_t subquery_nodes(int b) const;
};

std::vector<Block> find_blocks(const Query& q);
Block contract_block(Query& q, const Block& b, int new_id);
std::vector<Plan> enumerate_plans(const Query& q, size_t max_trees = 10000);

struct PlanScore {
  int max_cycle_length = 0;
  int boundary_total = 0;
  int annotation_total = 0;
  bool operator<(const PlanScore& o) const;
};
PlanScore plan_score(const Plan& p);
size_t select_plan(const std::vector<Plan>& plans);  // index of the chosen plan

}  // namespace mb

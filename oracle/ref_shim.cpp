// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the *unmodified* reference library (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libmotif_ref.so).  It lets pytest, __graft_entry__.smoke() and
// bench.py's `--impl reference` / cpu_baseline legs drive the reference's own
// public API:
//   DataGraph::from_edges        include/motif/graph.hpp:20
//   random_coloring              include/motif/graph.hpp:85
//   degree_rank                  include/motif/graph.hpp:68
//   QueryGraph::from_edges       include/motif/query.hpp:25
//   enumerate_trees/select_plan  include/motif/query.hpp:94,108
//   count_colorful               include/motif/engine.hpp:121
//   parallel_count / Partition   include/motif/runtime.hpp:87
//   brute_colorful               include/motif/oracle.hpp:195
//   estimate                     include/motif/estimate.hpp:34
// Nothing here re-implements the algorithm; it only marshals plain arrays.
#include <atomic>
#include <cstdint>
#include <mutex>
#include <thread>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "motif/engine.hpp"
#include "motif/errors.hpp"
#include "motif/estimate.hpp"
#include "motif/graph.hpp"
#include "motif/oracle.hpp"
#include "motif/query.hpp"
#include "motif/runtime.hpp"

namespace {

struct RefGraph {
  motif::DataGraph g;
  motif::VertexOrdering ord;
};

struct RefPlan {
  motif::QueryGraph q;
  std::vector<motif::DecompositionTree> trees;
  size_t selected = 0;
};

thread_local std::string g_err;

int classify(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const motif::ParseError*>(&e)) return 2;
  if (dynamic_cast<const motif::TreewidthError*>(&e)) return 3;
  if (dynamic_cast<const motif::OverflowError*>(&e)) return 4;
  if (dynamic_cast<const motif::BudgetError*>(&e)) return 5;
  if (dynamic_cast<const motif::SchemaError*>(&e)) return 6;
  if (dynamic_cast<const motif::ContractError*>(&e)) return 7;
  if (dynamic_cast<const motif::SpecError*>(&e)) return 8;
  return 1;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_graph_new(uint32_t n, const uint32_t* eu, const uint32_t* ev, uint64_t m, void** out) {
  return guarded([&] {
    std::vector<std::pair<uint32_t, uint32_t>> e(m);
    for (uint64_t i = 0; i < m; ++i) e[i] = {eu[i], ev[i]};
    auto* rg = new RefGraph;
    rg->g = motif::DataGraph::from_edges(n, std::move(e));
    rg->ord = motif::degree_rank(rg->g);
    *out = rg;
  });
}

void ref_graph_free(void* g) { delete static_cast<RefGraph*>(g); }

uint64_t ref_graph_num_edges(void* g) { return static_cast<RefGraph*>(g)->g.num_edges(); }

// Normalised CSR (offsets n+1, adj 2m) as the reference built it.
int ref_graph_csr(void* gp, uint64_t* offsets, uint32_t* adj) {
  return guarded([&] {
    const auto& g = static_cast<RefGraph*>(gp)->g;
    uint64_t pos = 0;
    for (uint32_t v = 0; v < g.num_vertices(); ++v) {
      offsets[v] = pos;
      for (uint32_t w : g.neighbors(v)) adj[pos++] = w;
    }
    offsets[g.num_vertices()] = pos;
  });
}

int ref_graph_ranks(void* gp, uint32_t* rank) {
  return guarded([&] {
    auto* rg = static_cast<RefGraph*>(gp);
    for (uint32_t v = 0; v < rg->g.num_vertices(); ++v) rank[v] = rg->ord.rank(v);
  });
}

int ref_random_coloring(void* gp, int k, uint64_t seed, uint8_t* out) {
  return guarded([&] {
    motif::Coloring c = motif::random_coloring(static_cast<RefGraph*>(gp)->g, k, seed);
    std::memcpy(out, c.chi.data(), c.chi.size());
  });
}

int ref_plan_new(int k, const int32_t* edges, int m, uint64_t max_trees, void** out) {
  return guarded([&] {
    std::vector<std::pair<int, int>> e;
    for (int i = 0; i < m; ++i) e.emplace_back(edges[2 * i], edges[2 * i + 1]);
    auto p = std::make_unique<RefPlan>();
    p->q = motif::QueryGraph::from_edges(k, e);
    p->trees = motif::enumerate_trees(p->q, max_trees);
    const motif::DecompositionTree* best = &motif::select_plan(p->trees);
    p->selected = static_cast<size_t>(best - p->trees.data());
    *out = p.release();
  });
}

void ref_plan_free(void* p) { delete static_cast<RefPlan*>(p); }

int ref_plan_num_trees(void* p) { return static_cast<int>(static_cast<RefPlan*>(p)->trees.size()); }

// Canonical serialisation of tree `idx` (-1: the selected plan).
int ref_plan_canonical(void* pp, int idx, char* buf, int len) {
  return guarded([&] {
    auto* p = static_cast<RefPlan*>(pp);
    const auto& t = p->trees[idx < 0 ? p->selected : static_cast<size_t>(idx)];
    std::string s = t.canonical();
    if (static_cast<int>(s.size()) + 1 > len) throw motif::SpecError("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int ref_count_colorful(void* gp, const uint8_t* chi, int k, void* pp, int tree_idx, int engine,
                       int workers, uint64_t* out) {
  return guarded([&] {
    auto* rg = static_cast<RefGraph*>(gp);
    auto* p = static_cast<RefPlan*>(pp);
    motif::Coloring c;
    c.k = k;
    c.chi.assign(chi, chi + rg->g.num_vertices());
    const auto& tree = p->trees[tree_idx < 0 ? p->selected : static_cast<size_t>(tree_idx)];
    const auto kind = engine == 0 ? motif::EngineKind::PS : motif::EngineKind::DB;
    if (workers <= 1) {
      *out = motif::count_colorful(rg->g, c, rg->ord, tree, kind);
    } else {
      *out = motif::parallel_count(rg->g, c, tree, kind,
                                   motif::Partition(rg->g.num_vertices(), workers));
    }
  });
}

// count_colorful for `nc` colourings (n bytes each) on up to `threads` host
// threads, one colouring per thread at a time (workers > 1: each colouring
// through parallel_count's BSP executor, runtime.cpp:311-324) (the reference's estimate()
// parallelises the same way, estimate.cpp:108-117).  Returns the first error.
int ref_count_batch(void* gp, const uint8_t* chis, int nc, int k, void* pp, int engine, int threads,
                    int workers, uint64_t* out) {
  auto* rg = static_cast<RefGraph*>(gp);
  auto* p = static_cast<RefPlan*>(pp);
  const uint32_t n = rg->g.num_vertices();
  std::atomic<int> next{0}, rc{0};
  std::string err;
  std::mutex mu;
  auto worker = [&] {
    for (;;) {
      const int c = next.fetch_add(1);
      if (c >= nc) return;
      try {
        motif::Coloring col;
        col.k = k;
        col.chi.assign(chis + static_cast<size_t>(c) * n, chis + static_cast<size_t>(c + 1) * n);
        const auto kind = engine == 0 ? motif::EngineKind::PS : motif::EngineKind::DB;
        if (workers <= 1)
          out[c] = motif::count_colorful(rg->g, col, rg->ord, p->trees[p->selected], kind);
        else  // the reference's BSP executor: one colouring over `workers` OpenMP workers
          out[c] = motif::parallel_count(rg->g, col, p->trees[p->selected], kind, motif::Partition(n, workers));
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(mu);
        if (!rc) {
          rc = classify(e);
          err = g_err;
        }
      }
    }
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < std::max(1, std::min(threads, nc)); ++t) ts.emplace_back(worker);
  for (auto& t : ts) t.join();
  if (rc) g_err = err;
  return rc;
}

// JoinStats::ops of the serial engine (the reference's load metric).
int ref_count_ops(void* gp, const uint8_t* chi, int k, void* pp, int engine, uint64_t* count,
                  uint64_t* ops) {
  return guarded([&] {
    auto* rg = static_cast<RefGraph*>(gp);
    auto* p = static_cast<RefPlan*>(pp);
    motif::Coloring c;
    c.k = k;
    c.chi.assign(chi, chi + rg->g.num_vertices());
    motif::JoinStats st;
    *count = motif::count_colorful(rg->g, c, rg->ord, p->trees[p->selected],
                                   engine == 0 ? motif::EngineKind::PS : motif::EngineKind::DB,
                                   &st);
    *ops = st.ops;
  });
}

int ref_brute_colorful(void* gp, void* pp, const uint8_t* chi, int k, uint64_t budget,
                       uint64_t* out) {
  return guarded([&] {
    auto* rg = static_cast<RefGraph*>(gp);
    auto* p = static_cast<RefPlan*>(pp);
    motif::Coloring c;
    c.k = k;
    c.chi.assign(chi, chi + rg->g.num_vertices());
    *out = motif::brute_colorful(rg->g, p->q, c, motif::OracleBudget{budget});
  });
}

int ref_brute_matches(void* gp, void* pp, uint64_t budget, uint64_t* out) {
  return guarded([&] {
    *out = motif::brute_matches(static_cast<RefGraph*>(gp)->g, static_cast<RefPlan*>(pp)->q,
                                motif::OracleBudget{budget});
  });
}

int ref_automorphism_count(void* pp, uint64_t* out) {
  return guarded([&] { *out = motif::automorphism_count(static_cast<RefPlan*>(pp)->q); });
}

double ref_normalization_factor(int k) { return motif::normalization_factor(k); }

int ref_estimate(void* gp, void* pp, int engine, uint64_t trials, uint64_t seed,
                 uint64_t* per_trial, double* mean, double* cv, double* subgraph) {
  return guarded([&] {
    auto* rg = static_cast<RefGraph*>(gp);
    auto* p = static_cast<RefPlan*>(pp);
    auto r = motif::estimate(rg->g, p->q, p->trees[p->selected],
                             engine == 0 ? motif::EngineKind::PS : motif::EngineKind::DB, trials,
                             seed);
    std::memcpy(per_trial, r.per_trial_colorful.data(), trials * sizeof(uint64_t));
    *mean = r.mean_estimate;
    *cv = r.cv;
    *subgraph = r.subgraph_estimate;
  });
}

}  // extern "C"

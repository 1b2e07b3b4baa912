// extern "C" boundary of libmotif_b200.so (declarations: include/motif_b200.h).
#include "../../include/motif_b200.h"

#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "engine/engine.hpp"
#include "host/errors.hpp"
#include "host/estimate.hpp"
#include "host/graph.hpp"
#include "host/plan.hpp"

struct mb_graph {
  mb::CsrGraph g;
  std::unique_ptr<mb::GpuEngine> eng;
  const mb_plan* bound = nullptr;
  int bound_tree = -1;
  uint64_t bound_version = 0;
  bool timing = false;
};

struct mb_plan {
  mb::Query q;
  std::vector<mb::Plan> trees;
  int selected = 0;
  int in_use = 0;
  uint64_t version = 0;
};

namespace {

thread_local std::string g_err;
uint64_t g_plan_version = 0;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return mb::kOk;
  } catch (const mb::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return mb::kInternal;
  }
}

mb::GpuEngine& engine_for(mb_graph* g, mb_plan* p) {
  if (!g->eng) {
    // created on the caller's current device (torch.cuda.set_device(local_rank)
    // under torchrun); every later call runs there and restores the caller's
    g->eng = std::make_unique<mb::GpuEngine>(g->g, -1);
    g->eng->enable_timing(g->timing);
    g->bound = nullptr;
  }
  if (g->bound != p || g->bound_tree != p->in_use || g->bound_version != p->version) {
    g->eng->bind_plan(p->trees[p->in_use], p->q.k);
    g->bound = p;
    g->bound_tree = p->in_use;
    g->bound_version = p->version;
  }
  return *g->eng;
}

void finish_plan(mb_plan* p, uint64_t max_trees) {
  p->trees = mb::enumerate_plans(p->q, max_trees);
  p->selected = static_cast<int>(mb::select_plan(p->trees));
  p->in_use = p->selected;
  p->version = ++g_plan_version;
}

}  // namespace

extern "C" {

const char* mb_last_error(void) { return g_err.c_str(); }
const char* mb_version(void) { return "motif_b200 0.1 (sm_100a)"; }

int mb_graph_from_edges(uint32_t n, const uint32_t* eu, const uint32_t* ev, uint64_t m, mb_graph** out,
                        uint64_t* loops, uint64_t* dups) {
  return guarded([&] {
    mb::LoadStats st;
    auto g = std::make_unique<mb_graph>();
    g->g = mb::CsrGraph::from_arrays(n, eu, ev, m, &st);
    if (loops) *loops = st.self_loops_dropped;
    if (dups) *dups = st.duplicates_dropped;
    *out = g.release();
  });
}

int mb_graph_load_edge_list(const char* path, mb_graph** out, uint64_t* loops, uint64_t* dups) {
  return guarded([&] {
    mb::LoadStats st;
    auto g = std::make_unique<mb_graph>();
    g->g = mb::load_edge_list_file(path, &st);
    if (loops) *loops = st.self_loops_dropped;
    if (dups) *dups = st.duplicates_dropped;
    *out = g.release();
  });
}

int mb_graph_gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed, mb_graph** out) {
  return guarded([&] {
    auto g = std::make_unique<mb_graph>();
    g->g = mb::gen_erdos_renyi(n, m, seed);
    *out = g.release();
  });
}

int mb_graph_gen_chung_lu(uint32_t n, double gamma, double avg_degree, double max_w, uint64_t seed,
                          mb_graph** out) {
  return guarded([&] {
    auto g = std::make_unique<mb_graph>();
    g->g = mb::gen_chung_lu(n, gamma, avg_degree, max_w, seed);
    *out = g.release();
  });
}

int mb_graph_gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed, mb_graph** out) {
  return guarded([&] {
    auto g = std::make_unique<mb_graph>();
    g->g = mb::gen_rmat(scale, edge_factor, a, b, c, seed);
    *out = g.release();
  });
}

void mb_graph_free(mb_graph* g) { delete g; }
uint32_t mb_graph_num_vertices(const mb_graph* g) { return g->g.n; }
uint64_t mb_graph_num_edges(const mb_graph* g) { return g->g.m; }

int mb_graph_csr(const mb_graph* g, uint64_t* offsets, uint32_t* adj) {
  return guarded([&] {
    std::memcpy(offsets, g->g.offsets.data(), (g->g.n + 1) * sizeof(uint64_t));
    std::memcpy(adj, g->g.adj.data(), g->g.adj.size() * sizeof(uint32_t));
  });
}

int mb_graph_edges(const mb_graph* g, uint32_t* eu, uint32_t* ev) {
  return guarded([&] {
    uint64_t w = 0;
    for (uint32_t u = 0; u < g->g.n; ++u)
      for (uint64_t i = g->g.offsets[u]; i < g->g.offsets[u + 1]; ++i)
        if (u < g->g.adj[i]) eu[w] = u, ev[w] = g->g.adj[i], ++w;
  });
}

int mb_graph_degree_rank(const mb_graph* g, uint32_t* rank) {
  return guarded([&] {
    const auto r = mb::degree_rank(g->g);
    std::memcpy(rank, r.data(), r.size() * sizeof(uint32_t));
  });
}

int mb_graph_validate(const mb_graph* g) {
  return guarded([&] { g->g.validate(); });
}

int mb_random_coloring(uint32_t n, int k, uint64_t seed, uint8_t* chi) {
  return guarded([&] {
    const auto c = mb::random_coloring(n, k, seed);
    std::memcpy(chi, c.data(), n);
  });
}

uint64_t mb_derive_seed(uint64_t master, uint64_t stream) { return mb::derive_seed(master, stream); }

int mb_plan_create(int k, const int32_t* edges, int m, uint64_t max_trees, mb_plan** out) {
  return guarded([&] {
    std::vector<std::pair<int, int>> e;
    for (int i = 0; i < m; ++i) e.emplace_back(edges[2 * i], edges[2 * i + 1]);
    auto p = std::make_unique<mb_plan>();
    p->q = mb::Query::from_edges(k, e);
    finish_plan(p.get(), max_trees ? max_trees : 10000);
    *out = p.release();
  });
}

int mb_plan_load_query(const char* path, uint64_t max_trees, mb_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<mb_plan>();
    p->q = mb::load_query_file(path);
    finish_plan(p.get(), max_trees ? max_trees : 10000);
    *out = p.release();
  });
}

void mb_plan_free(mb_plan* p) { delete p; }
int mb_plan_k(const mb_plan* p) { return p->q.k; }
int mb_plan_num_trees(const mb_plan* p) { return static_cast<int>(p->trees.size()); }
int mb_plan_selected(const mb_plan* p) { return p->selected; }

int mb_plan_use_tree(mb_plan* p, int idx) {
  return guarded([&] {
    if (idx < 0 || idx >= static_cast<int>(p->trees.size())) mb::fail(mb::kSpec, "tree index out of range");
    p->in_use = idx;
  });
}

int mb_plan_canonical(const mb_plan* p, int idx, char* buf, int len) {
  return guarded([&] {
    const int i = idx < 0 ? p->in_use : idx;
    if (i >= static_cast<int>(p->trees.size())) mb::fail(mb::kSpec, "tree index out of range");
    const std::string s = p->trees[i].canonical();
    if (static_cast<int>(s.size()) + 1 > len) mb::fail(mb::kSpec, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int mb_plan_score(const mb_plan* p, int idx, int* score3) {
  return guarded([&] {
    const int i = idx < 0 ? p->in_use : idx;
    if (i >= static_cast<int>(p->trees.size())) mb::fail(mb::kSpec, "tree index out of range");
    const auto s = mb::plan_score(p->trees[i]);
    score3[0] = s.max_cycle_length, score3[1] = s.boundary_total, score3[2] = s.annotation_total;
  });
}

int mb_count_colorful(mb_graph* g, mb_plan* p, const uint8_t* chi, int ncol, int engine, uint64_t* out) {
  return guarded([&] {
    if (engine != 0 && engine != 1) mb::fail(mb::kSpec, "engine must be 0 (PS) or 1 (DB)");
    engine_for(g, p).count(chi, ncol, true, out);
  });
}

// colourings per device call of the seeded entry points
static int seed_batch(uint32_t n) {
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(256, (1ull << 30) / std::max<uint32_t>(n, 1))));
}

int mb_count_colorful_seeds(mb_graph* g, mb_plan* p, const uint64_t* seeds, int ncol, int engine,
                            uint64_t* out) {
  return guarded([&] {
    if (engine != 0 && engine != 1) mb::fail(mb::kSpec, "engine must be 0 (PS) or 1 (DB)");
    if (ncol < 0) mb::fail(mb::kSpec, "negative colouring count");
    auto& eng = engine_for(g, p);
    // the colourings are generated on the device (GpuEngine::count_seeds), in
    // bounded batches: at most 256 colourings or 1 GB of colours per call
    eng.count_seeds_batched(seeds, static_cast<uint64_t>(ncol), seed_batch(g->g.n), out);
  });
}

int mb_device_random_colorings(mb_graph* g, int k, const uint64_t* seeds, int ncol, uint64_t limit, uint8_t* out) {
  return guarded([&] {
    if (ncol < 0) mb::fail(mb::kSpec, "negative colouring count");
    if (!g->eng) {
      g->eng = std::make_unique<mb::GpuEngine>(g->g, -1);
      g->eng->enable_timing(g->timing);
      g->bound = nullptr;
    }
    g->eng->random_colorings(k, seeds, ncol, limit, out);
  });
}

int mb_count_colorful_shard(mb_graph* g, mb_plan* p, const uint8_t* chi, int ncol, int engine, int rank, int world,
                            uint64_t* partial, int* split) {
  return guarded([&] {
    if (engine != 0 && engine != 1) mb::fail(mb::kSpec, "engine must be 0 (PS) or 1 (DB)");
    if (world < 1 || rank < 0 || rank >= world) mb::fail(mb::kSpec, "shard rank out of range");
    auto& eng = engine_for(g, p);
    if (split) *split = eng.root_shardable() ? 1 : 0;
    eng.set_shard(static_cast<uint32_t>(rank), static_cast<uint32_t>(world));
    try {
      eng.count(chi, ncol, true, partial);
    } catch (...) {
      eng.set_shard(0, 1);
      throw;
    }
    eng.set_shard(0, 1);
  });
}

int mb_count_colorful_sharded(mb_graph* g, mb_plan* p, const uint8_t* chi, int ncol, int engine, int rank, int world,
                              mb_allgather_fn allgather, void* ctx, uint64_t* partial, int* split) {
  return guarded([&] {
    if (engine != 0 && engine != 1) mb::fail(mb::kSpec, "engine must be 0 (PS) or 1 (DB)");
    if (world < 1 || rank < 0 || rank >= world) mb::fail(mb::kSpec, "shard rank out of range");
    if (!allgather && world > 1) mb::fail(mb::kSpec, "sharded count needs an all-gather callback");
    auto& eng = engine_for(g, p);
    eng.set_shard(static_cast<uint32_t>(rank), static_cast<uint32_t>(world));
    if (world > 1)
      eng.set_exchange([allgather, ctx](void* buf, uint64_t bytes, void* stream) {
        if (allgather(ctx, buf, bytes, stream) != 0) mb::fail(mb::kCuda, "table exchange (all-gather callback) failed");
      });
    auto reset = [&] {
      eng.set_exchange(nullptr);
      eng.set_shard(0, 1);
    };
    try {
      if (split) *split = eng.root_shardable() ? 1 : 0;
      eng.count(chi, ncol, true, partial);
    } catch (...) {
      reset();
      throw;
    }
    reset();
  });
}

int mb_count_colorful_device(mb_graph* g, mb_plan* p, const uint8_t* chi_dev, int ncol, uint64_t* out) {
  return guarded([&] { engine_for(g, p).count(chi_dev, ncol, false, out); });
}

int mb_automorphism_count(int k, const int32_t* edges, int m, uint64_t* out) {
  return guarded([&] {
    std::vector<std::pair<int, int>> e;
    for (int i = 0; i < m; ++i) e.emplace_back(edges[2 * i], edges[2 * i + 1]);
    *out = mb::automorphism_count(mb::Query::from_edges(k, e));
  });
}

double mb_normalization_factor(int k) {
  try {
    return mb::normalization_factor(k);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 0.0;
  }
}

int mb_estimate_from_counts(int k, uint64_t aut, const uint64_t* per_trial, uint64_t trials, double* mean,
                            double* cv, double* subgraph) {
  return guarded([&] {
    if (trials < 1) mb::fail(mb::kSpec, "trials must be >= 1");
    const double norm = mb::normalization_factor(k);
    long double sum = 0;
    for (uint64_t i = 0; i < trials; ++i) sum += static_cast<long double>(per_trial[i]);
    *mean = static_cast<double>(norm * (sum / static_cast<long double>(trials)));
    *cv = mb::coefficient_of_variation(std::vector<uint64_t>(per_trial, per_trial + trials));
    *subgraph = *mean / static_cast<double>(aut);
  });
}

double mb_coefficient_of_variation(const uint64_t* counts, uint64_t n) {
  return mb::coefficient_of_variation(std::vector<uint64_t>(counts, counts + n));
}

int mb_estimate(mb_graph* g, mb_plan* p, int engine, uint64_t trials, uint64_t seed, uint64_t* per_trial,
                double* mean, double* cv, uint64_t* aut, double* subgraph) {
  return guarded([&] {
    if (trials < 1) mb::fail(mb::kSpec, "trials must be >= 1");
    if (engine != 0 && engine != 1) mb::fail(mb::kSpec, "engine must be 0 (PS) or 1 (DB)");
    const double norm = mb::normalization_factor(p->q.k);
    auto& eng = engine_for(g, p);
    const uint32_t n = g->g.n;
    // Trial i's colouring is random_coloring(n, k, derive_seed(seed, i))
    // (estimate.cpp:108-117), generated on the device in bounded batches
    std::vector<uint64_t> seeds(trials);
    for (uint64_t i = 0; i < trials; ++i) seeds[i] = mb::derive_seed(seed, i);
    eng.count_seeds_batched(seeds.data(), trials, seed_batch(n), per_trial);
    (void)norm;
    *aut = mb::automorphism_count(p->q);
    const int rc = mb_estimate_from_counts(p->q.k, *aut, per_trial, trials, mean, cv, subgraph);
    if (rc) mb::fail(static_cast<mb::Status>(rc), g_err);
  });
}

int mb_partition_block(uint32_t n, int p, int w, uint32_t* begin, uint32_t* size) {
  return guarded([&] {
    if (p < 1) mb::fail(mb::kSpec, "worker count must be >= 1");
    if (static_cast<uint32_t>(p) > n) mb::fail(mb::kSpec, "more workers than vertices");
    if (w < 0 || w >= p) mb::fail(mb::kSpec, "worker index out of range");
    const uint32_t base = n / p, rem = n % p;
    const uint32_t big = std::min<uint32_t>(w, rem);
    *begin = big * (base + 1) + (static_cast<uint32_t>(w) - big) * base;
    *size = base + (static_cast<uint32_t>(w) < rem ? 1 : 0);
  });
}

int mb_partition_owner(uint32_t n, int p, uint32_t v, int* owner) {
  return guarded([&] {
    if (p < 1) mb::fail(mb::kSpec, "worker count must be >= 1");
    if (static_cast<uint32_t>(p) > n) mb::fail(mb::kSpec, "more workers than vertices");
    if (v >= n) mb::fail(mb::kSpec, "vertex out of range");
    const uint32_t base = n / p, rem = n % p;
    const uint64_t big_span = static_cast<uint64_t>(base + 1) * rem;
    *owner = v < big_span ? static_cast<int>(v / (base + 1)) : static_cast<int>(rem + (v - big_span) / base);
  });
}

int mb_engine_enable_timing(mb_graph* g, int on) {
  return guarded([&] {
    g->timing = on != 0;
    if (g->eng) g->eng->enable_timing(g->timing);
  });
}

int mb_engine_kernel_timing(mb_graph* g, int idx, char* name, int len, double* ms, uint64_t* launches,
                            uint64_t* bytes) {
  return guarded([&] {
    if (!g->eng) mb::fail(mb::kSpec, "no engine");
    const auto t = g->eng->kernel_timings();
    if (idx < 0 || idx >= static_cast<int>(t.size())) mb::fail(mb::kSpec, "timing index out of range");
    std::snprintf(name, len, "%s", t[idx].name.c_str());
    *ms = t[idx].ms;
    *launches = t[idx].launches;
    *bytes = t[idx].bytes;
  });
}

void* mb_engine_stream(mb_graph* g) { return g->eng ? g->eng->stream() : nullptr; }

int mb_engine_device(const mb_graph* g) { return g->eng ? g->eng->device() : -1; }

double mb_engine_prep_ms(mb_graph* g) { return g->eng ? g->eng->stats().prep_ms : 0.0; }

uint64_t mb_engine_launches(mb_graph* g) { return g->eng ? g->eng->launches() : 0; }
uint64_t mb_engine_exchanged_bytes(mb_graph* g) { return g->eng ? g->eng->exchanged_bytes() : 0; }

int mb_engine_stats(mb_graph* g, uint64_t* triangles, uint64_t* table_bytes, uint64_t* dp_updates) {
  return guarded([&] {
    if (!g->eng) mb::fail(mb::kSpec, "no engine");
    const auto& s = g->eng->stats();
    *triangles = s.triangles;
    *table_bytes = s.table_bytes;
    *dp_updates = s.dp_updates;
  });
}

int mb_engine_reset_derived(mb_graph* g) {
  return guarded([&] {
    if (g->eng) g->eng->reset_derived();
  });
}

int mb_engine_release(mb_graph* g) {
  return guarded([&] {
    g->eng.reset();
    g->bound = nullptr;
  });
}

}  // extern "C"

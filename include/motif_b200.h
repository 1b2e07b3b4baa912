/*
 * motif_b200.h — C ABI of the B200 colour-coding engine (libmotif_b200.so).
 *
 * Drop-in boundary for the counting path of the arXiv 1602.04478 artifact
 * (/root/reference/proj, C++ namespace motif).  Every entry point below names
 * the reference interface it replaces (file:line).  Plain pointers and sizes
 * only; no C++ or torch types cross this boundary.
 *
 * Status codes (the reference's exception taxonomy, include/motif/errors.hpp,
 * and its CLI exit codes, tools/motif_main.cpp:387-406):
 *   0 ok, 1 internal, 2 ParseError, 3 TreewidthError, 4 OverflowError,
 *   5 BudgetError, 6 SchemaError, 7 ContractError, 8 SpecError, 9 CUDA error.
 * mb_last_error() returns the message of the last failure on this thread.
 *
 * Colourings use the reference convention: chi[v] in 1..k.
 */
#ifndef MOTIF_B200_H
#define MOTIF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mb_graph mb_graph;
typedef struct mb_plan mb_plan;

/* Message of the last failing call on this thread. */
const char* mb_last_error(void);
/* Library version string. */
const char* mb_version(void);

/* ---- data graph (include/motif/graph.hpp) ---------------------------------- */

/* DataGraph::from_edges (graph.hpp:20): duplicates, both orientations and self
 * loops are normalised away.  loops/dups (nullable) receive LoadStats. */
int mb_graph_from_edges(uint32_t n, const uint32_t* eu, const uint32_t* ev, uint64_t m,
                        mb_graph** out, uint64_t* loops, uint64_t* dups);
/* load_edge_list_file (graph.hpp:48), same grammar and ParseError messages. */
int mb_graph_load_edge_list(const char* path, mb_graph** out, uint64_t* loops, uint64_t* dups);
/* Seeded synthetic graphs for the benchmark configs (no reference counterpart
 * at this scale; chunglu.hpp:29 is the O(n^2) desk-scale sampler). */
int mb_graph_gen_erdos_renyi(uint32_t n, uint64_t m, uint64_t seed, mb_graph** out);
int mb_graph_gen_chung_lu(uint32_t n, double gamma, double avg_degree, double max_w,
                          uint64_t seed, mb_graph** out);
int mb_graph_gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                      mb_graph** out);
void mb_graph_free(mb_graph* g);
uint32_t mb_graph_num_vertices(const mb_graph* g);
uint64_t mb_graph_num_edges(const mb_graph* g);
/* Normalised CSR: offsets[n+1], adj[2m] (DataGraph::neighbors, graph.hpp:25). */
int mb_graph_csr(const mb_graph* g, uint64_t* offsets, uint32_t* adj);
/* Undirected edge list u<v, sorted (serialize_edge_list, graph.hpp:51). */
int mb_graph_edges(const mb_graph* g, uint32_t* eu, uint32_t* ev);
/* degree_rank (graph.hpp:68): rank[v] = position in the (degree, id) order. */
int mb_graph_degree_rank(const mb_graph* g, uint32_t* rank);
/* DataGraph::validate (graph.hpp:31). */
int mb_graph_validate(const mb_graph* g);

/* random_coloring (graph.hpp:85): chi[v] in 1..k, std::mt19937_64(seed). */
int mb_random_coloring(uint32_t n, int k, uint64_t seed, uint8_t* chi);
/* derive_seed (rng.hpp:18): per-trial seed stream of estimate(). */
uint64_t mb_derive_seed(uint64_t master, uint64_t stream);

/* ---- query and plan (include/motif/query.hpp) ------------------------------ */

/* QueryGraph::from_edges (query.hpp:25) + enumerate_trees (query.hpp:94) +
 * select_plan (query.hpp:108).  edges: m pairs (2*m ints). */
int mb_plan_create(int k, const int32_t* edges, int m, uint64_t max_trees, mb_plan** out);
/* parse_query / load_query_file (query.hpp:36-37) then as above. */
int mb_plan_load_query(const char* path, uint64_t max_trees, mb_plan** out);
void mb_plan_free(mb_plan* p);
int mb_plan_k(const mb_plan* p);
int mb_plan_num_trees(const mb_plan* p);
/* Index of the tree select_plan chose; mb_plan_use_tree switches the tree
 * the counting calls run (plan-invariance checks, tests/test_engine.cpp:187-200). */
int mb_plan_selected(const mb_plan* p);
int mb_plan_use_tree(mb_plan* p, int idx);
/* DecompositionTree::canonical (query.hpp:76) of tree idx (-1 = in use). */
int mb_plan_canonical(const mb_plan* p, int idx, char* buf, int len);
/* plan_score (query.hpp:104) of tree idx: {max_cycle_length, boundary_total, annotation_total}. */
int mb_plan_score(const mb_plan* p, int idx, int* score3);

/* ---- counting (include/motif/engine.hpp:121, runtime.hpp:87) --------------- */

/* engine: 0 = PS, 1 = DB (EngineKind, engine.hpp:12).  Both return the same
 * count; the device path always anchors cycles at their degree-highest vertex
 * (the DB partition, paper Eq. 1). */

/* count_colorful for `ncol` colourings stored back to back (n bytes each) in
 * HOST memory; the graph, colourings and results cross PCIe inside the call. */
int mb_count_colorful(mb_graph* g, mb_plan* p, const uint8_t* chi, int ncol, int engine,
                      uint64_t* out);
/* Same, colourings generated from seeds with random_coloring(n, k, seed) ON
 * THE DEVICE: seeds in, counts out, no colouring crosses PCIe. */
int mb_count_colorful_seeds(mb_graph* g, mb_plan* p, const uint64_t* seeds, int ncol, int engine,
                            uint64_t* out);
/* The colourings random_coloring(n, k, seeds[i]) as the DEVICE generates them
 * for mb_count_colorful_seeds / mb_estimate (one CTA per colouring runs the
 * mt19937_64 stream; bit-identical to mb_random_coloring), copied to host
 * memory (n bytes per seed): for tests and callers that want to inspect them.
 * limit = 0 uses the reference's rejection limit 2^64 - 1 - (2^64 - 1) % k. */
int mb_device_random_colorings(mb_graph* g, int k, const uint64_t* seeds, int ncol, uint64_t limit,
                               uint8_t* out);
/* Vertex-sharded count (one rank of a multi-GPU job; the
 * reference's BspExecutor over Partition, runtime.cpp:11-25, 297-324): this
 * rank's partial count of each colouring, the matches of the root block
 * anchored at its share of the data-graph vertices (device vertices in degree
 * order dealt cyclically over `world` ranks).  The partials of ranks
 * 0..world-1 add up to mb_count_colorful's count.  *split (nullable) = 1 when
 * the root block was split, 0 when rank 0 returned the whole count. */
int mb_count_colorful_shard(mb_graph* g, mb_plan* p, const uint8_t* chi, int ncol, int engine,
                            int rank, int world, uint64_t* partial, int* split);
/* Vertex-sharded count with table exchange: as
 * mb_count_colorful_shard, and in addition every leaf block of the plan is
 * computed for this rank's vertices only and its rows are exchanged — the
 * reference's BSP rounds ship table entries to the owner of their key vertex
 * (redistribute / extend, runtime.cpp:94-114, 173-202); here each rank packs
 * its rows into slice `rank` of a DEVICE buffer of `world` slices of
 * `bytes_per_rank` bytes and calls `allgather(ctx, buf, bytes_per_rank,
 * stream)`, which must fill the other slices with the other ranks' (an
 * in-place all-gather).  `stream` is the engine's cudaStream_t: the packed
 * rows are ready in stream order on it, and the callback must leave the
 * gathered buffer ready in stream order on it — enqueue ncclAllGather on that
 * stream and return (nothing blocks the host), or synchronise it, gather
 * through the host and copy back.  Returns 0 on success.  Every rank makes the
 * same sequence of calls.  A root 3-cycle block with a scalar output is dealt
 * over the ranks by warp batch of oriented edges, a root cycle block by anchor
 * vertex, a root leaf block by vertex; *split as above. */
typedef int (*mb_allgather_fn)(void* ctx, void* dev_buf, uint64_t bytes_per_rank, void* cuda_stream);
int mb_count_colorful_sharded(mb_graph* g, mb_plan* p, const uint8_t* chi, int ncol, int engine,
                              int rank, int world, mb_allgather_fn allgather, void* ctx,
                              uint64_t* partial, int* split);
/* Device-resident colourings (n*ncol bytes, colours 1..k, cudaMalloc'd). */
int mb_count_colorful_device(mb_graph* g, mb_plan* p, const uint8_t* chi_dev, int ncol,
                             uint64_t* out);

/* ---- estimator (include/motif/estimate.hpp) -------------------------------- */

/* automorphism_count (estimate.hpp:14), k <= 10. */
int mb_automorphism_count(int k, const int32_t* edges, int m, uint64_t* out);
/* normalization_factor k^k/k! (estimate.hpp:18). */
double mb_normalization_factor(int k);
/* coefficient_of_variation (estimate.hpp:39). */
double mb_coefficient_of_variation(const uint64_t* counts, uint64_t n);
/* estimate (estimate.hpp:34): per-trial colourings from derive_seed(seed, i);
 * per_trial (trials entries), mean_estimate, cv, aut, subgraph_estimate. */
int mb_estimate(mb_graph* g, mb_plan* p, int engine, uint64_t trials, uint64_t seed,
                uint64_t* per_trial, double* mean, double* cv, uint64_t* aut, double* subgraph);

/* The report of estimate() from per-trial colourful counts gathered elsewhere
 * (the sharded multi-rank estimate): norm * mean in long double exactly as
 * estimate.cpp:124-127, cv, and mean / aut. */
int mb_estimate_from_counts(int k, uint64_t aut, const uint64_t* per_trial, uint64_t trials,
                            double* mean, double* cv, double* subgraph);

/* ---- 1-D partition (include/motif/runtime.hpp:14-36) ----------------------- */

/* Partition(n, p): block_begin / block_size / owner; returns 8 if p<1 or p>n. */
int mb_partition_block(uint32_t n, int p, int w, uint32_t* begin, uint32_t* size);
int mb_partition_owner(uint32_t n, int p, uint32_t v, int* owner);

/* ---- device engine introspection (benchmark / roofline) -------------------- */

int mb_engine_enable_timing(mb_graph* g, int on);
/* Per-kernel-name device time (ms, summed), launches, compulsory HBM bytes
 * (summed) and name of entry idx; returns 8 when idx is past the end. */
int mb_engine_kernel_timing(mb_graph* g, int idx, char* name, int len, double* ms,
                            uint64_t* launches, uint64_t* bytes);
/* cudaStream_t the engine launches on (for CUDA-event timing by callers).
 * mb_count_colorful_device reads chi_dev on this stream: a caller that fills
 * chi_dev on another stream must synchronise that stream first. */
void* mb_engine_stream(mb_graph* g);
/* CUDA device of the graph's engine (-1 before the first count).  The engine
 * is created on the caller's current device at the first counting call and
 * every later call runs there, restoring the caller's current device. */
int mb_engine_device(const mb_graph* g);
/* Milliseconds spent building plan-derived graph indexes (triangle lists). */
double mb_engine_prep_ms(mb_graph* g);
uint64_t mb_engine_launches(mb_graph* g);
/* Bytes this rank has received through mb_count_colorful_sharded's exchanges. */
uint64_t mb_engine_exchanged_bytes(mb_graph* g);
int mb_engine_stats(mb_graph* g, uint64_t* triangles, uint64_t* table_bytes,
                    uint64_t* dp_updates);
/* Drop plan-derived graph structures so the next count rebuilds them. */
int mb_engine_reset_derived(mb_graph* g);
/* Release the device engine (graph stays on the host). */
int mb_engine_release(mb_graph* g);

#ifdef __cplusplus
}
#endif

#endif /* MOTIF_B200_H */

// B200 colour-coding engine: host-side orchestration of the device kernels.
//
// Replaces the reference's counting engine (include/motif/engine.hpp:118-123,
// count_colorful / count_colorful_exec, and the Executor table primitives of
// engine.hpp:39-65) for every treewidth-2 plan the planner emits.  Projection
// tables (reference: hash maps, table.hpp:36) live in HBM as dense rows indexed
// by colour set (sig.cuh):
//   - unary tables   : one row per vertex           [n][C(k-1, s-1)]
//   - edge tables    : one row per CSR slot (u->v)  [2m][C(k-2, s-2)]
//   - scalars        : the root's colourful count
// Blocks are solved by fused kernels instead of the reference's op-by-op
// table algebra:
//   - leaf blocks      -> leaf_extend_kernel   (path-table extension along CSR rows)
//   - 3-cycle blocks   -> triangle_block_kernel over the degree-ordered triangle list
//   - longer cycles    -> cycle engine (degree-capped half paths, DB, Eq. 1)
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../host/graph.hpp"
#include "../host/plan.hpp"

namespace mb {

struct EngineStats {
  uint64_t triangles = 0;       // degree-ordered triangles listed
  uint64_t table_bytes = 0;     // bytes of DP tables resident
  uint64_t dp_updates = 0;      // table-entry updates (nonzero contributions) of the last count
  double last_ms = 0;
  double prep_ms = 0;           // wall time of the last plan-derived index build
};

int current_device();  // the calling thread's current CUDA device

class GpuEngine {
 public:
  // device < 0: the caller's current CUDA device
  explicit GpuEngine(const CsrGraph& g, int device = -1);
  ~GpuEngine();
  GpuEngine(const GpuEngine&) = delete;
  GpuEngine& operator=(const GpuEngine&) = delete;

  uint32_t num_vertices() const;
  uint64_t num_edges() const;

  // Binds a plan (allocates its tables, builds the structures it needs).
  void bind_plan(const Plan& plan, int k);

  // Colourful count for each colouring.  `chi` holds `count` colourings of n
  // vertices each, colours 1..k, in host memory (host=true) or device memory.
  void count(const uint8_t* chi, int count_colorings, bool host, uint64_t* out);
  // The same for the colourings random_coloring(n, k, seeds[i]), generated on
  // the device (k_random_colorings): nothing but the seeds and the counts
  // crosses PCIe.  `count_colorings` is bounded by the caller (n bytes each).
  void count_seeds(const uint64_t* seeds, int count_colorings, uint64_t* out);
  // ... for any number of seeds, `batch` colourings per device call, batch i + 1
  // generated on a side stream while batch i is counted.
  void count_seeds_batched(const uint64_t* seeds, uint64_t total, int batch, uint64_t* out);
  // The device-generated colourings themselves (tests): n bytes per seed into
  // host memory; limit = 0 uses the reference's rejection limit.
  void random_colorings(int k, const uint64_t* seeds, int count_colorings, uint64_t limit, uint8_t* out_host);

  // Drops plan-derived graph structures (triangle list); the next count
  // rebuilds them.  Used by the benchmark to keep that work inside a step.
  void reset_derived();

  // Kernel-level timing hooks for the roofline: average duration (ms) of the
  // dominant DP kernel over the last count() and its algorithmic bytes.
  struct KernelTiming {
    std::string name;
    double ms = 0;
    uint64_t bytes = 0;
    uint64_t launches = 0;
  };
  std::vector<KernelTiming> kernel_timings() const;
  void enable_timing(bool on);
  uint64_t launches() const;
  const EngineStats& stats() const;
  void* stream() const;
  int device() const;
  // Vertex sharding: count() then returns this rank's partial
  // count, the matches anchored at the device vertices x with
  // x % world == rank; the partials of all ranks add up to the count.  Only a
  // root cycle block with a scalar output is split (root_shardable());
  // otherwise rank 0 returns the whole count and the other ranks 0.
  void set_shard(uint32_t rank, uint32_t world);
  bool root_shardable() const;
  // Table exchange for sharded leaf blocks (the reference's
  // redistribute / extend shipping rows to their owners, runtime.cpp:94-114,
  // 173-202): with an exchange set, every leaf block computes only the rows of
  // this rank's vertices, packs them into slice `rank` of a device buffer of
  // `world` equal slices and calls the exchange, which must fill the other
  // slices with the other ranks' rows (an in-place all-gather: NCCL on
  // NVLink, or staged through the host), in stream order on the engine's
  // stream (passed along: a collective enqueued on it needs no host
  // synchronisation); the rows are then unpacked so every rank holds the
  // whole table again.  Blocks above the leaves read whole tables, so only
  // these rows ever cross ranks.
  using AllGather = std::function<void(void* dev_buf, uint64_t bytes_per_rank, void* cuda_stream)>;
  void set_exchange(AllGather fn);
  uint64_t exchanged_bytes() const;  // bytes received through the exchange so far

  struct Impl;

 private:
  std::unique_ptr<Impl> impl_;
};

}  // namespace mb

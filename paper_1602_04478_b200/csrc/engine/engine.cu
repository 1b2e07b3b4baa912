// B200 colour-coding engine (see engine.hpp for the design summary).
#include "engine.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdlib>
#include <functional>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "../host/errors.hpp"
#include "sig.cuh"

namespace mb {

// ----------------------------------------------------------------- helpers

#define MB_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      ::mb::fail(::mb::kCuda, std::string(#call) + ": " + cudaGetErrorString(_e));     \
  } while (0)

using u64 = unsigned long long;

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  explicit DBuf(size_t b) { alloc(b); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr, o.bytes = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    p = o.p, bytes = o.bytes;
    o.p = nullptr, o.bytes = 0;
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t b) {
    release();
    if (b) MB_CUDA(cudaMalloc(&p, b));
    bytes = b;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

__constant__ SigLut c_lut;

namespace {

uint64_t binom_host(int n, int r) {
  if (r < 0 || r > n) return 0;
  uint64_t b = 1;
  for (int i = 1; i <= r; ++i) b = b * (n - r + i) / i;
  return b;
}

// Device-side LUT holder; initialised once per process.
struct LutHolder {
  DBuf unrank;
  bool ready = false;
  void init() {
    if (ready) return;
    std::vector<uint16_t> masks;
    SigLut L{};
    for (int t = 0; t <= kMaxColors; ++t) {
      L.off[t] = static_cast<uint32_t>(masks.size());
      for (uint32_t m = 0; m < (1u << kMaxColors); ++m)
        if (__builtin_popcount(m) == t) masks.push_back(static_cast<uint16_t>(m));
    }
    L.off[kMaxColors + 1] = static_cast<uint32_t>(masks.size());
    for (int c = 0; c <= kMaxColors; ++c)
      for (int i = 0; i <= kMaxColors + 1; ++i) L.binom[c][i] = static_cast<uint32_t>(binom_host(c, i));
    unrank.alloc(masks.size() * sizeof(uint16_t));
    MB_CUDA(cudaMemcpy(unrank.p, masks.data(), masks.size() * sizeof(uint16_t),
                       cudaMemcpyHostToDevice));
    L.unrank = unrank.as<uint16_t>();
    MB_CUDA(cudaMemcpyToSymbol(c_lut, &L, sizeof(L)));
    ready = true;
  }
};

LutHolder& lut_holder() {
  static LutHolder h;
  return h;
}

// Checked arithmetic: the reference throws OverflowError (errors.hpp:52); the
// device raises a flag that the host turns into the same error.
__device__ __forceinline__ uint64_t mul_ck(uint64_t a, uint64_t b, int* err) {
  if (__umul64hi(a, b)) atomicOr(err, 1);
  return a * b;
}

__device__ __forceinline__ void atomic_add_ck(u64* p, uint64_t v, int* err) {
  const u64 old = atomicAdd(p, static_cast<u64>(v));
  if (old + v < old) atomicOr(err, 1);
}

__device__ __forceinline__ uint64_t add_ck(uint64_t a, uint64_t b, int* err) {
  const uint64_t r = a + b;
  if (r < a) atomicOr(err, 1);
  return r;
}

// ------------------------------------------------------- graph preprocessing

__global__ void k_slot_rows(uint32_t n, const uint64_t* __restrict__ off, uint32_t* __restrict__ src) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  for (uint64_t e = off[v]; e < off[v + 1]; ++e) src[e] = v;
}

// rev[e] = slot of (v -> u) for e = (u -> v).
__global__ void k_reverse_slots(uint64_t m2, const uint64_t* __restrict__ off,
                                const uint32_t* __restrict__ adj, const uint32_t* __restrict__ src,
                                uint32_t* __restrict__ rev) {
  const uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (e >= m2) return;
  const uint32_t u = src[e], v = adj[e];
  uint64_t lo = off[v], hi = off[v + 1];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (adj[mid] < u) lo = mid + 1; else hi = mid;
  }
  rev[e] = static_cast<uint32_t>(lo);
}

__global__ void k_recolor(uint64_t total, const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                          int k, int* err) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= total) return;
  const int c = in[i];
  if (c < 1 || c > k) atomicOr(err, 2);
  out[i] = static_cast<uint8_t>(c - 1);
}

// Degree-ordered orientation: out(x) = neighbours ranked below x, kept in id
// order, remembered with their CSR slot.
__global__ void k_out_degree(uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                             const uint32_t* __restrict__ rank, uint64_t* __restrict__ outdeg) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const uint32_t rx = rank[x];
  uint64_t c = 0;
  for (uint64_t e = off[x]; e < off[x + 1]; ++e) c += rank[adj[e]] < rx;
  outdeg[x] = c;
}

__global__ void k_out_fill(uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                           const uint32_t* __restrict__ rank, const uint64_t* __restrict__ out_off,
                           uint32_t* __restrict__ out_nbr, uint32_t* __restrict__ out_slot) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const uint32_t rx = rank[x];
  uint64_t w = out_off[x];
  for (uint64_t e = off[x]; e < off[x + 1]; ++e) {
    const uint32_t y = adj[e];
    if (rank[y] < rx) {
      out_nbr[w] = y;
      out_slot[w] = static_cast<uint32_t>(e);
      ++w;
    }
  }
}

// ------------------------------------------------------------- leaf blocks

struct LeafArgs {
  const uint64_t* off;   // relation rows (graph CSR or a pair table's CSR)
  const uint32_t* adj;
  const uint32_t* rev;
  const uint8_t* chi;
  const uint64_t* ua;  // node child on the boundary a (row = img a), may be null
  const uint64_t* ub;  // node child on the leaf b (row = img b), may be null
  const uint64_t* ue;  // edge child (edge table), may be null
  uint32_t Pa, Pb, Pe, PZ, Pout;
  int sa, sb, se, sZ;
  int e_rev;           // edge child stored keyed (b, a): read rev[slot]
  uint64_t* out;       // unary [n][Pout]
  int* err;
  u64* updates;
};

// Path-table extension along CSR rows (paper §5.2 leaf block: joins of the
// edge, the leaf's annotation and the boundary's annotation, projected to the
// boundary).  One GROUP (warp or CTA) per boundary vertex x: the group streams
// x's neighbour rows (lanes over (neighbour, entry) pairs, so consecutive lanes
// read consecutive words of a row), folds each into a shared-memory
// accumulator Z over colour sets, then joins Z with x's own annotation row and
// writes the output row once.
template <int GROUP>
__global__ void __launch_bounds__(GROUP >= 128 ? GROUP : 128)
leaf_extend_kernel(LeafArgs A, const uint32_t* __restrict__ vlist, uint32_t nv) {
  extern __shared__ u64 smem[];
  constexpr int kGroups = (GROUP >= 128 ? GROUP : 128) / GROUP;
  const int g = threadIdx.x / GROUP, lane = threadIdx.x % GROUP;
  u64* Z = smem + static_cast<size_t>(g) * (A.PZ + A.Pout);
  u64* O = Z + A.PZ;
  const uint32_t gi = blockIdx.x * kGroups + g;
  const bool active = gi < nv;
  const uint32_t x = active ? vlist[gi] : 0;
  uint64_t upd = 0;
  for (uint32_t i = lane; i < A.PZ + A.Pout; i += GROUP) Z[i] = 0;
  if (GROUP == 32) __syncwarp(); else __syncthreads();
  if (active) {
    const uint32_t cx = A.chi[x], fx = 1u << cx;
    const uint64_t base = A.off[x], deg = A.off[x + 1] - base;
    const uint32_t pe = A.ue ? A.Pe : 1u, pb = A.ub ? A.Pb : 1u, per = pe * pb;
    const uint64_t items = deg * per;
    for (uint64_t it = lane; it < items; it += GROUP) {
      const uint64_t j = it / per;
      const uint32_t r = static_cast<uint32_t>(it - j * per);
      const uint32_t ie = r / pb, ib = r - ie * pb;
      const uint64_t slot = base + j;
      const uint32_t y = __ldg(A.adj + slot);
      const uint32_t cy = __ldg(A.chi + y), fy = 1u << cy;
      if (cy == cx) continue;
      uint32_t M = fx | fy;
      uint64_t val = 1;
      if (A.ue) {
        const uint64_t e = A.e_rev ? __ldg(A.rev + slot) : slot;
        const uint64_t v = __ldg(A.ue + e * A.Pe + ie);
        if (!v) continue;
        M = sig_expand(sig_unrank(c_lut, A.se - 2, ie), fx | fy);
        val = v;
      }
      if (A.ub) {
        const uint64_t v = __ldg(A.ub + static_cast<uint64_t>(y) * A.Pb + ib);
        if (!v) continue;
        const uint32_t Mb = sig_expand(sig_unrank(c_lut, A.sb - 1, ib), fy);
        if ((M & Mb) != fy) continue;
        M |= Mb;
        val = mul_ck(val, v, A.err);
      }
      atomic_add_ck(&Z[sig_index(c_lut, M, fx)], val, A.err);
      ++upd;
    }
  }
  if (GROUP == 32) __syncwarp(); else __syncthreads();
  if (active) {
    const uint32_t cx = A.chi[x], fx = 1u << cx;
    if (!A.ua) {
      for (uint32_t i = lane; i < A.Pout; i += GROUP) A.out[static_cast<uint64_t>(x) * A.Pout + i] = Z[i];
    } else {
      const uint64_t items = static_cast<uint64_t>(A.PZ) * A.Pa;
      for (uint64_t it = lane; it < items; it += GROUP) {
        const uint32_t iz = static_cast<uint32_t>(it / A.Pa), ia = static_cast<uint32_t>(it - iz * A.Pa);
        const uint64_t z = Z[iz];
        if (!z) continue;
        const uint64_t a = __ldg(A.ua + static_cast<uint64_t>(x) * A.Pa + ia);
        if (!a) continue;
        const uint32_t Mz = sig_expand(sig_unrank(c_lut, A.sZ - 1, iz), fx);
        const uint32_t Ma = sig_expand(sig_unrank(c_lut, A.sa - 1, ia), fx);
        if ((Mz & Ma) != fx) continue;
        atomic_add_ck(&O[sig_index(c_lut, Mz | Ma, fx)], mul_ck(z, a, A.err), A.err);
        ++upd;
      }
      if (GROUP == 32) __syncwarp(); else __syncthreads();
      for (uint32_t i = lane; i < A.Pout; i += GROUP) A.out[static_cast<uint64_t>(x) * A.Pout + i] = O[i];
    }
  }
  if (upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// Total of a table (singleton-root plans, reference engine.cpp:398).
__global__ void k_table_total(const uint64_t* __restrict__ t, uint64_t count, u64* out, int* err) {
  uint64_t local = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    local = add_ck(local, t[i], err);
  for (int o = 16; o > 0; o >>= 1) local = add_ck(local, __shfl_down_sync(0xffffffffu, local, o), err);
  if ((threadIdx.x & 31) == 0 && local) atomic_add_ck(out, local, err);
}

unsigned grid_for(uint64_t work, unsigned block) {
  const uint64_t g = (work + block - 1) / block;
  return static_cast<unsigned>(std::max<uint64_t>(1, g));
}

#include "cycle_engine.cuh"
#include "leaf.cuh"
#include "tri_edge.cuh"

}  // namespace

// ---------------------------------------------------------------- the engine

enum class TKind { None, Scalar, Vertex, Edge, Pair };

struct DevTable {
  TKind kind = TKind::None;
  int s = 0;
  uint32_t P = 0;
  uint64_t rows = 0;  // Vertex: n, Edge: 2m, Pair: number of pairs
  DBuf buf;           // payload rows
  // Pair tables: sorted packed keys, CSR by first key, transposed copy
  DBuf keys, off, cols, off_t, cols_t, buf_t;
  uint64_t* data() const { return buf.as<uint64_t>(); }
};

struct StepPlan {
  int block = -1;
  BlockKind kind = BlockKind::Cycle;
  int L = 0;
  std::vector<int> node_tab, edge_tab;
  std::vector<char> edge_fwd;
  std::vector<int> bpos;
  int s_out = 0;
  bool general = false;  // cycle solved by the general half-path engine
};

struct GpuEngine::Impl {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t n = 0;
  uint64_t m2 = 0;
  DBuf off, adj, rank, src, rev, vlight, vheavy;
  uint32_t nlight = 0, nheavy = 0;
  uint64_t slots_light = 0;  // CSR slots owned by light vertices
  // derived: degree-ordered triangle list
  bool tri_ready = false;
  uint64_t ntri = 0, ncn = 0, nout = 0;
  DBuf out_nbr, out_slot, out_src, cn_off, cn;  // oriented edges + their CN lists
  // plan
  bool plan_bound = false;
  int k = 0;
  Plan plan;
  std::vector<StepPlan> steps;
  std::vector<DevTable> tables;
  bool needs_triangles = false;
  // per-count scratch
  DBuf chi, chi_in, flags;  // flags: [0] err (int), [1..] scalar (u64), updates (u64)
  DBuf scratch;
  // stats / timing
  EngineStats st;
  bool timing = false;
  std::map<std::string, KernelTiming> timings;
  uint64_t launch_count = 0;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<uint64_t> pending_bytes;
  std::vector<cudaEvent_t> event_pool;

  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    MB_CUDA(cudaEventCreate(&e));
    return e;
  }

  // Launch wrapper: error check, launch count, optional CUDA-event timing on
  // the engine stream.  `bytes` = the kernel's compulsory (algorithmic) HBM
  // bytes for this launch, used for the roofline.
  template <class F>
  void launch(const char* name, F&& f, uint64_t bytes = 0) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (timing) {
      a = get_event();
      b = get_event();
      MB_CUDA(cudaEventRecord(a, stream));
    }
    f();
    MB_CUDA(cudaGetLastError());
    ++launch_count;
    if (timing) {
      MB_CUDA(cudaEventRecord(b, stream));
      pending.push_back({name, {a, b}});
      pending_bytes.push_back(bytes);
    }
  }

  void collect_timings() {
    for (size_t i = 0; i < pending.size(); ++i) {
      auto& p = pending[i];
      float ms = 0;
      MB_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
      auto& t = timings[p.first];
      t.name = p.first;
      t.ms += ms;
      t.bytes += pending_bytes[i];
      t.launches++;
      event_pool.push_back(p.second.first);
      event_pool.push_back(p.second.second);
    }
    pending.clear();
    pending_bytes.clear();
  }

  void upload(const CsrGraph& g) {
    lut_holder().init();
    n = g.n;
    m2 = 2 * g.m;
    if (m2 >= 0xFFFFFFFFULL) fail(kSpec, "graph exceeds 2^32 half-edges (32-bit CSR slots)");
    off.alloc((n + 1) * sizeof(uint64_t));
    adj.alloc(std::max<uint64_t>(m2, 1) * sizeof(uint32_t));
    MB_CUDA(cudaMemcpyAsync(off.p, g.offsets.data(), (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, stream));
    if (m2) MB_CUDA(cudaMemcpyAsync(adj.p, g.adj.data(), m2 * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    const auto rk = degree_rank(g);
    rank.alloc(std::max<uint32_t>(n, 1) * sizeof(uint32_t));
    if (n) MB_CUDA(cudaMemcpyAsync(rank.p, rk.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    src.alloc(std::max<uint64_t>(m2, 1) * sizeof(uint32_t));
    rev.alloc(std::max<uint64_t>(m2, 1) * sizeof(uint32_t));
    if (n) launch("slot_rows", [&] { k_slot_rows<<<grid_for(n, 256), 256, 0, stream>>>(n, off.as<uint64_t>(), src.as<uint32_t>()); });
    if (m2)
      launch("reverse_slots", [&] {
        k_reverse_slots<<<grid_for(m2, 256), 256, 0, stream>>>(m2, off.as<uint64_t>(), adj.as<uint32_t>(),
                                                              src.as<uint32_t>(), rev.as<uint32_t>());
      });
    // degree bins for the vertex-centric kernels: warp per light vertex,
    // CTA per heavy vertex (threshold = 8 warp-iterations of a unit row).
    std::vector<uint32_t> light, heavy;
    for (uint32_t v = 0; v < n; ++v) (g.degree(v) > 256 ? heavy : light).push_back(v);
    nlight = static_cast<uint32_t>(light.size());
    nheavy = static_cast<uint32_t>(heavy.size());
    slots_light = 0;
    for (uint32_t v : light) slots_light += g.degree(v);
    vlight.alloc(std::max<size_t>(light.size(), 1) * 4);
    vheavy.alloc(std::max<size_t>(heavy.size(), 1) * 4);
    if (nlight) MB_CUDA(cudaMemcpyAsync(vlight.p, light.data(), light.size() * 4, cudaMemcpyHostToDevice, stream));
    if (nheavy) MB_CUDA(cudaMemcpyAsync(vheavy.p, heavy.data(), heavy.size() * 4, cudaMemcpyHostToDevice, stream));
    flags.alloc(64);
    MB_CUDA(cudaStreamSynchronize(stream));
  }

  void build_triangles() {
    if (tri_ready) return;
    const auto t0 = std::chrono::steady_clock::now();
    DBuf outdeg((n + 1) * sizeof(uint64_t)), out_off((n + 1) * sizeof(uint64_t));
    MB_CUDA(cudaMemsetAsync(outdeg.p, 0, (n + 1) * sizeof(uint64_t), stream));
    launch("tri_outdeg", [&] {
      k_out_degree<<<grid_for(n, 256), 256, 0, stream>>>(n, off.as<uint64_t>(), adj.as<uint32_t>(),
                                                         rank.as<uint32_t>(), outdeg.as<uint64_t>());
    });
    exclusive_scan(outdeg.as<uint64_t>(), out_off.as<uint64_t>(), n + 1);
    uint64_t nout = 0;
    MB_CUDA(cudaMemcpyAsync(&nout, out_off.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, stream));
    MB_CUDA(cudaStreamSynchronize(stream));
    DBuf out_nbr(std::max<uint64_t>(nout, 1) * 4), out_slot(std::max<uint64_t>(nout, 1) * 4),
        out_src(std::max<uint64_t>(nout, 1) * 4);
    launch("tri_outfill", [&] {
      k_out_fill<<<grid_for(n, 256), 256, 0, stream>>>(n, off.as<uint64_t>(), adj.as<uint32_t>(), rank.as<uint32_t>(),
                                                       out_off.as<uint64_t>(), out_nbr.as<uint32_t>(),
                                                       out_slot.as<uint32_t>());
    });
    // out_src[j] = src[out_slot[j]]
    gather_src(out_slot.as<uint32_t>(), out_src.as<uint32_t>(), nout);
    // per-oriented-edge common-neighbour lists: count, scan, fill
    DBuf cnt((nout + 1) * 8);
    cn_off.alloc((nout + 1) * 8);
    MB_CUDA(cudaMemsetAsync(cnt.p, 0, (nout + 1) * 8, stream));
    if (nout)
      launch("cn_count", [&] {
        k_cn_build<0><<<grid_for(nout, 128), 128, 0, stream>>>(nout, out_off.as<uint64_t>(), out_nbr.as<uint32_t>(),
                                                               out_slot.as<uint32_t>(), out_src.as<uint32_t>(),
                                                               rev.as<uint32_t>(), reinterpret_cast<u64*>(cnt.p),
                                                               nullptr, nullptr, nullptr, nullptr);
      });
    exclusive_scan(cnt.as<uint64_t>(), cn_off.as<uint64_t>(), nout + 1);
    uint64_t ncn_h = 0;
    MB_CUDA(cudaMemcpyAsync(&ncn_h, cn_off.as<uint64_t>() + nout, 8, cudaMemcpyDeviceToHost, stream));
    MB_CUDA(cudaStreamSynchronize(stream));
    ncn = ncn_h;
    ntri = ncn / 3;
    cn.alloc(std::max<uint64_t>(3 * ncn, 1) * sizeof(uint32_t));  // SoA: w | slot a->w | slot b->w
    MB_CUDA(cudaMemsetAsync(cnt.p, 0, (nout + 1) * 8, stream));
    if (nout && ncn)
      launch("cn_fill", [&] {
        k_cn_build<1><<<grid_for(nout, 128), 128, 0, stream>>>(nout, out_off.as<uint64_t>(), out_nbr.as<uint32_t>(),
                                                               out_slot.as<uint32_t>(), out_src.as<uint32_t>(),
                                                               rev.as<uint32_t>(), reinterpret_cast<u64*>(cnt.p),
                                                               cn_off.as<uint64_t>(), cn.as<uint32_t>(), cn.as<uint32_t>() + ncn, cn.as<uint32_t>() + 2 * ncn);
      });
    MB_CUDA(cudaStreamSynchronize(stream));
    this->nout = nout;
    this->out_nbr = std::move(out_nbr);
    this->out_slot = std::move(out_slot);
    this->out_src = std::move(out_src);
    st.triangles = ntri;
    tri_ready = true;
    st.prep_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }

  void exclusive_scan(const uint64_t* in, uint64_t* out, uint64_t count) {
    size_t tmp = 0;
    MB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int64_t>(count), stream));
    if (scratch.bytes < tmp) scratch.alloc(tmp);
    MB_CUDA(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, in, out, static_cast<int64_t>(count), stream));
  }

  void gather_src(const uint32_t* slots, uint32_t* outp, uint64_t count);

  // ------------------------------------------------------------ plan binding

  static uint64_t binom(int a, int b) { return binom_host(a, b); }

  void bind(const Plan& p, int kk) {
    if (kk > kMaxColors) fail(kSpec, "GPU engine supports k <= 16 colours");
    k = kk;
    plan = p;
    steps.clear();
    tables.clear();
    tables.resize(p.blocks.size());
    needs_triangles = false;
    for (int id : p.bottom_up()) {
      const Block& b = p.blocks[id];
      StepPlan sp;
      sp.block = id;
      sp.kind = b.kind;
      sp.L = b.size();
      sp.s_out = __builtin_popcount(p.subquery_nodes(id));
      for (int c : b.node_child) sp.node_tab.push_back(c);
      for (int c : b.edge_child) sp.edge_tab.push_back(c);
      sp.edge_fwd = b.edge_fwd;
      for (int x : b.boundary) sp.bpos.push_back(b.pos(x));
      DevTable& out = tables[id];
      out.s = sp.s_out;
      if (b.kind == BlockKind::Leaf || b.boundary.size() == 1) {
        out.kind = TKind::Vertex;
        out.P = static_cast<uint32_t>(binom(k - 1, sp.s_out - 1));
        out.rows = n;
      } else if (b.boundary.empty()) {
        out.kind = TKind::Scalar;
      } else {
        // two boundary nodes: stored per CSR slot when the pair is always a
        // graph edge (cycle-adjacent through an original or edge-keyed edge),
        // otherwise as a sorted pair table
        const int d = (sp.bpos[1] - sp.bpos[0] + sp.L) % sp.L;
        int e = -1;
        if (d == 1) e = sp.bpos[0];
        if (d == sp.L - 1) e = sp.bpos[1];
        const bool on_edges = e >= 0 && (sp.edge_tab[e] < 0 || tables[sp.edge_tab[e]].kind == TKind::Edge);
        out.kind = on_edges ? TKind::Edge : TKind::Pair;
        out.P = static_cast<uint32_t>(binom(k - 2, sp.s_out - 2));
        out.rows = on_edges ? m2 : 0;
      }
      if (b.kind == BlockKind::Cycle) {
        bool edge_children_on_edges = true;
        for (int e = 0; e < sp.L; ++e)
          if (sp.edge_tab[e] >= 0 && tables[sp.edge_tab[e]].kind != TKind::Edge) edge_children_on_edges = false;
        static const bool force_general = std::getenv("MB_FORCE_GENERAL_CYCLES") != nullptr;
        // the CN kernel keeps the pivot factors' partial products per edge in
        // shared memory; bound them by the product of all factor widths
        uint64_t fixed_bound = 1;
        for (int q = 0; q < sp.L; ++q) {
          if (sp.node_tab[q] >= 0) fixed_bound *= tables[sp.node_tab[q]].P;
          if (sp.edge_tab[q] >= 0) fixed_bound *= tables[sp.edge_tab[q]].P;
        }
        if (sp.L == 3 && edge_children_on_edges && out.kind != TKind::Pair && !force_general &&
            fixed_bound <= static_cast<uint64_t>(kTriFixedCap))
          needs_triangles = true;
        else
          sp.general = true;
      }
      if (out.kind == TKind::Vertex || out.kind == TKind::Edge) {
        out.buf.alloc(std::max<uint64_t>(out.rows * out.P, 1) * sizeof(uint64_t));
        st.table_bytes += out.buf.bytes;
      }
      steps.push_back(std::move(sp));
    }
    plan_bound = true;
  }

  // ---------------------------------------------------------------- solving

  void run_leaf(const StepPlan& sp, int* err, u64* upd) {
    DevTable& out = tables[sp.block];
    LeafArgs A{};
    A.off = off.as<uint64_t>();
    A.adj = adj.as<uint32_t>();
    A.rev = rev.as<uint32_t>();
    A.chi = chi.as<uint8_t>();
    A.err = err;
    A.updates = upd;
    int s_right = 2;
    if (sp.edge_tab[0] >= 0) {
      const DevTable& t = tables[sp.edge_tab[0]];
      if (t.kind == TKind::Pair) {
        // rows keyed by the boundary image: the stored table when the child is
        // keyed (a, b), its transpose otherwise
        const bool fwd = sp.edge_fwd[0];
        A.off = (fwd ? t.off : t.off_t).as<uint64_t>();
        A.adj = (fwd ? t.cols : t.cols_t).as<uint32_t>();
        A.ue = (fwd ? t.buf : t.buf_t).as<uint64_t>();
        A.e_rev = 0;
      } else {
        A.ue = t.data(), A.e_rev = !sp.edge_fwd[0];
      }
      A.Pe = t.P, A.se = t.s;
      s_right = t.s;
    }
    if (sp.node_tab[1] >= 0) {
      const DevTable& t = tables[sp.node_tab[1]];
      A.ub = t.data(), A.Pb = t.P, A.sb = t.s;
      s_right += t.s - 1;
    }
    if (sp.node_tab[0] >= 0) {
      const DevTable& t = tables[sp.node_tab[0]];
      A.ua = t.data(), A.Pa = t.P, A.sa = t.s;
    }
    A.sZ = s_right;
    A.PZ = static_cast<uint32_t>(binom(k - 1, s_right - 1));
    A.Pout = out.P;
    A.out = out.data();
    if (!A.ua && A.PZ != A.Pout) fail(kInternal, "leaf popcount mismatch");
    const size_t per_group = (A.PZ + (A.ua ? A.Pout : 0)) * sizeof(u64);
    if (!A.ua) A.Pout = out.P;  // O unused
    const size_t group_bytes = (A.PZ + A.Pout) * sizeof(u64);
    (void)per_group;
    if (group_bytes * 4 > 200 * 1024) fail(kSpec, "leaf table row too wide for shared memory (k too large)");
    // compulsory bytes: CSR rows + neighbour colours + every input row once + output
    const uint64_t leaf_bytes = 8 * (uint64_t(n) + 1) + 5 * m2 + n + (A.ub ? uint64_t(n) * A.Pb * 8 : 0) +
                                (A.ua ? uint64_t(n) * A.Pa * 8 : 0) + (A.ue ? m2 * A.Pe * 8 : 0) +
                                uint64_t(n) * out.P * 8;
    // table-driven kernel (leaf.cuh) whenever the edge is a plain graph edge
    LeafMapArgs M{};
    M.off = A.off, M.adj = A.adj, M.chi = A.chi, M.ub = A.ub, M.ua = A.ua;
    M.Pb = A.Pb, M.Pa = A.Pa, M.PZ = A.PZ, M.Pout = A.Pout, M.sb = A.sb, M.sa = A.sa, M.sZ = A.sZ, M.k = k;
    M.out = A.out, M.err = err, M.updates = upd;
    const size_t map_bytes = ((static_cast<size_t>(k) * k * (A.ub ? A.Pb : 1) * 2 + 7) / 8) * 8;
    if (!A.ue && map_bytes + group_bytes * 8 <= 160 * 1024) {
      if (nlight) {
        const size_t smem = map_bytes + group_bytes * 8;  // 8 warps per CTA
        if (smem > 48 * 1024)
          MB_CUDA(cudaFuncSetAttribute(leaf_map_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((nlight + 7) / 8, 148 * 32));
        launch("leaf_map", [&] { leaf_map_kernel<32><<<grid, 256, smem, stream>>>(M, vlight.as<uint32_t>(), nlight); },
               leaf_bytes * (m2 ? double(slots_light) / m2 : 1.0));
      }
      if (nheavy) {
        const size_t smem = map_bytes + group_bytes;
        if (smem > 48 * 1024)
          MB_CUDA(cudaFuncSetAttribute(leaf_map_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(nheavy, 148 * 8));
        launch("leaf_map_heavy",
               [&] { leaf_map_kernel<256><<<grid, 256, smem, stream>>>(M, vheavy.as<uint32_t>(), nheavy); },
               leaf_bytes * (m2 ? double(m2 - slots_light) / m2 : 0.0));
      }
      return;
    }
    if (nlight) {
      const size_t smem = group_bytes * 4;  // 4 warps per CTA
      if (smem > 48 * 1024)
        MB_CUDA(cudaFuncSetAttribute(leaf_extend_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      launch("leaf_extend", [&] {
        leaf_extend_kernel<32><<<grid_for(nlight, 4), 128, smem, stream>>>(A, vlight.as<uint32_t>(), nlight);
      });
    }
    if (nheavy) {
      const size_t smem = group_bytes;
      if (smem > 48 * 1024)
        MB_CUDA(cudaFuncSetAttribute(leaf_extend_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      launch("leaf_extend_heavy", [&] {
        leaf_extend_kernel<256><<<nheavy, 256, smem, stream>>>(A, vheavy.as<uint32_t>(), nheavy);
      });
    }
  }

  // 3-cycle block over the CN lists (tri_edge.cuh).  The pivot edge (P0, P1)
  // is the boundary pair (|B| = 2), an edge at the boundary (|B| = 1) or an
  // annotated edge when there is one, so the pivot-fixed factors are read once
  // per graph edge.
  void run_tri_edge(const StepPlan& sp, int* err, u64* scalar, u64* upd) {
    DevTable& out = tables[sp.block];
    auto edge_idx = [](int a, int b) { return b == (a + 1) % 3 ? a : b; };
    int P0 = 0, P1 = 1;
    if (sp.bpos.size() == 2) {
      P0 = sp.bpos[0], P1 = sp.bpos[1];
    } else if (sp.bpos.size() == 1) {
      P0 = sp.bpos[0];
      const int nxt = (P0 + 1) % 3, prv = (P0 + 2) % 3;
      P1 = (sp.edge_tab[edge_idx(P0, nxt)] < 0 && sp.edge_tab[edge_idx(P0, prv)] >= 0) ? prv : nxt;
    } else {
      for (int e = 0; e < 3; ++e)
        if (sp.edge_tab[e] >= 0) {
          P0 = e, P1 = (e + 1) % 3;
          break;
        }
    }
    const int P2 = 3 - P0 - P1;
    TriEdgeArgs A{};
    A.nout = nout;
    A.cn_off = cn_off.as<uint64_t>();
    A.cn_w = cn.as<uint32_t>(), A.cn_sa = A.cn_w + ncn, A.cn_sb = A.cn_w + 2 * ncn, A.k = k;
    A.out_src = out_src.as<uint32_t>();
    A.out_nbr = out_nbr.as<uint32_t>();
    A.out_slot = out_slot.as<uint32_t>();
    A.rev = rev.as<uint32_t>();
    A.chi = chi.as<uint8_t>();
    A.err = err, A.updates = upd, A.scalar = scalar;
    const bool per_w = sp.node_tab[P2] >= 0 || sp.edge_tab[edge_idx(P1, P2)] >= 0 || sp.edge_tab[edge_idx(P2, P0)] >= 0;
    uint64_t bytes = (per_w ? 12 : 4) * ncn + 8 * (nout + 1) + 12 * nout + n + 4 * m2;
    auto node = [&](int pos, const uint64_t*& t, uint32_t& P, int& s) {
      if (sp.node_tab[pos] < 0) return;
      const DevTable& d = tables[sp.node_tab[pos]];
      t = d.data(), P = d.P, s = d.s;
      bytes += d.buf.bytes;
    };
    auto edge = [&](int pa, int pb, const uint64_t*& t, uint32_t& P, int& s, int& sw) {
      const int i = edge_idx(pa, pb);
      if (sp.edge_tab[i] < 0) return;
      const DevTable& d = tables[sp.edge_tab[i]];
      const bool keyed_ab = (i == pa) ? sp.edge_fwd[i] : !sp.edge_fwd[i];
      t = d.data(), P = d.P, s = d.s, sw = !keyed_ab;
      bytes += d.buf.bytes;
    };
    node(P0, A.n0, A.Pn0, A.sn0);
    node(P1, A.n1, A.Pn1, A.sn1);
    node(P2, A.n2, A.Pn2, A.sn2);
    edge(P0, P1, A.e01, A.Pe01, A.se01, A.sw01);
    edge(P1, P2, A.e12, A.Pe12, A.se12, A.sw12);
    edge(P2, P0, A.e20, A.Pe20, A.se20, A.sw20);
    A.out_kind = out.kind == TKind::Scalar ? 0 : out.kind == TKind::Vertex ? 1 : 2;
    A.out = out.data();
    A.Pout = out.P;
    if (out.kind != TKind::Scalar) bytes += out.buf.bytes;
    // histogram path (tri_hist_kernel): nothing depends on the third vertex
    // and at most one factor sits on the pivot
    const int nfixed = (A.n0 != nullptr) + (A.n1 != nullptr) + (A.e01 != nullptr);
    if (!per_w && nfixed <= 1) {
      TriHistArgs H{};
      H.nout = nout;
      H.cn_off = A.cn_off, H.cn_w = A.cn_w, H.out_src = A.out_src, H.out_nbr = A.out_nbr;
      H.out_slot = A.out_slot, H.rev = A.rev, H.chi = A.chi, H.k = k;
      H.s_out = sp.s_out;
      H.P2 = static_cast<uint32_t>(binom(k - 2, sp.s_out - 2));
      H.nterm = sp.s_out - 2;
      if (A.n0) H.fkind = 1, H.F = A.n0, H.PF = A.Pn0;
      else if (A.n1) H.fkind = 2, H.F = A.n1, H.PF = A.Pn1;
      else if (A.e01) H.fkind = 3, H.F = A.e01, H.PF = A.Pe01, H.sw01 = A.sw01;
      H.out_kind = A.out_kind, H.out = A.out, H.Pout = A.Pout;
      H.scalar = scalar, H.err = err, H.updates = upd;
      const size_t tsize = static_cast<size_t>(k) * k * H.P2 * H.nterm;
      const size_t isize = H.out_kind == 1 ? static_cast<size_t>(k) * k * H.P2 : 0;
      const size_t hsmem = (tsize + (isize + 1) / 2 + static_cast<size_t>(kHistWarps) * 32 * k) * 4;
      if (hsmem <= 200 * 1024) {
        if (hsmem > 48 * 1024)
          MB_CUDA(cudaFuncSetAttribute(tri_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem));
        const uint64_t nbatch = (nout + 31) / 32;
        const unsigned grid = static_cast<unsigned>(
            std::max<uint64_t>(1, std::min<uint64_t>((nbatch + kHistWarps - 1) / kHistWarps, 148 * 8)));
        if (nout)
          launch("tri_hist", [&] { tri_hist_kernel<<<grid, 32 * kHistWarps, hsmem, stream>>>(H); }, bytes);
        return;
      }
    }
    const size_t smem = static_cast<size_t>(kTriWarps) * (3 * kTriFixedCap + 2 * A.Pout + 2 + kMaxColors) * sizeof(u64);
    if (smem > 48 * 1024)
      MB_CUDA(cudaFuncSetAttribute(tri_edge_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((nout + kTriWarps - 1) / kTriWarps, 148 * 64));
    if (nout)
      launch("tri_edge_block", [&] { tri_edge_block_kernel<<<std::max(grid, 1u), 32 * kTriWarps, smem, stream>>>(A); },
             bytes);
  }

  TabView view(int tab) const {
    TabView v;
    if (tab < 0) return v;
    const DevTable& t = tables[tab];
    v.kind = t.kind == TKind::Scalar ? 1 : t.kind == TKind::Vertex ? 2 : t.kind == TKind::Edge ? 3
           : t.kind == TKind::Pair ? 4 : 0;
    v.s = t.s;
    v.P = t.P;
    v.data = t.data();
    if (t.kind == TKind::Pair) {
      v.off = t.off.as<uint64_t>(), v.cols = t.cols.as<uint32_t>();
      v.off_t = t.off_t.as<uint64_t>(), v.cols_t = t.cols_t.as<uint32_t>();
      v.data_t = t.buf_t.as<uint64_t>();
    }
    return v;
  }

  void run_general(const StepPlan& sp, int* err, u64* scalar, u64* upd) {
    CycleDesc C;
    C.L = sp.L;
    for (int q = 0; q < sp.L; ++q) C.node.push_back(view(sp.node_tab[q]));
    for (int e = 0; e < sp.L; ++e) C.edge.push_back(view(sp.edge_tab[e]));
    C.edge_fwd = sp.edge_fwd;
    C.bpos = sp.bpos;
    C.out = view(sp.block);
    C.s_out = sp.s_out;
    CycleRunner R;
    R.G = GraphView{n, m2, off.as<uint64_t>(), adj.as<uint32_t>(), rev.as<uint32_t>(), rank.as<uint32_t>(),
                    chi.as<uint8_t>()};
    R.k = k;
    int bits = 1;
    while (bits < 32 && (1ull << bits) < n) ++bits;
    R.bits = bits;
    const bool rec = sp.bpos.size() == 2;
    if ((rec ? 3 : 2) * bits > 64)
      fail(kSpec, "graph too large for the general cycle engine's packed keys");
    R.stream = stream;
    R.err = err;
    R.scalar = scalar;
    R.upd = upd;
    R.launch = [this](const char* name, const std::function<void()>& f) { launch(name, f); };
    R.scan = [this](const uint64_t* in, uint64_t* o, uint64_t c) { exclusive_scan(in, o, c); };
    R.solve(C);
    DevTable& out = tables[sp.block];
    if (out.kind == TKind::Pair) {
      R.finish_pairs(out.P, out.keys, out.buf, out.rows, out.off, out.cols, out.off_t, out.cols_t, out.buf_t);
    }
  }

  void count(const uint8_t* chi_src, int nc, bool host, uint64_t* result) {
    if (!plan_bound) fail(kSpec, "no plan bound");
    if (k == 1) {
      for (int c = 0; c < nc; ++c) result[c] = n;
      return;
    }
    if (needs_triangles) build_triangles();
    if (chi.bytes < std::max<uint64_t>(n, 1)) chi.alloc(std::max<uint64_t>(n, 1));
    int* err = flags.as<int>();
    u64* scalar = reinterpret_cast<u64*>(flags.as<char>() + 8);
    u64* upd = reinterpret_cast<u64*>(flags.as<char>() + 16);
    st.dp_updates = 0;
    if (host && chi_in.bytes < static_cast<uint64_t>(n) * nc) chi_in.alloc(std::max<uint64_t>(static_cast<uint64_t>(n) * nc, 1));
    if (host && n)
      MB_CUDA(cudaMemcpyAsync(chi_in.p, chi_src, static_cast<uint64_t>(n) * nc, cudaMemcpyHostToDevice, stream));
    const uint8_t* dchi = host ? chi_in.as<uint8_t>() : chi_src;
    std::vector<uint64_t> host_flags(3 * nc);
    DBuf res(static_cast<size_t>(nc) * 24);
    for (int c = 0; c < nc; ++c) {
      MB_CUDA(cudaMemsetAsync(flags.p, 0, 24, stream));
      if (n)
        launch("recolor", [&] {
          k_recolor<<<grid_for(n, 256), 256, 0, stream>>>(n, dchi + static_cast<uint64_t>(c) * n, chi.as<uint8_t>(), k, err);
        });
      for (const StepPlan& sp : steps) {
        DevTable& out = tables[sp.block];
        // outputs accumulated with atomics start from zero; the CN kernel writes
        // every row of its edge outputs and the leaf kernels every vertex row
        if ((out.kind == TKind::Edge && sp.general) || (out.kind == TKind::Vertex && sp.kind == BlockKind::Cycle))
          MB_CUDA(cudaMemsetAsync(out.buf.p, 0, out.buf.bytes, stream));
        if (sp.kind == BlockKind::Leaf) run_leaf(sp, err, upd);
        else if (sp.general) run_general(sp, err, scalar, upd);
        else run_tri_edge(sp, err, scalar, upd);
      }
      if (plan.singleton_root) {
        const DevTable& t = tables[plan.root];
        launch("table_total", [&] {
          k_table_total<<<296, 256, 0, stream>>>(t.data(), t.rows * t.P, scalar, err);
        });
      }
      MB_CUDA(cudaMemcpyAsync(res.as<char>() + 24 * c, flags.p, 24, cudaMemcpyDeviceToDevice, stream));
    }
    MB_CUDA(cudaMemcpyAsync(host_flags.data(), res.p, 24 * static_cast<size_t>(nc), cudaMemcpyDeviceToHost, stream));
    MB_CUDA(cudaStreamSynchronize(stream));
    if (timing) collect_timings();
    for (int c = 0; c < nc; ++c) {
      const int e = static_cast<int>(host_flags[3 * c] & 0xffffffffu);
      if (e & 2) fail(kSpec, "colouring has a colour outside 1..k");
      if (e & 4) fail(kInternal, "edge-keyed output received a non-adjacent vertex pair");
      if (e & 1) fail(kOverflow, "count overflow (64-bit)");
      result[c] = host_flags[3 * c + 1];
      st.dp_updates += host_flags[3 * c + 2];
    }
  }
};

namespace {
__global__ void k_gather_u32(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ src,
                             uint32_t* __restrict__ out, uint64_t count) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < count) out[i] = src[idx[i]];
}
}  // namespace

void GpuEngine::Impl::gather_src(const uint32_t* slots, uint32_t* outp, uint64_t count) {
  if (!count) return;
  launch("gather", [&] { k_gather_u32<<<grid_for(count, 256), 256, 0, stream>>>(slots, src.as<uint32_t>(), outp, count); });
}

GpuEngine::GpuEngine(const CsrGraph& g, int device) : impl_(new Impl) {
  impl_->device = device;
  MB_CUDA(cudaSetDevice(device));
  MB_CUDA(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking));
  impl_->upload(g);
}

GpuEngine::~GpuEngine() {
  if (!impl_) return;
  for (auto e : impl_->event_pool) cudaEventDestroy(e);
  for (auto& p : impl_->pending) {
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  if (impl_->stream) cudaStreamDestroy(impl_->stream);
}

uint32_t GpuEngine::num_vertices() const { return impl_->n; }
uint64_t GpuEngine::num_edges() const { return impl_->m2 / 2; }
void GpuEngine::bind_plan(const Plan& plan, int k) { impl_->bind(plan, k); }
void GpuEngine::count(const uint8_t* chi, int nc, bool host, uint64_t* out) { impl_->count(chi, nc, host, out); }
void GpuEngine::reset_derived() {
  impl_->tri_ready = false;
  impl_->cn.release();
  impl_->cn_off.release();
  impl_->out_nbr.release();
  impl_->out_slot.release();
  impl_->out_src.release();
}
void GpuEngine::enable_timing(bool on) {
  impl_->timing = on;
  impl_->timings.clear();
}
std::vector<GpuEngine::KernelTiming> GpuEngine::kernel_timings() const {
  std::vector<KernelTiming> v;
  for (auto& kv : impl_->timings) v.push_back(kv.second);
  return v;
}
uint64_t GpuEngine::launches() const { return impl_->launch_count; }
const EngineStats& GpuEngine::stats() const { return impl_->st; }
void* GpuEngine::stream() const { return impl_->stream; }

}  // namespace mb

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
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <utility>
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

// Device buffers are stream-ordered (cudaMallocAsync / cudaFreeAsync from the
// device's pool, which keeps freed blocks): the cycle engine allocates scratch
// per hop, and a plain cudaFree would synchronise the device every time.  A
// buffer is allocated on the calling thread's current engine stream
// (StreamScope) and freed on the stream it was allocated on.  `persistent`
// buffers (process-lifetime LUTs) use cudaMalloc.
thread_local cudaStream_t t_dbuf_stream = nullptr;
thread_local double t_dbuf_alloc_s = 0;  // host time in allocation calls (MB_DEBUG_BATCH)

struct StreamScope {  // sets the allocation stream for the engine entry point's duration
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(t_dbuf_stream) { t_dbuf_stream = s; }
  ~StreamScope() { t_dbuf_stream = prev; }
};

// Freed device blocks are cached per stream and handed to later requests of
// a similar size on the same stream (stream order makes the reuse safe):
// cudaMallocAsync alone spent up to 1 s per cycle-engine solve re-mapping
// pool memory (MB_DEBUG_BATCH).  Sizes are rounded to 64 KB (2 MB above
// 64 MB) classes; a cached block serves requests up to 25 % smaller.
struct DBufCache {
  std::mutex mu;
  std::map<cudaStream_t, std::multimap<size_t, void*>> blocks;
  size_t cached = 0;
  static constexpr size_t kCap = 24ull << 30;
  static size_t round(size_t b) {
    const size_t g = b > (64ull << 20) ? (2ull << 20) : (64ull << 10);
    return (b + g - 1) / g * g;
  }
  void* take(cudaStream_t s, size_t b, size_t* got) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = blocks.find(s);
    if (it == blocks.end()) return nullptr;
    auto jt = it->second.lower_bound(b);
    if (jt == it->second.end() || jt->first > b + b / 4) return nullptr;
    void* p = jt->second;
    *got = jt->first;
    cached -= jt->first;
    it->second.erase(jt);
    return p;
  }
  bool put(cudaStream_t s, size_t b, void* p) {
    std::lock_guard<std::mutex> lk(mu);
    if (cached + b > kCap) return false;
    blocks[s].emplace(b, p);
    cached += b;
    return true;
  }
  void clear(cudaStream_t s) {  // the stream is about to go away
    std::lock_guard<std::mutex> lk(mu);
    auto it = blocks.find(s);
    if (it == blocks.end()) return;
    for (auto& kv : it->second) {
      cudaFreeAsync(kv.second, s);
      cached -= kv.first;
    }
    blocks.erase(it);
  }
};
inline DBufCache& dbuf_cache() {
  static DBufCache* c = new DBufCache;  // never destroyed: outlives static engines at exit
  return *c;
}

// Bump arena for the cycle engine's per-batch scratch (frontiers, hash
// tables, work offsets): one block carved up in stream order and reset per
// anchor batch, instead of thousands of pool allocations per solve (those
// cost up to 10 s of host time per colouring on the theta query).
struct Arena {
  char* base = nullptr;
  size_t cap = 0, top = 0;
};
thread_local Arena* t_arena = nullptr;

struct ArenaScope {  // routes non-persistent DBuf allocations of this thread to `a` (nullptr: off)
  Arena* prev;
  explicit ArenaScope(Arena* a) : prev(t_arena) { t_arena = a; }
  ~ArenaScope() { t_arena = prev; }
};

struct DBuf {
  void* p = nullptr;
  size_t cap = 0;  // bytes actually allocated (size class)
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  bool persistent = false;
  bool in_arena = false;
  DBuf() = default;
  explicit DBuf(size_t b) { alloc(b); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept
      : p(o.p), cap(o.cap), bytes(o.bytes), s(o.s), persistent(o.persistent), in_arena(o.in_arena) {
    o.p = nullptr, o.bytes = 0, o.cap = 0, o.in_arena = false;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    p = o.p, cap = o.cap, bytes = o.bytes, s = o.s, persistent = o.persistent, in_arena = o.in_arena;
    o.p = nullptr, o.bytes = 0, o.cap = 0, o.in_arena = false;
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t b) {
    release();
    if (b && !persistent && t_arena) {
      const size_t r = (b + 255) & ~size_t(255);
      if (t_arena->top + r <= t_arena->cap) {
        p = t_arena->base + t_arena->top;
        t_arena->top += r;
        cap = r;
        bytes = b;
        in_arena = true;
        return;
      }
    }
    if (b) {
      if (persistent) {
        MB_CUDA(cudaMalloc(&p, b));
      } else {
        s = t_dbuf_stream;
        const auto t0 = std::chrono::steady_clock::now();
        cap = DBufCache::round(b);
        size_t got = 0;
        p = dbuf_cache().take(s, cap, &got);
        if (p) {
          cap = got;  // a cached block may be larger than asked for
        } else {
          cudaError_t e = cudaMallocAsync(&p, cap, s);
          if (e == cudaErrorMemoryAllocation) {
            // the size-class cache holds freed blocks the pool cannot hand
            // out for other sizes: give them all back and retry once
            (void)cudaGetLastError();  // not sticky: clear it for the next launch check
            dbuf_cache().clear(s);
            cudaMemPool_t pool;
            int dev = 0;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
              cudaStreamSynchronize(s);
              cudaMemPoolTrimTo(pool, 0);
            }
            e = cudaMallocAsync(&p, cap, s);
            if (e != cudaSuccess) (void)cudaGetLastError();
          }
          if (e != cudaSuccess)
            ::mb::fail(e == cudaErrorMemoryAllocation ? ::mb::kBudget : ::mb::kCuda,
                       std::string("device allocation of ") + std::to_string(cap >> 20) + " MB: " +
                           cudaGetErrorString(e));
        }
        t_dbuf_alloc_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
    }
    bytes = b;
  }
  void release() {
    if (p && in_arena) {
      p = nullptr, bytes = 0, cap = 0, in_arena = false;
      return;
    }
    if (p) {
      if (persistent) cudaFree(p);
      else if (!dbuf_cache().put(s, cap, p)) cudaFreeAsync(p, s);
    }
    p = nullptr;
    bytes = 0;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

__constant__ SigLut c_lut;

// Colourings are processed in batches of up to kChiStride: colours are stored
// interleaved [vertex][kChiStride] and every vertex/edge table is laid out
// [row][colouring][entry], so one pass over the graph serves the whole batch.
constexpr int kChiStride = 8;

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
    unrank.persistent = true;
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

// Colourings c0..c0+C-1 (row-major [colouring][vertex], colours 1..k) into the
// interleaved 0-based layout [vertex][kChiStride]; unused slots are zeroed.
// Row n is the dummy vertex the histogram kernels count for list slots past
// a row's end: colour 7 (never a real colour when k < 8) in every slot.
__global__ void k_recolor(uint32_t n, int C, const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int k,
                          int* err, const uint32_t* __restrict__ order) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v == n) reinterpret_cast<unsigned long long*>(out)[n] = 0x0707070707070707ull;
  if (v >= n) return;
  const uint32_t src = order[v];  // caller's id of device vertex v
  unsigned long long cols = 0;
#pragma unroll
  for (int c = 0; c < kChiStride; ++c) {
    if (c < C) {
      const int cc = in[static_cast<uint64_t>(c) * n + src];
      // an invalid colour raises SpecError after the batch; it is replaced by
      // colour 0 so that no kernel indexes its colour tables with it
      const bool ok = cc >= 1 && cc <= k;
      if (!ok) atomicOr(err, 2);
      cols |= static_cast<unsigned long long>(ok ? cc - 1 : 0) << (8 * c);
    }
  }
  reinterpret_cast<unsigned long long*>(out)[v] = cols;
}

// Seeded colourings on the device, bit-identical to random_coloring
// (reference graph.cpp:142-151: std::mt19937_64(seed), one draw per vertex in
// vertex order, draws >= limit = 2^64 - 1 - (2^64 - 1) % k rejected, colour
// 1 + x % k).  One 160-thread CTA per colouring: the 312-word MT state lives in
// shared memory and is regenerated 312 outputs at a time — the recurrence
// x[i] <- x[i+156] ^ twist(x[i], x[i+1]) is evaluated a half state per step,
// first i < 156 (reads only old words), then i >= 156 (reads the new lower
// half), which is the sequential order's data flow — then tempered, reduced
// mod k by a multiply-high, and compacted over rejections with ballots and a
// cross-warp prefix so the vertex order is exact.  estimate()'s trials therefore never cross PCIe:
// seeds in, counts out.
__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}
constexpr int kRngThreads = 160;  // 5 warps: one thread per element of a half state (156)
__global__ void __launch_bounds__(kRngThreads) k_random_colorings(const uint64_t* __restrict__ seeds, uint32_t n,
                                                                  uint32_t k, uint64_t limit,
                                                                  uint8_t* __restrict__ out) {
  constexpr int NN = 312, MM = 156;
  constexpr uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, MATRIX_A = 0xB5026F5AA96619E9ull;
  __shared__ uint64_t mt[NN];
  __shared__ uint32_t s_cnt[kRngThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint8_t* chi = out + static_cast<uint64_t>(blockIdx.x) * n;
  if (tid == 0) {
    uint64_t x = seeds[blockIdx.x];
    mt[0] = x;
    for (int i = 1; i < NN; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
      mt[i] = x;
    }
  }
  __syncthreads();
  const uint64_t magic = k > 1 ? ~0ull / k : 0;  // floor((2^64 - 1) / k): quotient estimate low by at most 1
  uint32_t v = 0;  // next vertex (the same in every thread)
  while (v < n) {
    // regenerate the state: each half in one step (reads of old words, barrier, writes)
    for (int half = 0; half < 2; ++half) {
      const int i = half * MM + static_cast<int>(tid);
      uint64_t nx = 0;
      if (tid < MM) {
        const uint64_t y = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
        nx = mt[(i + MM) % NN] ^ (y >> 1) ^ ((y & 1ull) ? MATRIX_A : 0ull);
      }
      __syncthreads();
      if (tid < MM) mt[i] = nx;
      __syncthreads();
    }
    // consume the 312 outputs in order, kRngThreads per step
    for (int base = 0; base < NN && v < n; base += kRngThreads) {
      const int i = base + static_cast<int>(tid);
      const uint64_t x = i < NN ? mt_temper(mt[i]) : ~0ull;
      const bool ok = i < NN && x < limit;
      const unsigned acc = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) s_cnt[wid] = __popc(acc);
      __syncthreads();
      uint32_t before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kRngThreads / 32; ++w) {
        const uint32_t c = s_cnt[w];
        before += w < static_cast<int>(wid) ? c : 0u;
        total += c;
      }
      const uint32_t dst = v + before + __popc(acc & ((1u << lane) - 1u));
      if (ok && dst < n) {
        uint64_t r = 0;
        if (k > 1) {
          const uint64_t q = __umul64hi(x, magic);
          r = x - q * k;
          if (r >= k) r -= k;
          if (r >= k) r -= k;
        }
        chi[dst] = static_cast<uint8_t>(1 + r);
      }
      v += total;
      __syncthreads();  // s_cnt is rewritten by the next step
    }
  }
}

// The kChiStride colours of vertex v (one 8-byte load) and colour slot c of them.
__device__ __forceinline__ uint64_t load_colors(const uint8_t* chi, uint32_t v) {
  return __ldg(reinterpret_cast<const unsigned long long*>(chi) + v);
}
__device__ __forceinline__ uint32_t color_of(uint64_t cols, int c) {
  return static_cast<uint32_t>(cols >> (8 * c)) & 0xFFu;
}
// 1 << (4 * colour of slot c) from the half word holding slots c & ~3 .. c | 3:
// the funnel shift uses the low 5 bits of its amount, and shifting the half
// right by 8*(c&3) - 2 leaves 4 * colour there (colours < 8 leave bits 6-7 of
// every byte zero, so nothing from the byte below leaks in).
__device__ __forceinline__ uint32_t nibble_onehot(uint32_t half, int c) {
  const uint32_t sh = (c & 3) ? (half >> (8 * (c & 3) - 2)) : (half << 2);
  return __funnelshift_l(0u, 1u, sh);
}

// flag1[v] = 1 when v is an endpoint of an oriented edge with a non-empty CN
// list (a vertex of some triangle), flag2[v] = 1 when of one with >= 2 entries.
__global__ void k_tri_vertices(uint64_t no, const uint64_t* __restrict__ cn_off, const uint32_t* __restrict__ src,
                               const uint32_t* __restrict__ nbr, uint8_t* __restrict__ flag1,
                               uint8_t* __restrict__ flag2) {
  const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (j >= no) return;
  const uint64_t len = cn_off[j + 1] - cn_off[j];
  if (len == 0) return;
  flag1[src[j]] = 1;
  flag1[nbr[j]] = 1;
  if (len < 2) return;
  flag2[src[j]] = 1;
  flag2[nbr[j]] = 1;
}

// Edge metadata in list-length order (eorder): meta[i] = (a, b, slot a->b,
// slot b->a) and range[i] = the CN list [lo, hi) of oriented edge eorder[i].
__global__ void k_edge_meta(uint64_t no, const uint32_t* __restrict__ eorder, const uint32_t* __restrict__ src,
                            const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ slot,
                            const uint32_t* __restrict__ rev, const uint64_t* __restrict__ cn_off,
                            uint4* __restrict__ meta, ulonglong2* __restrict__ range) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= no) return;
  const uint32_t j = eorder[i], s = slot[j];
  meta[i] = make_uint4(src[j], nbr[j], s, rev[s]);
  range[i] = make_ulonglong2(cn_off[j], cn_off[j + 1]);
}

// Warp-interleaved copy of the CN lists for the lane-per-edge kernels
// (tri_canon.cuh).  Batch bt holds the 32 edges at eorder positions
// [32 bt, 32 bt + 32); its lists are cut into 4-entry chunks and chunk ch of
// lane l is the uint4 at il[(base[bt] + ch) * 32 + l], so one 16-byte load per
// lane reads 512 contiguous bytes per warp (4 lines instead of 32 lane-private
// ones).  Lists shorter than the batch's longest are padded with the dummy
// vertex `pad` (colour 7 in every slot: counted in an unused nibble).
// k_il_count: nch[bt] = chunks of the batch's longest list.
__global__ void k_il_count(uint64_t no, const ulonglong2* __restrict__ range, uint64_t* __restrict__ nch) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  uint32_t c = 0;
  if (i < no) {
    const ulonglong2 r = range[i];
    c = static_cast<uint32_t>((r.y - r.x + 3) >> 2);
  }
  for (int o = 16; o > 0; o >>= 1) c = max(c, __shfl_xor_sync(0xffffffffu, c, o));
  if ((threadIdx.x & 31) == 0 && (i >> 5) < ((no + 31) >> 5)) nch[i >> 5] = c;
}
__global__ void k_il_fill(uint64_t no, const ulonglong2* __restrict__ range, const uint64_t* __restrict__ nch,
                          const uint64_t* __restrict__ base, const uint32_t* __restrict__ cw, uint32_t pad,
                          uint4* __restrict__ il, uint32_t* __restrict__ nch32) {
  const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (w >= ((no + 31) >> 5)) return;
  const uint64_t i = w * 32 + lane;
  ulonglong2 r = make_ulonglong2(0, 0);
  if (i < no) r = range[i];
  const uint32_t n = static_cast<uint32_t>(nch[w]);
  if (lane == 0) nch32[w] = n;
  uint4* dst = il + base[w] * 32 + lane;
  for (uint32_t ch = 0; ch < n; ++ch) {
    const uint64_t p = r.x + 4ull * ch;
    uint4 q;
    q.x = p < r.y ? cw[p] : pad;
    q.y = p + 1 < r.y ? cw[p + 1] : pad;
    q.z = p + 2 < r.y ? cw[p + 2] : pad;
    q.w = p + 3 < r.y ? cw[p + 3] : pad;
    dst[static_cast<uint64_t>(ch) * 32] = q;
  }
}

// Table exchange of vertex-sharded leaf blocks (GpuEngine::set_exchange): rank
// r owns the device vertices v with v % world == r; its rows are packed in
// ownership order (row i of the slice = vertex i * world + r) into slice r of
// the exchange buffer, and the other ranks' slices are scattered back into the
// table after the all-gather.  Rows are copied in units of U bytes.
template <class U>
__global__ void k_rows_pack(const U* __restrict__ table, U* __restrict__ slice, uint32_t n, uint32_t rank,
                            uint32_t world, uint64_t units_per_row, uint64_t rows) {
  const uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * units_per_row) return;
  const uint64_t i = idx / units_per_row, u = idx - i * units_per_row;
  const uint64_t v = i * world + rank;
  if (v < n) slice[idx] = table[v * units_per_row + u];
}
template <class U>
__global__ void k_rows_unpack(U* __restrict__ table, const U* __restrict__ buf, uint32_t n, uint32_t rank,
                              uint32_t world, uint64_t units_per_row, uint64_t rows) {
  const uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t per = rows * units_per_row;
  if (idx >= per * world) return;
  const uint64_t q = idx / per, r = idx - q * per;
  if (q == rank) return;
  const uint64_t i = r / units_per_row, u = r - i * units_per_row;
  const uint64_t v = i * world + q;
  if (v < n) table[v * units_per_row + u] = buf[idx];
}

// The same exchange restricted to a vertex list (leaf tables computed at the
// demanded vertices only): idx[q * rows + i] = the i-th listed vertex owned by
// rank q, ~0u past the end of q's share.
template <class U>
__global__ void k_rows_pack_idx(const U* __restrict__ table, U* __restrict__ slice, const uint32_t* __restrict__ idx,
                                uint64_t units_per_row, uint64_t rows) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (t >= rows * units_per_row) return;
  const uint64_t i = t / units_per_row, u = t - i * units_per_row;
  const uint32_t v = idx[i];
  if (v != ~0u) slice[t] = table[static_cast<uint64_t>(v) * units_per_row + u];
}
template <class U>
__global__ void k_rows_unpack_idx(U* __restrict__ table, const U* __restrict__ buf, const uint32_t* __restrict__ idx,
                                  uint32_t rank, uint32_t world, uint64_t units_per_row, uint64_t rows) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t per = rows * units_per_row;
  if (t >= per * world) return;
  const uint64_t q = t / per, r = t - q * per;
  if (q == rank) return;
  const uint64_t i = r / units_per_row, u = r - i * units_per_row;
  const uint32_t v = idx[q * rows + i];
  if (v != ~0u) table[static_cast<uint64_t>(v) * units_per_row + u] = buf[t];
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
  uint32_t rsa, rsb, rse, rso;  // row strides; pointers are pre-offset to one colouring
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
    const uint32_t cx = A.chi[static_cast<uint64_t>(x) * kChiStride], fx = 1u << cx;
    const uint64_t base = A.off[x], deg = A.off[x + 1] - base;
    const uint32_t pe = A.ue ? A.Pe : 1u, pb = A.ub ? A.Pb : 1u, per = pe * pb;
    const uint64_t items = deg * per;
    for (uint64_t it = lane; it < items; it += GROUP) {
      const uint64_t j = it / per;
      const uint32_t r = static_cast<uint32_t>(it - j * per);
      const uint32_t ie = r / pb, ib = r - ie * pb;
      const uint64_t slot = base + j;
      const uint32_t y = __ldg(A.adj + slot);
      const uint32_t cy = __ldg(A.chi + static_cast<uint64_t>(y) * kChiStride), fy = 1u << cy;
      if (cy == cx) continue;
      uint32_t M = fx | fy;
      uint64_t val = 1;
      if (A.ue) {
        const uint64_t e = A.e_rev ? __ldg(A.rev + slot) : slot;
        const uint64_t v = __ldg(A.ue + e * A.rse + ie);
        if (!v) continue;
        M = sig_expand(sig_unrank(c_lut, A.se - 2, ie), fx | fy);
        val = v;
      }
      if (A.ub) {
        const uint64_t v = __ldg(A.ub + static_cast<uint64_t>(y) * A.rsb + ib);
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
    const uint32_t cx = A.chi[static_cast<uint64_t>(x) * kChiStride], fx = 1u << cx;
    if (!A.ua) {
      for (uint32_t i = lane; i < A.Pout; i += GROUP) A.out[static_cast<uint64_t>(x) * A.rso + i] = Z[i];
    } else {
      const uint64_t items = static_cast<uint64_t>(A.PZ) * A.Pa;
      for (uint64_t it = lane; it < items; it += GROUP) {
        const uint32_t iz = static_cast<uint32_t>(it / A.Pa), ia = static_cast<uint32_t>(it - iz * A.Pa);
        const uint64_t z = Z[iz];
        if (!z) continue;
        const uint64_t a = __ldg(A.ua + static_cast<uint64_t>(x) * A.rsa + ia);
        if (!a) continue;
        const uint32_t Mz = sig_expand(sig_unrank(c_lut, A.sZ - 1, iz), fx);
        const uint32_t Ma = sig_expand(sig_unrank(c_lut, A.sa - 1, ia), fx);
        if ((Mz & Ma) != fx) continue;
        atomic_add_ck(&O[sig_index(c_lut, Mz | Ma, fx)], mul_ck(z, a, A.err), A.err);
        ++upd;
      }
      if (GROUP == 32) __syncwarp(); else __syncthreads();
      for (uint32_t i = lane; i < A.Pout; i += GROUP) A.out[static_cast<uint64_t>(x) * A.rso + i] = O[i];
    }
  }
  if (upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// Total of one colouring's slice of a table (singleton-root plans,
// reference engine.cpp:398): rows x P entries at row stride rs.
__global__ void k_table_total(const uint64_t* __restrict__ t, uint64_t rows, uint32_t P, uint32_t rs, u64* out,
                              int* err) {
  uint64_t local = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < rows * P;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    local = add_ck(local, t[(i / P) * rs + i % P], err);
  for (int o = 16; o > 0; o >>= 1) local = add_ck(local, __shfl_down_sync(0xffffffffu, local, o), err);
  if ((threadIdx.x & 31) == 0 && local) atomic_add_ck(out, local, err);
}

unsigned grid_for(uint64_t work, unsigned block) {
  const uint64_t g = (work + block - 1) / block;
  return static_cast<unsigned>(std::max<uint64_t>(1, g));
}

// Sort keys for the CN-length edge order: ~length so an ascending sort yields
// decreasing lengths.
// Sort key of oriented edge j for the lane-per-edge histogram kernels:
// decreasing CN-length bucket (quarter octaves, so a warp's 32 lists are
// within ~25% of each other), then j itself — oriented edges are stored by
// source vertex, so lanes of a warp share sources and their factor rows.
__global__ void k_cn_len_keys(const uint64_t* __restrict__ cn_off, uint64_t nout, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ vals, u64* __restrict__ nonempty,
                              unsigned* __restrict__ maxlen, uint32_t fmask /* fraction bits */) {
  const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t len = j < nout ? cn_off[j + 1] - cn_off[j] : 0;
  const unsigned nz = __ballot_sync(0xffffffffu, len > 0);
  if ((threadIdx.x & 31) == 0 && nz) atomicAdd(nonempty, static_cast<u64>(__popc(nz)));
  const unsigned n2 = __ballot_sync(0xffffffffu, len > 1);  // lists of >= 2 entries: nonempty[1]
  if ((threadIdx.x & 31) == 0 && n2) atomicAdd(nonempty + 1, static_cast<u64>(__popc(n2)));
  if (j >= nout) return;
  const uint32_t l = static_cast<uint32_t>(len > 0xFFFFFFFFull ? 0xFFFFFFFFull : len);
  if (l) atomicMax(maxlen, l);
  uint32_t bucket = 0;  // 0 for empty lists: sorted last
  if (l) {
    // fmask = number of fraction bits F: 2^F buckets per octave
    const uint32_t b = 31 - __clz(l), F = fmask;
    const uint32_t frac = b >= F ? (l >> (b - F)) & ((1u << F) - 1u) : (l << (F - b)) & ((1u << F) - 1u);
    bucket = 1 + (b << F) + frac;
    if (l == 1) bucket = 1;  // one-entry lists stay the last non-empty bucket
  }
  keys[j] = (static_cast<uint64_t>(0xFFFFu - bucket) << 32) | static_cast<uint32_t>(j);
  vals[j] = static_cast<uint32_t>(j);
}

__global__ void k_gather_u32(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ src,
                             uint32_t* __restrict__ out, uint64_t count) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < count) out[i] = src[idx[i]];
}

#include "engine_host.inc"

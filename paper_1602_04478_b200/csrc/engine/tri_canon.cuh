// Histogram-path 3-cycle blocks in relative colour coordinates.  Included by
// engine_host.inc after tri_edge.cuh (uses TriHistArgs and its helpers).
//
// Same work as tri_hist_kernel's lane mode (one lane per oriented edge, the
// common neighbours' colours counted in registers for all colourings of the
// batch), but the join is evaluated without per-term tables.  For a pivot
// colour pair {c0, c1} every colour set the block touches contains both, so
// it is a subset of the M = k - 2 remaining colours R = [k] \ {c0, c1} — and
// indexing R by rank ("relative coordinates") makes the whole join static:
//   stage 1  T[A] = sum_{r in A} h[r] * F'[A \ r]        |A| = s_out - 2
//   stage 2  U[A] = sum_{r in A} h[r] * T[A \ r]          |A| = s_parent - 2
// where h[r] is the histogram count of colour R[r] and F' the pivot factor's
// entries restricted to R.  Each relative subset A ranks to the row index of
// the squeezed colex layout (sig.cuh) directly for edge-keyed rows (the fixed
// colours are exactly {c0, c1}), so subset lists, ranks and term structure are
// compile-time constants and every product is a register multiply-add.  Only
// three things still depend on the lane's colours: which histogram counts
// form h (R[r] = r-th colour not in {c0, c1}), where a node factor keyed by one
// pivot colour keeps its R-entries (a per-CTA map over (c_f, c_other), 4 bits
// per entry packed in one word), and the index of a unary output entry (the
// idx1 maps).  A fused child + parent collapses into one bilinear form in h
// (see the BIL path below).
//
// Per edge: metadata and list range are read coalesced (permuted into the
// list-length order at prep) one iteration ahead; the list scan is a
// two-stage pipeline (lane_histogram_row); the colouring loop is unrolled
// twice only (instruction cache) with the factor gathers one colouring ahead.
// MB_TRI_DEBUG (timing split only; counts are wrong): 1 skips the join, 2
// the scan, 4 the factor gathers.
//
// Reference semantics: the same 3-cycle block evaluation by DB as
// tri_hist_kernel (engine.cpp:212-241, table.cpp:135-284 for the joins).

namespace canon {

constexpr int cbinom(int n, int r) {
  if (r < 0 || r > n) return 0;
  int b = 1;
  for (int i = 1; i <= r; ++i) b = b * (n - r + i) / i;
  return b;
}
constexpr int cpopc(uint32_t x) {
  int c = 0;
  for (; x; x &= x - 1u) ++c;
  return c;
}
// j-th t-subset of {0..m-1} in colex order (= increasing mask value)
constexpr uint32_t nth_subset(int m, int t, int j) {
  int cnt = 0;
  for (uint32_t x = 0; x < (1u << m); ++x)
    if (cpopc(x) == t) {
      if (cnt == j) return x;
      ++cnt;
    }
  return 0;
}
// colex rank among masks of the same popcount (sig_rank with constant binomials)
constexpr int crank(uint32_t mask) {
  int r = 0, i = 1;
  for (int c = 0; c < 32; ++c)
    if ((mask >> c) & 1u) r += cbinom(c, i++);
  return r;
}
// the b-th set bit of mask (b counted from the lowest)
constexpr int nth_bit(uint32_t mask, int b) {
  for (int c = 0; c < 32; ++c)
    if ((mask >> c) & 1u) {
      if (b == 0) return c;
      --b;
    }
  return -1;
}

template <class F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
// f(integral_constant<int, i>) for i = 0..N-1, fully expanded at compile time
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl(f, std::make_integer_sequence<int, N>{});
}

}  // namespace canon

// The lane's histogram row for oriented edge j, written to hrow[c*K + d]
// (u16: lane-mode lists are shorter than 65536).  Three counter levels keep
// the per-entry work to one funnel shift and one add per colouring:
//   N[c]  4-bit fields, all colours of colouring slot c in one word (an entry
//         adds 1 << (4 * colour): one shift and one funnel shift,
//         nibble_onehot), moved every 12 entries into
//   B[c]  8-bit fields (even / odd colours), moved every 240 entries into
//   hrow  the 16-bit row in shared memory (read-modify-write, rare).
// The list is read with 16-byte loads, the next chunk in flight while the
// current one is counted.  For K < 8 slots outside the list count vertex
// A.nv, whose colours are 7 (unused) in every slot, so the inner loop
// has no branches; for K = 8 they are skipped.
#ifndef MB_HIST_PIPE
#define MB_HIST_PIPE 1  // measured 0.876 vs 0.896 ms per config-1 batch
#endif
template <int K>
__device__ __forceinline__ void lane_histogram_row(const TriHistArgs& A, uint64_t lo, uint64_t hi, uint16_t* hrow) {
  uint32_t N[kChiStride], Be[kChiStride], Bo[kChiStride];
#pragma unroll
  for (int c = 0; c < kChiStride; ++c) N[c] = Be[c] = Bo[c] = 0;
  bool spilled = false;
  auto flushN = [&]() {
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
      Be[c] += N[c] & 0x0F0F0F0Fu;
      Bo[c] += (N[c] >> 4) & 0x0F0F0F0Fu;
      N[c] = 0;
    }
  };
  auto flushB = [&]() {
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
#pragma unroll
      for (int d = 0; d < K; ++d) {
        const uint32_t v = (((d & 1) ? Bo[c] : Be[c]) >> (8 * (d >> 1))) & 0xFFu;
        hrow[c * K + d] = static_cast<uint16_t>(spilled ? hrow[c * K + d] + v : v);
      }
      Be[c] = Bo[c] = 0;
    }
    spilled = true;
  };
  const uint64_t p0 = lo & ~3ull;
  const uint32_t head = static_cast<uint32_t>(lo - p0), n = static_cast<uint32_t>(hi - p0);
  const uint32_t nch = (n + 3) >> 2;
  const uint4* src = reinterpret_cast<const uint4*>(A.cn_w + p0);
  int pend = 0, nfl = 0;
#if MB_HIST_PIPE
  // two-stage pipeline: list chunk ch+2 and the colours of chunk ch+1 are in
  // flight while chunk ch is counted
  auto gather = [&](const uint4& qq, uint32_t ch, uint64_t (&cw)[4]) {
    const uint32_t ws[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t idx = 4 * ch + u;
      const bool in = idx >= head && idx < n;
      if (K < 8) cw[u] = load_colors(A.chi, in ? ws[u] : A.nv);
      else cw[u] = in ? load_colors(A.chi, ws[u]) : ~0ull;
    }
  };
  uint4 q1 = nch > 1 ? __ldg(src + 1) : make_uint4(0, 0, 0, 0);
  uint64_t cwc[4];
  {
    const uint4 q0 = nch ? __ldg(src) : make_uint4(0, 0, 0, 0);
    gather(q0, 0, cwc);
  }
  for (uint32_t ch = 0; ch < nch; ++ch) {
    const uint4 q2 = ch + 2 < nch ? __ldg(src + ch + 2) : q1;
    uint64_t cwn[4];
    gather(q1, ch + 1, cwn);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (K == 8 && cwc[u] == ~0ull) continue;
      const uint32_t lo32 = static_cast<uint32_t>(cwc[u]), hi32 = static_cast<uint32_t>(cwc[u] >> 32);
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        const uint32_t half = c < 4 ? lo32 : hi32;
        N[c] += nibble_onehot(half, c);
      }
    }
    if (++pend == 3) {
      flushN();
      pend = 0;
      if (++nfl == 20) {
        flushB();
        nfl = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) cwc[u] = cwn[u];
    q1 = q2;
  }
#else
  uint4 q = nch ? __ldg(src) : make_uint4(0, 0, 0, 0);
  for (uint32_t ch = 0; ch < nch; ++ch) {
    const uint4 qn = ch + 1 < nch ? __ldg(src + ch + 1) : q;
    const uint32_t ws[4] = {q.x, q.y, q.z, q.w};
    uint64_t cw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t idx = 4 * ch + u;
      const bool in = idx >= head && idx < n;
      if (K < 8) cw[u] = load_colors(A.chi, in ? ws[u] : A.nv);
      else cw[u] = in ? load_colors(A.chi, ws[u]) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (K == 8 && cw[u] == ~0ull) continue;
      const uint32_t lo32 = static_cast<uint32_t>(cw[u]), hi32 = static_cast<uint32_t>(cw[u] >> 32);
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        const uint32_t half = c < 4 ? lo32 : hi32;
        N[c] += nibble_onehot(half, c);
      }
    }
    if (++pend == 3) {
      flushN();
      pend = 0;
      if (++nfl == 20) {
        flushB();
        nfl = 0;
      }
    }
    q = qn;
  }
#endif
  flushN();
  flushB();
}

// The same histogram row from the warp-interleaved list copy (TriHistArgs::il):
// `src` is the lane's first chunk, chunks are 32 uint4 apart, and every lane of
// the warp runs the batch's `nch` chunks (shorter lists are padded with the
// dummy vertex A.nv), so the loop is warp-uniform and a warp's chunk load is
// 512 contiguous bytes.  Chunks are loaded three ahead and their colours
// gathered one ahead of the counting.
template <int K>
__device__ __forceinline__ void lane_histogram_row_il(const TriHistArgs& A, const uint4* __restrict__ src,
                                                      uint32_t nch, uint16_t* hrow) {
  uint32_t N[kChiStride], Be[kChiStride], Bo[kChiStride];
#pragma unroll
  for (int c = 0; c < kChiStride; ++c) N[c] = Be[c] = Bo[c] = 0;
  bool spilled = false;
  auto flushN = [&]() {
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
      Be[c] += N[c] & 0x0F0F0F0Fu;
      Bo[c] += (N[c] >> 4) & 0x0F0F0F0Fu;
      N[c] = 0;
    }
  };
  auto flushB = [&]() {
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
#pragma unroll
      for (int d = 0; d < K; ++d) {
        const uint32_t v = (((d & 1) ? Bo[c] : Be[c]) >> (8 * (d >> 1))) & 0xFFu;
        hrow[c * K + d] = static_cast<uint16_t>(spilled ? hrow[c * K + d] + v : v);
      }
      Be[c] = Bo[c] = 0;
    }
    spilled = true;
  };
  auto gather = [&](const uint4& qq, uint64_t (&cw)[4]) {
    const uint32_t ws[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (K < 8) cw[u] = load_colors(A.chi, ws[u]);
      else cw[u] = ws[u] != A.nv ? load_colors(A.chi, ws[u]) : ~0ull;
    }
  };
  const uint4 pad = make_uint4(A.nv, A.nv, A.nv, A.nv);
  auto chunk = [&](uint32_t ch) { return ch < nch ? __ldg(src + static_cast<uint64_t>(ch) * 32) : pad; };
  int pend = 0, nfl = 0;
  uint4 q1 = chunk(1), q2 = chunk(2);
  uint64_t cwc[4];
  gather(chunk(0), cwc);
  for (uint32_t ch = 0; ch < nch; ++ch) {
    const uint4 q3 = chunk(ch + 3);
    uint64_t cwn[4];
    gather(q1, cwn);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (K == 8 && cwc[u] == ~0ull) continue;
      const uint32_t lo32 = static_cast<uint32_t>(cwc[u]), hi32 = static_cast<uint32_t>(cwc[u] >> 32);
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        const uint32_t half = c < 4 ? lo32 : hi32;
        N[c] += nibble_onehot(half, c);
      }
    }
    if (++pend == 3) {
      flushN();
      pend = 0;
      if (++nfl == 20) {
        flushB();
        nfl = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) cwc[u] = cwn[u];
    q1 = q2;
    q2 = q3;
  }
  flushN();
  flushB();
}

// K colours; S1 = this block's s_out; FK = pivot factor kind (0 none, 1 node
// at P0, 2 node at P1, 3 edge (P0, P1)); SP = the fused parent's s_out (0: not
// fused); NARROW = node factor stored as u32.
// BIL: fused shape whose host bound allows only the bilinear path (the
// general two-stage code is not compiled in: fewer live registers).
#ifndef MB_BIL_MINB
#define MB_BIL_MINB MB_TRI_MINB
#endif
template <int K, int S1, int FK, int SP, bool NARROW, bool BIL = false>
__global__ void __launch_bounds__(32 * kHistWarps, BIL ? MB_BIL_MINB : MB_TRI_MINB) tri_canon_kernel(TriHistArgs A) {
  constexpr int M = K - 2;                       // |R|
  constexpr int T1 = S1 - 2;                     // stage-1 subset size
  constexpr int P2 = canon::cbinom(M, T1);       // stage-1 entries
  constexpr int NB = FK ? canon::cbinom(M, T1 - 1) : 1;  // factor entries restricted to R
  constexpr int TP = SP ? SP - 2 : 0;
  constexpr int P2p = SP ? canon::cbinom(M, TP) : 0;
  static_assert(K <= 8 && T1 >= 1 && (FK != 0 || T1 == 1), "shape");

  extern __shared__ uint32_t hsm[];
  // per-CTA maps: fmap[(cf*K + cx)*NB + j] = row index, in the node factor keyed
  // by colour cf, of the j-th (T1-1)-subset of R = [K] \ {cf, cx};
  // idx1/idx1p[(c0*K + c1)*P + i] = unary-output index of relative entry i
  // rows of <= 16 entries: the NB indices of a colour pair packed 4 bits each in one word
  constexpr bool PACK = (FK == 1 || FK == 2) && NB <= 8 && canon::cbinom(K - 1, T1 - 1) <= 16;
  constexpr int FMAP = (FK == 1 || FK == 2) ? K * K * (NB > 4 ? NB : 4) : 0;
  uint8_t* fmap = reinterpret_cast<uint8_t*>(hsm);
  uint16_t* idx1 = reinterpret_cast<uint16_t*>(hsm + (FMAP + 3) / 4);
  const int n1 = A.out_kind == 1 ? K * K * P2 : 0;
  uint16_t* idx1p = idx1 + n1;
  const int n1p = (SP && A.pout_kind == 1) ? K * K * P2p : 0;
  uint16_t* hist16_base = idx1p + n1p + ((n1 + n1p) & 1);  // 4-byte aligned
  for (int i = threadIdx.x; i < (FMAP + 3) / 4; i += blockDim.x) hsm[i] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < K * K * (NB + P2 + P2p); e += blockDim.x) {
    // one pass over (c0, c1, slot) triples fills whichever maps this launch needs
    const int q = e / (K * K), pr = e % (K * K), c0 = pr / K, c1 = pr % K;
    if (c0 == c1) continue;
    const uint32_t f2 = (1u << c0) | (1u << c1);
    if (q < NB) {
      if (FMAP) {
        const uint32_t S = sig_expand(sig_unrank(c_lut, T1 - 1, q), f2) & ~(1u << c1);
        const uint32_t ix = sig_index(c_lut, S, 1u << c0);
        if (PACK) atomicOr(reinterpret_cast<uint32_t*>(fmap) + pr, ix << (4 * q));
        else fmap[pr * NB + q] = static_cast<uint8_t>(ix);
      }
    } else if (q < NB + P2) {
      const int i = q - NB;
      if (n1) idx1[pr * P2 + i] = static_cast<uint16_t>(sig_index(c_lut, sig_expand(sig_unrank(c_lut, T1, i), f2), 1u << c0));
    } else {
      const int i = q - NB - P2;
      if (n1p)
        idx1p[pr * P2p + i] = static_cast<uint16_t>(sig_index(c_lut, sig_expand(sig_unrank(c_lut, TP, i), f2), 1u << c0));
    }
  }
  __syncthreads();

  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t LS = 2 * ((((kChiStride * K) + 1) / 2) | 1u);  // u16 per edge row, odd word stride
  uint16_t* hrow = hist16_base + static_cast<size_t>(threadIdx.x) * LS;
  const int C = A.C;
  uint32_t ovf = 0;
  // per-thread scalar sums per colouring slot in shared memory ([c][thread]):
  // the rolled colouring loop indexes them dynamically
  u64* lsum = reinterpret_cast<u64*>(
      (reinterpret_cast<uintptr_t>(hist16_base + static_cast<size_t>(blockDim.x) * LS) + 7) & ~uintptr_t(7));
#pragma unroll
  for (int c = 0; c < kChiStride; ++c) lsum[c * blockDim.x + threadIdx.x] = 0;
  uint64_t upd = 0;
  const uint64_t nbatch = (A.nitems + 31) / 32;
  // edge metadata one iteration ahead (its DRAM latency would otherwise
  // stall every edge)
  // vertex sharding (TriHistArgs::shard_*): this rank visits the warp batches
  // bt with bt % world == rank (list-length order: every rank gets its share
  // of long and short lists)
  const uint64_t bstride = static_cast<uint64_t>(gridDim.x) * kHistWarps * A.shard_world;
  uint64_t bt = (static_cast<uint64_t>(blockIdx.x) * kHistWarps + wid) * A.shard_world + A.shard_rank;
  uint4 emn = make_uint4(0, 0, 0, 0);
  ulonglong2 ern = make_ulonglong2(0, 0);
  if (bt * 32 + lane < A.nitems) emn = A.emeta[bt * 32 + lane], ern = A.erange[bt * 32 + lane];
  for (; bt < nbatch; bt += bstride) {
    const uint64_t jj = bt * 32 + lane;
    const uint4 em = emn;
    const ulonglong2 er = ern;
    const uint64_t jn = jj + bstride * 32;
    if (jn < A.nitems) emn = A.emeta[jn], ern = A.erange[jn];
    if (jj >= A.nitems) continue;
    const uint32_t a = em.x, b = em.y, sab = em.z, sba = em.w;
    if (!(A.debug & 2)) {
      if (A.il) lane_histogram_row_il<K>(A, A.il + __ldg(A.ilbase + bt) * 32 + lane, __ldg(A.ilnch + bt), hrow);
      else lane_histogram_row<K>(A, er.x, er.y, hrow);
    }
    if (A.debug & 1) continue;
    const uint64_t cas = load_colors(A.chi, a), cbs = load_colors(A.chi, b);
    uint32_t updl = 0;
    using FT = typename std::conditional<NARROW, uint32_t, uint64_t>::type;
    // F'[o][q]: the pivot factor's entry for the q-th (T1-1)-subset of R in
    // orientation o; loaded one colouring ahead of its use
    auto load_f = [&](int c, FT (&Fo)[2][NB]) {
      const uint32_t ca = color_of(cas, c), cb = color_of(cbs, c);
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
        if (FK == 0 || (A.debug & 4)) {
#pragma unroll
          for (int q = 0; q < NB; ++q) Fo[o][q] = 1;
        } else if (ca == cb) {
#pragma unroll
          for (int q = 0; q < NB; ++q) Fo[o][q] = 0;
        } else if (FK == 3) {
          const uint64_t s = (o == 0) != (A.sw01 != 0) ? sab : sba;
          const uint64_t* row = A.F + s * A.rsF + c * A.psF;
#pragma unroll
          for (int q = 0; q < NB; ++q) Fo[o][q] = static_cast<FT>(__ldg(row + q));
        } else {
          const uint32_t v = FK == 1 ? (o ? b : a) : (o ? a : b);
          const uint32_t cf = FK == 1 ? c0 : c1, cx = FK == 1 ? c1 : c0;
          const uint8_t* mp = fmap + (cf * K + cx) * NB;
          const uint32_t pk = PACK ? reinterpret_cast<const uint32_t*>(fmap)[cf * K + cx] : 0u;
          const uint64_t ro = static_cast<uint64_t>(v) * A.rsF + c * A.psF;
#pragma unroll
          for (int q = 0; q < NB; ++q) {
            const uint32_t ix = PACK ? (pk >> (4 * q)) & 15u : mp[q];
            if (NARROW) Fo[o][q] = static_cast<FT>(__ldg(reinterpret_cast<const uint32_t*>(A.F) + ro + ix));
            else Fo[o][q] = static_cast<FT>(__ldg(A.F + ro + ix));
          }
        }
      }
    };
    FT Fc[2][NB];
    load_f(0, Fc);
    // unrolled twice only: the 8-fold body overflowed the instruction cache
    // (ncu: 16 % of stall samples "no_instructions"); 2 lets the compiler
    // rename the Fc/Fn double buffer instead of copying it (1 % faster than 1)
#pragma unroll 2
    for (int c = 0; c < C; ++c) {
      FT Fn[2][NB];
      if (c + 1 < C) load_f(c + 1, Fn);  // in flight while colouring c is joined
      const uint32_t ca = color_of(cas, c), cb = color_of(cbs, c);
      if (ca == cb) {
        // no colourful match on this edge: materialised edge rows are zero
        if (A.out_kind == 2)
          for (int o = 0; o < 2; ++o)
            for (uint32_t i = 0; i < A.Pout; ++i) A.out[static_cast<uint64_t>(o ? sba : sab) * A.rso + c * A.Pout + i] = 0;
        if (SP && A.pout_kind == 2)
          for (int o = 0; o < 2; ++o)
            for (uint32_t i = 0; i < A.Poutp; ++i)
              A.pout[static_cast<uint64_t>(o ? sba : sab) * A.rsop + c * A.Poutp + i] = 0;
      } else {
      const uint32_t lo = min(ca, cb), hi = max(ca, cb);
      // h[r] = count of the r-th colour not in {ca, cb}
      uint32_t h[M];
#pragma unroll
      for (int r = 0; r < M; ++r) {
        uint32_t d = r;
        d += d >= lo;
        d += d >= hi;
        h[r] = hrow[c * K + d];
      }
      uint64_t acc = 0;
      if (BIL || (SP && A.t_safe)) {
        // Fused child and parent as one bilinear form in h: with
        //   T[S] = sum_{r' in S} h[r'] F'[S \ r'],  U[A] = sum_{r in A} h[r] T[A \ r]
        // U[A] = 2 * sum over pairs {r, r'} in A of h[r] h[r'] F'[A \ {r, r'}].
        // The pair products (< 2^32) are shared by both orientations; every
        // term is one 32x32->64 (or 32x64) multiply-add, and the host bound on
        // the child's entries (< 2^44) keeps U below 2^63.
        constexpr int NPAIR = M * (M - 1) / 2;
        uint32_t PP[NPAIR > 0 ? NPAIR : 1];
        canon::sfor<M>([&](auto r1c) {
          canon::sfor<M>([&](auto r2c) {
            constexpr int r1 = decltype(r1c)::value, r2 = decltype(r2c)::value;
            if constexpr (r1 < r2) PP[canon::crank((1u << r1) | (1u << r2))] = h[r1] * h[r2];
          });
        });
        auto pairs = [&](int o, const FT (&Fs)[NB]) {
          const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
          canon::sfor<P2p>([&](auto ii) {
            constexpr int i = decltype(ii)::value;
            constexpr uint32_t Ai = canon::nth_subset(M, TP, i);
            uint64_t v = 0;
            canon::sfor<M>([&](auto r1c) {
              canon::sfor<M>([&](auto r2c) {
                constexpr int r1 = decltype(r1c)::value, r2 = decltype(r2c)::value;
                if constexpr (r1 < r2 && ((Ai >> r1) & 1u) && ((Ai >> r2) & 1u)) {
                  constexpr uint32_t pr = (1u << r1) | (1u << r2);
                  constexpr int q = FK ? canon::crank(Ai & ~pr) : 0;
                  v += static_cast<uint64_t>(PP[canon::crank(pr)]) * Fs[q];
                }
              });
            });
            v *= 2;
            updl += v != 0;
            if (A.pout_kind == 2) {
              A.pout[static_cast<uint64_t>(o ? sba : sab) * A.rsop + c * A.Poutp + i] = v;
            } else if (A.pout_kind == 0) {
              acc += v;
              ovf |= acc < v;
            } else if (v) {
              atomic_add_ck(reinterpret_cast<u64*>(A.pout) + static_cast<uint64_t>(o ? b : a) * A.rsop +
                                c * A.Poutp + idx1p[(c0 * K + c1) * P2p + i],
                            v, A.err);
            }
          });
        };
        if (A.pout_kind == 0 || !A.sw01p) {
          pairs(0, Fc[0]);
          pairs(1, Fc[1]);
        } else {
          pairs(0, Fc[1]);
          pairs(1, Fc[0]);
        }
      } else if constexpr (!BIL) {
      uint64_t T[2][P2];
      uint64_t tmax = 0;
      // stage-1 products stay below 2^63 when every factor entry is < 2^44
      // (host bound, or a u32 table): counters < 2^16, at most 6 terms
      const bool safe = A.f_safe != 0 || NARROW || FK == 0;
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
        // stage 1: T[i] = sum over r in A_i of h[r] * F'[A_i \ r]
        canon::sfor<P2>([&](auto ii) {
          constexpr int i = decltype(ii)::value;
          constexpr uint32_t Ai = canon::nth_subset(M, T1, i);
          uint64_t v = 0;
          canon::sfor<T1>([&](auto bb) {
            constexpr int r = canon::nth_bit(Ai, decltype(bb)::value);
            constexpr int q = FK ? canon::crank(Ai & ~(1u << r)) : 0;
            const uint64_t f = Fc[o][q];
            if (safe) {
              v += f * h[r];
            } else {
              ovf |= __umul64hi(f, h[r]) != 0;
              const uint64_t fh = f * h[r];
              v += fh;
              ovf |= v < fh;
            }
          });
          T[o][i] = v;
          tmax |= v;
          if (!SP) {  // unfused: this block's output
            updl += v != 0;
            if (A.out_kind == 2) {
              A.out[static_cast<uint64_t>(o ? sba : sab) * A.rso + c * A.Pout + i] = v;
            } else if (A.out_kind == 0) {
              acc += v;
              ovf |= acc < v;
            } else if (v) {
              atomic_add_ck(reinterpret_cast<u64*>(A.out) + static_cast<uint64_t>(o ? b : a) * A.rso + c * A.Pout +
                                idx1[(c0 * K + c1) * P2 + i],
                            v, A.err);
            }
          }
        });
      }
      if (SP) {
        // stage 2: the fused parent on the same edge and histogram; its pivot
        // factor is this block's row for the orientation it reads (a scalar
        // output sums both orientations, so any pairing gives the same total)
        const bool safe2 = A.t_safe != 0 || (tmax >> 44) == 0;
        auto stage2 = [&](int o, const uint64_t (&Ts)[P2]) {
          const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
          canon::sfor<P2p>([&](auto ii) {
            constexpr int i = decltype(ii)::value;
            constexpr uint32_t Ai = canon::nth_subset(M, TP, i);
            uint64_t v = 0;
            canon::sfor<TP>([&](auto bb) {
              constexpr int r = canon::nth_bit(Ai, decltype(bb)::value);
              constexpr int q = canon::crank(Ai & ~(1u << r));
              const uint64_t f = Ts[q];
              if (safe2) {
                v += f * h[r];
              } else {
                ovf |= __umul64hi(f, h[r]) != 0;
                const uint64_t fh = f * h[r];
                v += fh;
                ovf |= v < fh;
              }
            });
            updl += v != 0;
            if (A.pout_kind == 2) {
              A.pout[static_cast<uint64_t>(o ? sba : sab) * A.rsop + c * A.Poutp + i] = v;
            } else if (A.pout_kind == 0) {
              acc += v;
              ovf |= acc < v;
            } else if (v) {
              atomic_add_ck(reinterpret_cast<u64*>(A.pout) + static_cast<uint64_t>(o ? b : a) * A.rsop +
                                c * A.Poutp + idx1p[(c0 * K + c1) * P2p + i],
                            v, A.err);
            }
          });
        };
        if (A.pout_kind == 0 || !A.sw01p) {
          stage2(0, T[0]);
          stage2(1, T[1]);
        } else {
          stage2(0, T[1]);
          stage2(1, T[0]);
        }
      }
      }
      if (acc) {
        u64& ls = lsum[c * blockDim.x + threadIdx.x];
        ls += acc;
        ovf |= ls < acc;
      }
      }
      if (c + 1 < C) {
#pragma unroll
        for (int o = 0; o < 2; ++o)
#pragma unroll
          for (int q = 0; q < NB; ++q) Fc[o][q] = Fn[o][q];
      }
    }
    upd += updl;
  }
  const bool scalar_out = (!SP && A.out_kind == 0) || (SP && A.pout_kind == 0);
  if (scalar_out) {
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
      uint64_t v = lsum[c * blockDim.x + threadIdx.x];
      for (int o = 16; o > 0; o >>= 1) v = add_ck(v, __shfl_down_sync(0xffffffffu, v, o), A.err);
      if (lane == 0 && v) atomic_add_ck(A.scalars + c, v, A.err);
    }
  }
  if (ovf) atomicOr(A.err, 1);
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if (lane == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// Shared-memory bytes of a tri_canon_kernel launch (the kernel's carve-up).
inline size_t tri_canon_smem(int K, int S1, int FK, int SP, int out_kind, int pout_kind) {
  auto bn = [](int n, int r) { return canon::cbinom(n, r); };
  const int M = K - 2, NB = FK ? bn(M, S1 - 3) : 1, P2 = bn(M, S1 - 2), P2p = SP ? bn(M, SP - 2) : 0;
  const int FMAP = (FK == 1 || FK == 2) ? K * K * (NB > 4 ? NB : 4) : 0;
  const int n1 = out_kind == 1 ? K * K * P2 : 0, n1p = (SP && pout_kind == 1) ? K * K * P2p : 0;
  const size_t LS = 2 * ((((kChiStride * K) + 1) / 2) | 1);
  return static_cast<size_t>((FMAP + 3) / 4) * 4 + 2 * static_cast<size_t>(n1 + n1p + ((n1 + n1p) & 1)) +
         static_cast<size_t>(32 * kHistWarps) * LS * 2 + 8 + static_cast<size_t>(32 * kHistWarps) * kChiStride * 8;
}

using TriCanonFn = void (*)(TriHistArgs);

// The instantiated shapes (K, S1, FK, SP, NARROW); others use tri_hist_kernel.
template <int K, int S1, int FK, int SP, bool N, bool BIL = false>
constexpr TriCanonFn canon_ptr() {
  if constexpr (S1 <= K && SP <= K && S1 >= 3 && (FK != 0 || S1 == 3) && K <= 8 && (!BIL || SP))
    return tri_canon_kernel<K, S1, FK, SP, N, BIL>;
  else return nullptr;
}
inline TriCanonFn tri_canon_find(int K, int S1, int FK, int SP, bool narrow, bool bil) {
  if (bil) {  // the config-1 shapes, and the same two-triangle + pendant-path shape at k = 7
    if (K == 6 && S1 == 5 && FK == 1 && SP == 6 && narrow) return canon_ptr<6, 5, 1, 6, true, true>();
    if (K == 6 && S1 == 5 && FK == 2 && SP == 6 && narrow) return canon_ptr<6, 5, 2, 6, true, true>();
    // two triangles on the pivot edge with a pendant tree at one pivot end,
    // fused into the root, at k = 5 and 7 (k - 1 = child size, k = root size)
    if (K == 5 && S1 == 4 && FK == 1 && SP == 5 && narrow) return canon_ptr<5, 4, 1, 5, true, true>();
    if (K == 5 && S1 == 4 && FK == 2 && SP == 5 && narrow) return canon_ptr<5, 4, 2, 5, true, true>();
    if (K == 7 && S1 == 6 && FK == 1 && SP == 7 && narrow) return canon_ptr<7, 6, 1, 7, true, true>();
    if (K == 7 && S1 == 6 && FK == 2 && SP == 7 && narrow) return canon_ptr<7, 6, 2, 7, true, true>();
  }
  // two triangles on one edge (diamond-like fused pairs) and plain triangles
  // at k = 3, 4, 5, 7
  if (!narrow && FK == 0 && S1 == 3 && (SP == 0 || SP == 4)) {
    if (K == 3 && !SP) return canon_ptr<3, 3, 0, 0, false>();
    if (K == 4) return SP ? canon_ptr<4, 3, 0, 4, false>() : canon_ptr<4, 3, 0, 0, false>();
    if (K == 5) return SP ? canon_ptr<5, 3, 0, 4, false>() : canon_ptr<5, 3, 0, 0, false>();
    if (K == 7) return SP ? canon_ptr<7, 3, 0, 4, false>() : canon_ptr<7, 3, 0, 0, false>();
  }
#define MB_CANON(k_, s_, f_, p_, n_) \
  if (K == k_ && S1 == s_ && FK == f_ && SP == p_ && narrow == n_) return canon_ptr<k_, s_, f_, p_, n_>();
#define MB_CANON_K(k_)                                                                                    \
  MB_CANON(k_, 3, 0, 0, false) MB_CANON(k_, 3, 0, 4, false)                                               \
  MB_CANON(k_, 4, 1, 0, false) MB_CANON(k_, 4, 1, 0, true) MB_CANON(k_, 4, 2, 0, false)                   \
  MB_CANON(k_, 4, 2, 0, true) MB_CANON(k_, 4, 3, 0, false) \
  MB_CANON(k_, 5, 1, 6, false) MB_CANON(k_, 5, 1, 6, true) MB_CANON(k_, 5, 2, 6, false)                   \
  MB_CANON(k_, 5, 2, 6, true)
  // the full shape list for k = 6 (the config-1 query and its trees) only:
  // each instance costs seconds of compile time; other shapes use
  // tri_hist_kernel
  MB_CANON_K(6)
#undef MB_CANON_K
#undef MB_CANON
  return nullptr;
}

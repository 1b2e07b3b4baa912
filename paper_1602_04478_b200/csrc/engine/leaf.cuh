// Leaf blocks, table-driven and colouring-batched.  Included by engine.cu.
//
// Path-table extension along CSR rows (paper §5.2 leaf blocks; reference
// engine.cpp:243-257: edge table -> node join on the leaf -> node join on the
// boundary -> projection to the boundary).  For a boundary vertex x the leaf
// side contributes, for every neighbour y, the row U_b[y] shifted by x's
// colour.  Which output colour-set index an entry (colour of x, colour of y,
// entry ib of U_b's row) lands in depends only on (chi x, chi y, ib), so the
// colour-set arithmetic is precomputed into a shared-memory map and the inner
// loop is: neighbour id, its colours, its rows, add through the map.
//
// Colouring batch: tables are laid out [row][colouring][entry] and colours
// [vertex][8], so one pass over x's CSR row serves all C colourings of the
// batch — the neighbour ids are read once and each neighbour's C rows are one
// contiguous span.
//
// Degree-binned scheduling: a warp per light vertex, a 256-thread CTA per
// heavy vertex (degree >= 512), so hubs do not serialise a warp.

struct LeafMapArgs {
  const uint64_t* off;
  const uint32_t* adj;
  const uint8_t* chi;  // [n][kChiStride], 0-based colours
  uint32_t nv;  // vertex count = the dummy row of chi (colour 7 in every slot)
  const uint64_t* ub;  // node child on the leaf (row = img b), may be null
  const uint64_t* ua;  // node child on the boundary (row = img a), may be null
  uint32_t Pb, Pa, PZ, Pout;
  uint32_t rsb, rsa, rso;  // row strides (C_alloc * P)
  int sb, sa, sZ, k, C;
  int unchecked;  // entries provably < 2^62 (host bound): plain adds
  uint32_t psb, psa, pso;  // per-colouring row strides: P, or 8 for padded u16 rows (bind())
  int ub_e, ua_e, out_e;  // entry bytes of the tables: 8, or narrow 4 (u32) / 2 (u16), see bind()
  uint64_t* out;
  int* err;
  u64* updates;
};

// entry idx of a table stored with `e` bytes per entry (8, 4 or 2)
__device__ __forceinline__ uint64_t ld_entry(const uint64_t* t, uint64_t idx, int e) {
  if (e == 2) return __ldg(reinterpret_cast<const uint16_t*>(t) + idx);
  if (e == 4) return __ldg(reinterpret_cast<const uint32_t*>(t) + idx);
  return __ldg(t + idx);
}
__device__ __forceinline__ void st_entry(uint64_t* t, uint64_t idx, int e, uint64_t v) {
  if (e == 2) reinterpret_cast<uint16_t*>(t)[idx] = static_cast<uint16_t>(v);
  else if (e == 4) reinterpret_cast<uint32_t*>(t)[idx] = static_cast<uint32_t>(v);
  else t[idx] = v;
}

__device__ __forceinline__ uint32_t leaf_map_size(const LeafMapArgs& A) {
  return static_cast<uint32_t>(A.k) * A.k * (A.ub ? A.Pb : 1u);
}

// Acc: the shared-memory accumulator type — uint32_t when the host's entry
// bound (maxdeg^(s-1)) is below 2^32 (native 32-bit shared atomics, half the
// banks), else u64 (checked unless the bound is below 2^62).
// PB: the child row length when it is a compile-time constant (common query
// shapes: 4, 5, 6, 10), else 0 = read from A.Pb — a constant row unrolls the
// loads and the consume loop exactly (no guarded 8-wide chunks).
template <int GROUP, class Acc, int PB>
__global__ void __launch_bounds__(256)
leaf_map_kernel(LeafMapArgs A, const uint32_t* __restrict__ vlist, uint32_t nv) {
  constexpr bool k32 = sizeof(Acc) == 4;
  extern __shared__ u64 lsm[];
  const int kThreads = blockDim.x;
  const int kGroups = kThreads / GROUP;
  const uint32_t msize = leaf_map_size(A);
  uint16_t* map = reinterpret_cast<uint16_t*>(lsm);
  Acc* acc = reinterpret_cast<Acc*>(lsm + (msize * 2 + 7) / 8);
  const uint32_t pb = PB ? static_cast<uint32_t>(PB) : (A.ub ? A.Pb : 1u);
  for (uint32_t i = threadIdx.x; i < msize; i += kThreads) {
    const uint32_t ib = i % pb, cy = (i / pb) % A.k, cx = i / (pb * A.k);
    uint16_t t = 0xFFFF;
    if (cx != cy) {
      const uint32_t fx = 1u << cx, fy = 1u << cy;
      const uint32_t Mb = A.ub ? sig_expand(sig_unrank(c_lut, A.sb - 1, ib), fy) : fy;
      if (!(Mb & fx)) t = static_cast<uint16_t>(sig_index(c_lut, Mb | fx, fx));
    }
    map[i] = t;
  }
  __syncthreads();
  const int g = threadIdx.x / GROUP, lane = threadIdx.x % GROUP;
  const uint32_t gstride = A.C * (A.PZ + A.Pout);
  // a CTA-sized group keeps one accumulator copy per warp (no cross-warp
  // contention on the same counters) and sums the copies at the end
  constexpr int kWarpsPerGroup = GROUP / 32;
  Acc* Zg = acc + static_cast<size_t>(g) * gstride * kWarpsPerGroup;
  Acc* Z = Zg;                      // [C][PZ] then [C][Pout]: the reduced copy
  Acc* Zw = Zg + (lane / 32) * gstride;  // this warp's copy
  Acc* O = Z + A.C * A.PZ;
  uint32_t upd = 0;  // per-thread contribution count (dp_updates)
  const bool cpow2 = (A.C & (A.C - 1)) == 0;  // full batches: C = 8
  const int clog = __ffs(A.C) - 1;
  for (uint32_t gi = blockIdx.x * kGroups + g; gi < nv; gi += gridDim.x * kGroups) {
    const uint32_t x = vlist[gi];
    for (uint32_t i = lane; i < gstride * kWarpsPerGroup; i += GROUP) Zg[i] = 0;
    if (GROUP == 32) __syncwarp(); else __syncthreads();
    const uint64_t cxs = load_colors(A.chi, x);
    const uint64_t base = A.off[x];
    const uint32_t deg = static_cast<uint32_t>(A.off[x + 1] - base);
    // one lane per (neighbour, colouring): low-degree rows still fill the
    // warp, and a neighbour's C rows are read as one contiguous span
    const uint32_t items = deg * static_cast<uint32_t>(A.C);
    if (PB > 0 && PB <= 8 && A.ub && A.ub_e != 8 && (k32 || A.unchecked)) {
      // constant child row: two items per lane in flight (their neighbour
      // ids, colours and rows are all loaded before either is consumed)
      constexpr int PBc = PB > 0 && PB <= 8 ? PB : 1;
      for (uint32_t it0 = lane; it0 < items; it0 += 2 * GROUP) {
        uint32_t y[2], cy[2];
        int cc[2];
        bool ok[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t it = it0 + u * GROUP;
          ok[u] = it < items;
          const uint32_t j = cpow2 ? it >> clog : it / static_cast<uint32_t>(A.C);
          cc[u] = static_cast<int>(it - j * static_cast<uint32_t>(A.C));
          y[u] = ok[u] ? __ldg(A.adj + base + j) : 0u;
        }
        uint32_t r[2][PBc];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          cy[u] = ok[u] ? A.chi[static_cast<uint64_t>(y[u]) * kChiStride + cc[u]] : 0xFFu;
          const uint64_t roff = static_cast<uint64_t>(y[u]) * A.rsb + cc[u] * A.psb;
          if (A.ub_e == 2) {
#pragma unroll
            for (int e = 0; e < PBc; ++e) r[u][e] = ok[u] ? ld_entry(A.ub, roff + e, 2) : 0u;
          } else {
#pragma unroll
            for (int e = 0; e < PBc; ++e) r[u][e] = ok[u] ? ld_entry(A.ub, roff + e, 4) : 0u;
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (!ok[u]) continue;
          const uint32_t cx = color_of(cxs, cc[u]);
          if (cy[u] == cx) continue;
          const uint16_t* my = map + (cx * A.k + cy[u]) * PBc;
          Acc* Zc = Zw + cc[u] * A.PZ;
#pragma unroll
          for (int e = 0; e < PBc; ++e) {
            if (!r[u][e]) continue;
            const uint16_t t = my[e];
            if (t == 0xFFFF) continue;
            atomicAdd(Zc + t, static_cast<Acc>(r[u][e]));
            ++upd;
          }
        }
      }
    } else for (uint32_t it = lane; it < items; it += GROUP) {
      const uint32_t j = cpow2 ? it >> clog : it / static_cast<uint32_t>(A.C);
      const int c = static_cast<int>(it - j * static_cast<uint32_t>(A.C));
      const uint32_t y = __ldg(A.adj + base + j);
      const uint32_t cx = color_of(cxs, c), cy = A.chi[static_cast<uint64_t>(y) * kChiStride + c];
      const uint16_t* my = map + (cx * A.k + cy) * pb;
      Acc* Zc = Zw + c * A.PZ;
      if (!A.ub) {
        const uint16_t t = my[0];
        if (t != 0xFFFF) {
          atomicAdd(Zc + t, static_cast<Acc>(1));
          ++upd;
        }
        continue;
      }
      if (cy == cx) continue;
      const uint64_t roff = static_cast<uint64_t>(y) * A.rsb + c * A.psb;
      for (uint32_t i0 = 0; i0 < pb; i0 += 8) {
        // the row's loads are issued together, then consumed
        uint64_t r[8];
        if (A.ub_e == 2) {
#pragma unroll
          for (int u = 0; u < 8; ++u) r[u] = i0 + u < pb ? ld_entry(A.ub, roff + i0 + u, 2) : 0u;
        } else if (A.ub_e == 4) {
#pragma unroll
          for (int u = 0; u < 8; ++u) r[u] = i0 + u < pb ? ld_entry(A.ub, roff + i0 + u, 4) : 0u;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) r[u] = i0 + u < pb ? ld_entry(A.ub, roff + i0 + u, 8) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (!r[u]) continue;
          const uint16_t t = my[i0 + u];
          if (t == 0xFFFF) continue;
          if (k32 || A.unchecked) atomicAdd(Zc + t, static_cast<Acc>(r[u]));
          else atomic_add_ck(reinterpret_cast<u64*>(Zc + t), r[u], A.err);
          ++upd;
        }
      }
    }
    if (GROUP == 32) {
      __syncwarp();
    } else {
      __syncthreads();
      for (uint32_t i = lane; i < A.C * A.PZ; i += GROUP) {
        uint64_t s = Zg[i];
        for (int w = 1; w < kWarpsPerGroup; ++w)
          s = (k32 || A.unchecked) ? s + Zg[w * gstride + i] : add_ck(s, Zg[w * gstride + i], A.err);
        Z[i] = static_cast<Acc>(s);
      }
      __syncthreads();
    }
    if (!A.ua) {
      for (uint32_t i = lane; i < A.C * A.Pout; i += GROUP)
        st_entry(A.out, static_cast<uint64_t>(x) * A.rso + (i / A.Pout) * A.pso + i % A.Pout, A.out_e,
                 static_cast<uint64_t>(Z[i]));
    } else {
      const uint64_t per = static_cast<uint64_t>(A.PZ) * A.Pa;
      for (uint64_t it = lane; it < per * A.C; it += GROUP) {
        const int c = static_cast<int>(it / per);
        const uint64_t r = it - c * per;
        const uint32_t iz = static_cast<uint32_t>(r / A.Pa), ia = static_cast<uint32_t>(r - iz * A.Pa);
        const uint64_t z = Z[c * A.PZ + iz];
        if (!z) continue;
        const uint64_t aoff = static_cast<uint64_t>(x) * A.rsa + c * A.psa + ia;
        const uint64_t a = ld_entry(A.ua, aoff, A.ua_e);
        if (!a) continue;
        const uint32_t fx = 1u << color_of(cxs, c);
        const uint32_t Mz = sig_expand(sig_unrank(c_lut, A.sZ - 1, iz), fx);
        const uint32_t Ma = sig_expand(sig_unrank(c_lut, A.sa - 1, ia), fx);
        if ((Mz & Ma) != fx) continue;
        if (k32 || A.unchecked) atomicAdd(O + c * A.Pout + sig_index(c_lut, Mz | Ma, fx), static_cast<Acc>(z * a));
        else atomic_add_ck(reinterpret_cast<u64*>(O + c * A.Pout + sig_index(c_lut, Mz | Ma, fx)), mul_ck(z, a, A.err),
                           A.err);
        ++upd;
      }
      if (GROUP == 32) __syncwarp(); else __syncthreads();
      for (uint32_t i = lane; i < A.C * A.Pout; i += GROUP)
        st_entry(A.out, static_cast<uint64_t>(x) * A.rso + (i / A.Pout) * A.pso + i % A.Pout, A.out_e,
                 static_cast<uint64_t>(O[i]));
    }
    if (GROUP == 32) __syncwarp(); else __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// First leaf level (no child tables on either end): the row of x is, per
// colouring, the colour histogram of x's neighbours without x's own colour —
// entry of colour d is d - [d > chi x] (the squeezed rank of {d}).  For light
// vertices (degree < 512, k <= 8) a thread owns one vertex and counts all
// colourings in registers: 4-bit fields (k <= 8 colours in one word) flushed
// every 12 neighbours into 16-bit fields, as in the 3-cycle histograms.  No
// shared memory, no atomics; vertices arrive in degree order, so a warp's
// rows have similar lengths.
// K: the colour count when known at compile time (vector row stores), else 0.
template <int K>
__global__ void __launch_bounds__(256) leaf_hist_kernel(LeafMapArgs A, const uint32_t* __restrict__ vlist,
                                                        uint32_t nv) {
  const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t upd = 0;
  if (gi < nv) {
    const uint32_t x = vlist[gi];
    uint32_t N[kChiStride], H[kChiStride][4];
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
      N[c] = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) H[c][w] = 0;
    }
    auto flush = [&]() {
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        const uint32_t ev = N[c] & 0x0F0F0F0Fu, od = (N[c] >> 4) & 0x0F0F0F0Fu;
#pragma unroll
        for (int w = 0; w < 4; ++w) H[c][w] += ((ev >> (8 * w)) & 0xFFu) | (((od >> (8 * w)) & 0xFFu) << 16);
        N[c] = 0;
      }
    };
    const uint64_t base = A.off[x], end = A.off[x + 1];
    int pend = 0;
    // 16-byte loads of the row (adj is padded by 16 bytes on upload), in a
    // two-stage pipeline as in the 3-cycle list scan: chunk i+2 and the
    // colours of chunk i+1 are in flight while chunk i is counted; slots
    // outside the row count the dummy vertex (colour 7, unused when k < 8)
    const uint64_t p0 = base & ~3ull;
    const uint32_t head = static_cast<uint32_t>(base - p0), nn = static_cast<uint32_t>(end - p0);
    const uint32_t nch = (nn + 3) >> 2;
    const uint4* src = reinterpret_cast<const uint4*>(A.adj + p0);
    const bool k8 = A.k >= 8;
    auto gather = [&](const uint4& qq, uint32_t ch, uint64_t (&cw)[4]) {
      const uint32_t ws[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t idx = 4 * ch + u;
        const bool in = idx >= head && idx < nn;
        cw[u] = k8 ? (in ? load_colors(A.chi, ws[u]) : ~0ull) : load_colors(A.chi, in ? ws[u] : A.nv);
      }
    };
    uint4 q1 = nch > 1 ? __ldg(src + 1) : make_uint4(0, 0, 0, 0);
    uint64_t cwc[4];
    gather(nch ? __ldg(src) : make_uint4(0, 0, 0, 0), 0, cwc);
    for (uint32_t ch = 0; ch < nch; ++ch) {
      const uint4 q2 = ch + 2 < nch ? __ldg(src + ch + 2) : q1;
      uint64_t cwn[4];
      gather(q1, ch + 1, cwn);
      uint64_t cw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) cw[u] = cwc[u], cwc[u] = cwn[u];
      q1 = q2;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (cw[u] == ~0ull) continue;
        const uint32_t lo32 = static_cast<uint32_t>(cw[u]), hi32 = static_cast<uint32_t>(cw[u] >> 32);
#pragma unroll
        for (int c = 0; c < kChiStride; ++c) {
          const uint32_t half = c < 4 ? lo32 : hi32;
          N[c] += 1u << (((half >> (8 * (c & 3))) & 7u) << 2);
        }
      }
      if (++pend == 3) {
        flush();
        pend = 0;
      }
    }
    flush();
    const uint64_t cxs = load_colors(A.chi, x);
    if (K > 0 && K <= 9 && A.out_e == 2 && A.pso == 8) {
      // padded u16 row: one 16-byte store per colouring (entries past K-1 are 0)
      constexpr int P = K > 0 ? K - 1 : 1;
      uint4* orow = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(A.out) + static_cast<uint64_t>(x) * A.rso);
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        const uint32_t cx = color_of(cxs, c);
        uint32_t q[4] = {0, 0, 0, 0};
#pragma unroll
        for (int e = 0; e < P && e < 8; ++e) {
          const uint32_t lo = (H[c][e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
          const uint32_t hi = (H[c][(e + 1) >> 1] >> (16 * ((e + 1) & 1))) & 0xFFFFu;
          const uint32_t v = c < A.C ? (static_cast<uint32_t>(e) >= cx ? hi : lo) : 0u;
          upd += v != 0;
          q[e >> 1] |= v << (16 * (e & 1));
        }
        orow[c] = make_uint4(q[0], q[1], q[2], q[3]);
      }
    } else if (K > 0 && A.out_e == 2 && A.pso == A.Pout) {
      // u16 row: two entries per word
      constexpr int P = K > 0 ? K - 1 : 1, W = kChiStride * P;
      uint4* orow = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(A.out) + static_cast<uint64_t>(x) * A.rso);
      uint32_t q[4];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int c = w / P, e = w % P;
        const uint32_t cx = color_of(cxs, c);
        const uint32_t lo = (H[c][e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
        const uint32_t hi = (H[c][(e + 1) >> 1] >> (16 * ((e + 1) & 1))) & 0xFFFFu;
        const uint32_t v = c < A.C ? (static_cast<uint32_t>(e) >= cx ? hi : lo) : 0u;
        upd += v != 0;
        if (w & 1) q[(w >> 1) & 3] |= v << 16;
        else q[(w >> 1) & 3] = v;
        if ((w & 7) == 7) orow[w >> 3] = make_uint4(q[0], q[1], q[2], q[3]);
      }
    } else if (K > 0 && A.out_e == 4 && A.pso == A.Pout) {
      // the whole row (kChiStride colourings x (K-1) entries, 16-byte aligned)
      // as 16-byte stores: entry e of colouring c is colour e or e + 1
      // (squeezed past chi x), a select between two static fields
      constexpr int P = K > 0 ? K - 1 : 1, W = kChiStride * P;
      uint4* orow = reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(A.out) + static_cast<uint64_t>(x) * A.rso);
      uint32_t q[4];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int c = w / P, e = w % P;
        const uint32_t cx = color_of(cxs, c);
        const uint32_t lo = (H[c][e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
        const uint32_t hi = (H[c][(e + 1) >> 1] >> (16 * ((e + 1) & 1))) & 0xFFFFu;
        const uint32_t v = c < A.C ? (static_cast<uint32_t>(e) >= cx ? hi : lo) : 0u;
        upd += v != 0;
        q[w & 3] = v;
        if ((w & 3) == 3) orow[w >> 2] = make_uint4(q[0], q[1], q[2], q[3]);
      }
    } else {
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
      if (c >= A.C) break;
      const uint32_t cx = color_of(cxs, c);
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        if (d >= A.k || d == static_cast<int>(cx)) continue;
        const uint32_t v = (H[c][d >> 1] >> (16 * (d & 1))) & 0xFFFFu;
        const uint32_t col = c * A.pso + d - (d > static_cast<int>(cx) ? 1 : 0);
        st_entry(A.out, static_cast<uint64_t>(x) * A.rso + col, A.out_e, v);
        upd += v != 0;
      }
    }
    }
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}


// First leaf level for heavy vertices (degree >= 512): a CTA per vertex, each
// thread counts a strided slice of the row in registers as leaf_hist_kernel
// does, then the CTA sums the packed 16-bit counters (warp shuffles, then
// across warps in shared memory).  Counts stay below 2^16 (the host checks
// maxdeg < 65536).  Replaces one shared-memory atomic per (neighbour,
// colouring) on a few hot counters.
__global__ void __launch_bounds__(256) leaf_hist_heavy_kernel(LeafMapArgs A, const uint32_t* __restrict__ vlist,
                                                              uint32_t nv) {
  __shared__ uint32_t red[8][kChiStride * 4];
  uint64_t upd = 0;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t gi = blockIdx.x; gi < nv; gi += gridDim.x) {
    const uint32_t x = vlist[gi];
    uint32_t N[kChiStride], H[kChiStride][4];
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
      N[c] = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) H[c][w] = 0;
    }
    auto flush = [&]() {
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        const uint32_t ev = N[c] & 0x0F0F0F0Fu, od = (N[c] >> 4) & 0x0F0F0F0Fu;
#pragma unroll
        for (int w = 0; w < 4; ++w) H[c][w] += ((ev >> (8 * w)) & 0xFFu) | (((od >> (8 * w)) & 0xFFu) << 16);
        N[c] = 0;
      }
    };
    const uint64_t base = A.off[x], end = A.off[x + 1];
    int pend = 0;
    for (uint64_t p = base + threadIdx.x; p < end; p += 256) {
      const uint64_t cw = load_colors(A.chi, __ldg(A.adj + p));
      const uint32_t lo32 = static_cast<uint32_t>(cw), hi32 = static_cast<uint32_t>(cw >> 32);
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        const uint32_t half = c < 4 ? lo32 : hi32;
        N[c] += 1u << (((half >> (8 * (c & 3))) & 7u) << 2);
      }
      if (++pend == 15) {
        flush();
        pend = 0;
      }
    }
    flush();
#pragma unroll
    for (int c = 0; c < kChiStride; ++c)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t v = H[c][w];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[wid][c * 4 + w] = v;
      }
    __syncthreads();
    if (threadIdx.x < kChiStride * 8) {
      const int c = threadIdx.x >> 3, d = threadIdx.x & 7;
      if (c < A.C && d < A.k) {
        const uint32_t cx = color_of(load_colors(A.chi, x), c);
        if (d != static_cast<int>(cx)) {
          uint32_t v = 0;
#pragma unroll
          for (int w = 0; w < 8; ++w) v += red[w][c * 4 + (d >> 1)];
          v = (v >> (16 * (d & 1))) & 0xFFFFu;
          st_entry(A.out, static_cast<uint64_t>(x) * A.rso + c * A.pso + d - (d > static_cast<int>(cx) ? 1 : 0),
                   A.out_e, v);
          upd += v != 0;
        }
      }
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if (lane == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// Leaf block with a child row on the leaf side and no annotation on the
// boundary (U_out[x] = sum over neighbours y of U_b[y] shifted by chi(x)),
// light vertices: a thread per (vertex, colouring slot) — 8 consecutive lanes
// share a vertex, a warp covers 4 vertices of similar degree.  Each thread
// walks its vertex's row and adds the child entries into private accumulators
// (shared memory, odd stride, uncontended shared atomics), then writes its
// output row; the 8 rows of a vertex are one contiguous span.  The output
// slots of a child row for colours (cx, cy) come from one packed map word
// (5 bits per entry, 31 = the entry holds cx).  UNR neighbours are in flight
// per thread.  Requires entries < 2^32 (host bound), a narrow child table,
// PB <= 12 and Pout < 31.
__device__ __forceinline__ void build_pmap(const LeafMapArgs& A, int PB, uint64_t* pmap) {
  for (uint32_t i = threadIdx.x; i < static_cast<uint32_t>(A.k * A.k); i += blockDim.x) {
    const uint32_t cy = i % A.k, cx = i / A.k;
    uint64_t w = ~0ull;
    if (cx != cy) {
      w = 0;
      for (int ib = 0; ib < PB; ++ib) {
        const uint32_t fx = 1u << cx, fy = 1u << cy;
        const uint32_t Mb = sig_expand(sig_unrank(c_lut, A.sb - 1, ib), fy);
        const uint64_t t = (Mb & fx) ? 31u : sig_index(c_lut, Mb | fx, fx);
        w |= t << (5 * ib);
      }
    }
    pmap[i] = w;
  }
}

template <int PB, int UNR, int EB>
__global__ void __launch_bounds__(256) leaf_pull_kernel(LeafMapArgs A, const uint32_t* __restrict__ vlist,
                                                        uint32_t nv) {
  extern __shared__ u64 lsm[];
  uint64_t* pmap = reinterpret_cast<uint64_t*>(lsm);
  uint32_t* accs = reinterpret_cast<uint32_t*>(lsm + A.k * A.k);
  build_pmap(A, PB, pmap);
  __syncthreads();
  // slot-major private accumulators (acc[slot * blockDim]): a lane always
  // hits bank lane % 32 whatever slot its data selects, so the data-dependent
  // slots never conflict (thread-major rows measured 2.1e7 bank conflicts per
  // launch, ncu r01zb).  One spare slot past Pout: map entries that hold x's
  // colour (slot code 31) land there, so the add loop has no branches.
  uint32_t* acc = accs + threadIdx.x;
  const uint32_t AS = blockDim.x;
  const int c = threadIdx.x & 7;
  uint32_t upd = 0;
  const uint32_t gpc = blockDim.x >> 3;  // vertex groups (of 8 slots) per CTA
  for (uint32_t gi = blockIdx.x * gpc + (threadIdx.x >> 3); gi < nv; gi += gridDim.x * gpc) {
    if (c >= A.C) continue;
    const uint32_t x = vlist[gi];
    for (uint32_t i = 0; i < A.Pout; ++i) acc[i * AS] = 0;
    const uint32_t cx = A.chi[static_cast<uint64_t>(x) * kChiStride + c];
    const uint64_t* mx = pmap + cx * A.k;
    const uint64_t base = A.off[x], end = A.off[x + 1];
    // neighbour ids one group ahead: the colour and row gathers of a group
    // do not wait behind its own id loads
    uint32_t yn[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) yn[u] = base + u < end ? __ldg(A.adj + base + u) : 0u;
    for (uint64_t p = base; p < end; p += UNR) {
      uint32_t y[UNR], cy[UNR], r[UNR][PB];
      bool ok[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        ok[u] = p + u < end;
        y[u] = yn[u];
      }
      if (p + UNR < end) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) yn[u] = p + UNR + u < end ? __ldg(A.adj + p + UNR + u) : 0u;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        cy[u] = ok[u] ? A.chi[static_cast<uint64_t>(y[u]) * kChiStride + c] : cx;
        const uint64_t roff = static_cast<uint64_t>(y[u]) * A.rsb + c * A.psb;
        if (PB <= 8 && EB == 2 && A.psb == 8) {
          // padded u16 row: one 16-byte load
          const uint4 v4 = ok[u] ? __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(A.ub) + roff))
                                 : make_uint4(0, 0, 0, 0);
          const uint32_t wv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int e = 0; e < PB; ++e) r[u][e] = (wv[(e >> 1) & 3] >> (16 * (e & 1))) & 0xFFFFu;
        } else {
#pragma unroll
          for (int e = 0; e < PB; ++e) r[u][e] = ok[u] ? ld_entry(A.ub, roff + e, EB) : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (cy[u] == cx) continue;
        const uint64_t w = mx[cy[u]];
#pragma unroll
        for (int e = 0; e < PB; ++e) {
          const uint32_t t = min(static_cast<uint32_t>(w >> (5 * e)) & 31u, A.Pout);
          atomicAdd(acc + t * AS, r[u][e]);
          upd += (t < A.Pout) & (r[u][e] != 0);
        }
      }
    }
    for (uint32_t i = 0; i < A.Pout; ++i)
      st_entry(A.out, static_cast<uint64_t>(x) * A.rso + c * A.pso + i, A.out_e, acc[i * AS]);
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// Heavy-vertex counterpart of leaf_pull_kernel: a CTA per vertex, thread t
// owns colouring slot t & 7 and every 32nd neighbour from t >> 3 (the 8 rows
// of a neighbour are read by 8 consecutive lanes), private accumulators, then
// the 32 partial rows of each colouring are summed in shared memory.
template <int PB, int UNR>
__global__ void __launch_bounds__(256) leaf_pull_heavy_kernel(LeafMapArgs A, const uint32_t* __restrict__ vlist,
                                                              uint32_t nv) {
  extern __shared__ u64 lsm[];
  uint64_t* pmap = reinterpret_cast<uint64_t*>(lsm);
  uint32_t* accs = reinterpret_cast<uint32_t*>(lsm + A.k * A.k);
  build_pmap(A, PB, pmap);
  // slot-major (acc[slot * blockDim]): conflict-free data-dependent slots
  const uint32_t AS = blockDim.x;
  uint32_t* acc = accs + threadIdx.x;
  const int c = threadIdx.x & 7, jl = threadIdx.x >> 3;
  uint32_t upd = 0;
  for (uint32_t gi = blockIdx.x; gi < nv; gi += gridDim.x) {
    const uint32_t x = vlist[gi];
    __syncthreads();  // map ready (first vertex) / previous vertex's sums read
    for (uint32_t i = 0; i < A.Pout; ++i) acc[i * AS] = 0;
    if (c < A.C) {
      const uint32_t cx = A.chi[static_cast<uint64_t>(x) * kChiStride + c];
      const uint64_t* mx = pmap + cx * A.k;
      const uint64_t base = A.off[x], end = A.off[x + 1];
      for (uint64_t p = base + jl; p < end; p += 32 * UNR) {
        uint32_t y[UNR], cy[UNR], r[UNR][PB];
        bool ok[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          ok[u] = p + 32 * u < end;
          y[u] = ok[u] ? __ldg(A.adj + p + 32 * u) : 0u;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          cy[u] = ok[u] ? A.chi[static_cast<uint64_t>(y[u]) * kChiStride + c] : cx;
          const uint64_t roff = static_cast<uint64_t>(y[u]) * A.rsb + c * A.psb;
          if (PB <= 8 && A.ub_e == 2 && A.psb == 8) {
            // padded u16 row: one 16-byte load
            const uint4 v4 = ok[u] ? __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(A.ub) + roff))
                                   : make_uint4(0, 0, 0, 0);
            const uint32_t wv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int e = 0; e < PB; ++e) r[u][e] = (wv[(e >> 1) & 3] >> (16 * (e & 1))) & 0xFFFFu;
          } else if (A.ub_e == 2) {
#pragma unroll
            for (int e = 0; e < PB; ++e) r[u][e] = ok[u] ? ld_entry(A.ub, roff + e, 2) : 0u;
          } else {
#pragma unroll
            for (int e = 0; e < PB; ++e) r[u][e] = ok[u] ? ld_entry(A.ub, roff + e, 4) : 0u;
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          if (cy[u] == cx) continue;
          const uint64_t w = mx[cy[u]];
#pragma unroll
          for (int e = 0; e < PB; ++e) {
            const uint32_t t = static_cast<uint32_t>(w >> (5 * e)) & 31u;
            if (t == 31u || !r[u][e]) continue;
            atomicAdd(acc + t * AS, r[u][e]);
            ++upd;
          }
        }
      }
    }
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < A.C * A.Pout; o += blockDim.x) {
      const uint32_t cc = o / A.Pout, i = o - cc * A.Pout;
      uint32_t s = 0;
      for (int l = 0; l < 32; ++l) s += accs[i * AS + l * 8 + cc];
      st_entry(A.out, static_cast<uint64_t>(x) * A.rso + cc * A.pso + i, A.out_e, s);
    }
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// Edge-centric 3-cycle blocks over per-edge common-neighbour (CN) lists.
// Included by engine.cu after its helpers (and after leaf.cuh).
//
// A labelled match of a 3-cycle block (positions P0, P1, P2) maps the pivot
// edge (P0, P1) onto an edge {a, b} of the graph and P2 onto a common
// neighbour w of a and b.  Every undirected edge is stored once, oriented from
// its (degree, id)-higher end a to the lower end b (the DB orientation of
// paper §5.1), together with the list of its common neighbours and the CSR
// slots (a->w, b->w) (structure of arrays).  Both orientations (P0,P1) = (a,b)
// and (b,a) are evaluated from the same list, so every labelled match is
// produced exactly once, the pivot's rows are read once per edge, and a block
// keyed by the pivot (|B| = 2) writes each of its two output rows exactly once,
// without atomics.
//
// The CN lists depend only on the graph; they are built once per graph (one
// degree-ordered triangle enumeration, counted then filled) and reused by
// every colouring and every 3-cycle block.

// Triangle enumeration over the degree-ordered out-lists.  PASS 0: count the
// CN entries of each oriented edge; PASS 1: claim positions and write them.
template <int PASS>
__global__ void k_cn_build(uint64_t nout, const uint64_t* __restrict__ out_off, const uint32_t* __restrict__ out_nbr,
                           const uint32_t* __restrict__ out_slot, const uint32_t* __restrict__ out_src,
                           const uint32_t* __restrict__ rev, u64* __restrict__ cnt,
                           const uint64_t* __restrict__ cn_off, uint32_t* __restrict__ cw,
                           uint32_t* __restrict__ csa, uint32_t* __restrict__ csb) {
  const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (j >= nout) return;
  const uint32_t x = out_src[j], y = out_nbr[j];
  uint64_t ia = out_off[x], ae = out_off[x + 1], ib = out_off[y], be = out_off[y + 1];
  while (ia < ae && ib < be) {
    const uint32_t za = out_nbr[ia], zb = out_nbr[ib];
    if (za < zb) {
      ++ia;
    } else if (zb < za) {
      ++ib;
    } else {
      // triangle x > y > z with oriented edges j = x->y, ia = x->z, ib = y->z
      if (PASS == 0) {
        atomicAdd(cnt + j, 1ull);
        atomicAdd(cnt + ia, 1ull);
        atomicAdd(cnt + ib, 1ull);
      } else {
        const uint32_t sxy = out_slot[j], sxz = out_slot[ia], syz = out_slot[ib];
        uint64_t p = cn_off[j] + atomicAdd(cnt + j, 1ull);
        cw[p] = za, csa[p] = sxz, csb[p] = syz;                 // edge x->y, third z
        p = cn_off[ia] + atomicAdd(cnt + ia, 1ull);
        cw[p] = y, csa[p] = sxy, csb[p] = rev[syz];             // edge x->z, third y
        p = cn_off[ib] + atomicAdd(cnt + ib, 1ull);
        cw[p] = x, csa[p] = rev[sxy], csb[p] = rev[sxz];        // edge y->z, third x
      }
      ++ia, ++ib;
    }
  }
}

// ---------------------------------------------------------------------------
// General 3-cycle kernel: any factors, one colouring per launch (a strided
// view into the batched tables).  One warp per oriented edge.
// ---------------------------------------------------------------------------

struct TriEdgeArgs {
  uint64_t nout;
  const uint64_t* cn_off;
  const uint32_t* cn_w;      // third vertex
  const uint32_t* cn_sa;     // slot a->w
  const uint32_t* cn_sb;     // slot b->w
  const uint32_t* out_src;   // a of oriented edge j
  const uint32_t* out_nbr;   // b of oriented edge j
  const uint32_t* out_slot;  // slot a->b
  const uint32_t* rev;
  const uint8_t* chi;        // colouring c's colours, stride kChiStride
  int k;
  // factors (null when absent), pre-offset to colouring c, row strides rs*.
  // Edge factors carry `sw`: stored keyed opposite to the walk in the name.
  const uint64_t* n0; uint32_t Pn0, rsn0; int sn0;   // node at P0
  const uint64_t* n1; uint32_t Pn1, rsn1; int sn1;   // node at P1
  const uint64_t* n2; uint32_t Pn2, rsn2; int sn2;   // node at P2 (per w)
  const uint64_t* e01; uint32_t Pe01, rse01; int se01; int sw01;  // keyed (P0,P1) unless sw
  const uint64_t* e12; uint32_t Pe12, rse12; int se12; int sw12;  // keyed (P1,P2) unless sw
  const uint64_t* e20; uint32_t Pe20, rse20; int se20; int sw20;  // keyed (P2,P0) unless sw
  int out_kind;  // 0 scalar, 1 unary keyed by img P0, 2 edge keyed (img P0, img P1)
  uint64_t* out;
  uint32_t Pout, rso;
  u64* scalar;
  int* err;
  u64* updates;
};

constexpr int kTriFixedCap = 128;  // pivot partial products per orientation
constexpr int kTriWarps = 4;

__device__ __forceinline__ uint32_t row_mask(int t, uint32_t idx, uint32_t fixed) {
  return sig_expand(sig_unrank(c_lut, t, idx), fixed);
}

// Folds one table row into (mask, value) pairs: out = {m | M : (m & M) == fixed}.
__device__ __forceinline__ int fold_row(const uint64_t* row, uint32_t P, int s, uint32_t fixed,
                                        const uint32_t* im, const uint64_t* iv, int ni, uint32_t* om,
                                        uint64_t* ov, int cap, int* err) {
  const int t = s - mb_popc(fixed);
  int no = 0;
  for (uint32_t j = 0; j < P; ++j) {
    const uint64_t v = row[j];
    if (!v) continue;
    const uint32_t M = row_mask(t, j, fixed);
    for (int i = 0; i < ni; ++i) {
      if ((im[i] & M) != fixed) continue;
      if (no == cap) {
        atomicOr(err, 8);
        return no;
      }
      om[no] = im[i] | M;
      ov[no] = mul_ck(iv[i], v, err);
      ++no;
    }
  }
  return no;
}

__global__ void __launch_bounds__(32 * kTriWarps) tri_edge_block_kernel(TriEdgeArgs A) {
  extern __shared__ u64 tsm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u64* base = tsm + static_cast<size_t>(wid) * (3 * kTriFixedCap + 2 * A.Pout + 2);
  uint32_t* lm = reinterpret_cast<uint32_t*>(base);            // [2][cap] masks
  u64* lv = base + kTriFixedCap;                               // [2][cap] values
  u64* orow = base + 3 * kTriFixedCap;                          // [2][Pout]
  int* lnum = reinterpret_cast<int*>(orow + 2 * A.Pout);       // [2]
  uint64_t local = 0, upd = 0;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kTriWarps + wid; j < A.nout;
       j += static_cast<uint64_t>(gridDim.x) * kTriWarps) {
    const uint32_t a = A.out_src[j], b = A.out_nbr[j];
    const uint32_t sab = A.out_slot[j], sba = A.rev[sab];
    const uint32_t ca = A.chi[static_cast<uint64_t>(a) * kChiStride], cb = A.chi[static_cast<uint64_t>(b) * kChiStride];
    for (uint32_t i = lane; i < 2 * A.Pout; i += 32) orow[i] = 0;
    if (lane < 2) {
      const int o = lane;
      int nl = 0;
      if (ca != cb) {
        const uint32_t v0 = o ? b : a, v1 = o ? a : b;
        const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
        uint32_t m1[kTriFixedCap], m2[kTriFixedCap];
        uint64_t x1[kTriFixedCap], x2[kTriFixedCap];
        m1[0] = (1u << c0) | (1u << c1);
        x1[0] = 1;
        nl = 1;
        if (A.n0) {
          nl = fold_row(A.n0 + static_cast<uint64_t>(v0) * A.rsn0, A.Pn0, A.sn0, 1u << c0, m1, x1, nl, m2, x2,
                        kTriFixedCap, A.err);
          for (int i = 0; i < nl; ++i) m1[i] = m2[i], x1[i] = x2[i];
        }
        if (A.n1) {
          nl = fold_row(A.n1 + static_cast<uint64_t>(v1) * A.rsn1, A.Pn1, A.sn1, 1u << c1, m1, x1, nl, m2, x2,
                        kTriFixedCap, A.err);
          for (int i = 0; i < nl; ++i) m1[i] = m2[i], x1[i] = x2[i];
        }
        if (A.e01) {
          const uint64_t s = (o == 0) != (A.sw01 != 0) ? sab : sba;
          nl = fold_row(A.e01 + s * A.rse01, A.Pe01, A.se01, (1u << c0) | (1u << c1), m1, x1, nl, m2, x2,
                        kTriFixedCap, A.err);
          for (int i = 0; i < nl; ++i) m1[i] = m2[i], x1[i] = x2[i];
        }
        for (int i = 0; i < nl; ++i) lm[o * kTriFixedCap + i] = m1[i], lv[o * kTriFixedCap + i] = x1[i];
      }
      lnum[o] = nl;
    }
    __syncwarp();
    const uint64_t c0 = A.cn_off[j], c1 = A.cn_off[j + 1];
    const uint64_t items = 2 * (c1 - c0);
    for (uint64_t it = lane; it < items; it += 32) {
      const int o = static_cast<int>(it & 1);
      const uint64_t ci = c0 + (it >> 1);
      const int nl = lnum[o];
      if (!nl) continue;
      const uint32_t w = __ldg(A.cn_w + ci), cw = A.chi[static_cast<uint64_t>(w) * kChiStride], fw = 1u << cw;
      const uint32_t saw = __ldg(A.cn_sa + ci), sbw = __ldg(A.cn_sb + ci);
      const uint32_t cp0 = o ? cb : ca, cp1 = o ? ca : cb;
      const uint32_t s_p0w = o ? sbw : saw, s_p1w = o ? saw : sbw;
      const uint64_t* rn2 = A.n2 ? A.n2 + static_cast<uint64_t>(w) * A.rsn2 : nullptr;
      const uint64_t* r12 = nullptr;
      const uint64_t* r20 = nullptr;
      if (A.e12) r12 = A.e12 + static_cast<uint64_t>(A.sw12 ? A.rev[s_p1w] : s_p1w) * A.rse12;
      if (A.e20) r20 = A.e20 + static_cast<uint64_t>(A.sw20 ? s_p0w : A.rev[s_p0w]) * A.rse20;
      const uint32_t f12 = (1u << cp1) | fw, f20 = fw | (1u << cp0);
      const int t2 = A.sn2 - 1, t12 = A.se12 - 2, t20 = A.se20 - 2;
      const uint32_t fx = A.out_kind == 1 ? (1u << cp0) : ((1u << cp0) | (1u << cp1));
      for (int i = 0; i < nl; ++i) {
        const uint32_t m0 = lm[o * kTriFixedCap + i];
        if (m0 & fw) continue;
        const uint64_t v0 = lv[o * kTriFixedCap + i];
        const uint32_t mA = m0 | fw;
        const uint32_t nn = rn2 ? A.Pn2 : 1u;
        for (uint32_t q = 0; q < nn; ++q) {
          uint32_t mB = mA;
          uint64_t vB = v0;
          if (rn2) {
            const uint64_t x = rn2[q];
            if (!x) continue;
            const uint32_t M = row_mask(t2, q, fw);
            if ((M & mA) != fw) continue;
            mB |= M;
            vB = mul_ck(vB, x, A.err);
          }
          const uint32_t ne1 = r12 ? A.Pe12 : 1u;
          for (uint32_t e1 = 0; e1 < ne1; ++e1) {
            uint32_t mC = mB;
            uint64_t vC = vB;
            if (r12) {
              const uint64_t x = r12[e1];
              if (!x) continue;
              const uint32_t M = row_mask(t12, e1, f12);
              if ((M & mB) != f12) continue;
              mC |= M;
              vC = mul_ck(vC, x, A.err);
            }
            const uint32_t ne2 = r20 ? A.Pe20 : 1u;
            for (uint32_t e2 = 0; e2 < ne2; ++e2) {
              uint32_t mD = mC;
              uint64_t vD = vC;
              if (r20) {
                const uint64_t x = r20[e2];
                if (!x) continue;
                const uint32_t M = row_mask(t20, e2, f20);
                if ((M & mC) != f20) continue;
                mD |= M;
                vD = mul_ck(vD, x, A.err);
              }
              ++upd;
              if (A.out_kind == 0)
                local = add_ck(local, vD, A.err);
              else
                atomic_add_ck(orow + o * A.Pout + sig_index(c_lut, mD, fx), vD, A.err);
            }
          }
        }
      }
    }
    __syncwarp();
    if (A.out_kind == 2) {
      for (uint32_t i = lane; i < 2 * A.Pout; i += 32) {
        const int o = i >= A.Pout;
        const uint64_t s = o ? sba : sab;
        A.out[s * A.rso + (i - o * A.Pout)] = orow[i];
      }
    } else if (A.out_kind == 1) {
      for (uint32_t i = lane; i < 2 * A.Pout; i += 32) {
        const int o = i >= A.Pout;
        const uint64_t v = orow[i];
        if (v)
          atomic_add_ck(reinterpret_cast<u64*>(A.out) + static_cast<uint64_t>(o ? b : a) * A.rso + (i - o * A.Pout),
                        v, A.err);
      }
    }
    __syncwarp();
  }
  if (A.out_kind == 0) {
    for (int o = 16; o > 0; o >>= 1) local = add_ck(local, __shfl_down_sync(0xffffffffu, local, o), A.err);
    if (lane == 0 && local) atomic_add_ck(A.scalar, local, A.err);
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if (lane == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// ---------------------------------------------------------------------------
// Histogram path, batched over colourings: one warp owns 32 consecutive
// oriented edges.
//
// Used when no factor depends on the third vertex and at most one factor
// sits on the pivot: a match's contribution then depends on w only through
// chi(w).
// (1) The warp scans the 32 edges' CN lists as one flat, coalesced range
//     (lane i reads entries i, i+32, ...), finds each entry's edge by a
//     5-step shuffle search over the 33 offsets, loads w's colours for all C
//     colourings at once (8 bytes) and bumps hist[edge][c][chi_c(w)].
// (2) Lane l evaluates edge j0+l for every colouring.  An output entry S
//     (a colour set containing the pivot colours c0, c1) receives
//         sum over c in S \ {c0, c1} of hist[c] * F[S \ {c}]
//     where F is the single pivot factor (node row at P0 or P1, edge row of
//     the pivot, or the bare edge).  Which (c, F-index) pairs feed S depends
//     only on (c0, c1, S): the CTA precomputes them into shared `terms`.
// (3) Fusion: when this block's edge table is consumed only as the pivot
//     factor of a parent 3-cycle block that is itself on the histogram path
//     (two triangles sharing an edge — the config-1 query), both blocks use
//     the same edge's histogram.  The child's two rows stay in shared memory
//     and the parent's terms are applied to them right away: the child's
//     edge table never reaches HBM.
// ---------------------------------------------------------------------------

struct TriHistArgs {
  uint64_t nout;
  uint64_t nitems;  // edges visited: nout, or in lane mode the non-empty prefix of eorder
  const uint64_t* cn_off;
  const uint32_t* cn_w;
  const uint32_t* out_src;
  const uint32_t* out_nbr;
  const uint32_t* out_slot;
  const uint32_t* rev;
  const uint8_t* chi;   // [n][kChiStride]
  uint32_t nv;           // vertex count = the dummy row of chi (colour 7 in every slot)
  int debug;             // MB_TRI_DEBUG timing split: 1 no join, 2 no list scan, 3 neither
  int t_safe;            // host bound: every fused-child entry < 2^44 (unchecked stage 2)
  int k, C;
  int lane_mode;
  int f_safe;               // host bound: every factor entry < 2^44 (lane mode: unchecked terms)
  int F_n;                  // pivot factor stored narrow (u32)            // 1: lane per edge, register counters (k <= 8, lists < 65536)
  const uint32_t* eorder;   // oriented edges in CN-length order (lane_mode)
  const uint4* emeta;       // (a, b, slot a->b, slot b->a) per eorder position
  const ulonglong2* erange; // CN list [lo, hi) per eorder position
  // warp-interleaved copy of the lists (k_il_fill): chunk ch of lane l of batch
  // bt is il[(ilbase[bt] + ch) * 32 + l]; ilnch[bt] chunks per lane
  const uint4* il;
  const uint64_t* ilbase;
  const uint32_t* ilnch;
  uint32_t shard_rank, shard_world;  // tri_canon_kernel: warp batches dealt over ranks (1 = all)
  // stage 1: this block
  int s_out;
  uint32_t P2;          // C(k-2, s_out-2): entries of S containing both pivot colours
  int nterm;            // s_out - 2
  int fkind;            // pivot factor: 0 none, 1 node at P0, 2 node at P1, 3 edge (P0,P1)
  const uint64_t* F;    // table base (colouring 0)
  uint32_t PF, rsF;
  uint32_t psF;         // per-colouring row stride of F (PF, or PF rounded up to 4 for 16-byte rows)
  int sw01;             // edge factor stored keyed (P1, P0)
  int out_kind;         // 0 scalar, 1 unary keyed by img P0, 2 edge keyed (img P0, img P1), 3 fused
  uint64_t* out;
  uint32_t Pout, rso;
  // stage 2: fused parent (out_kind == 3)
  uint32_t P2p;
  int ntermp, sw01p, pout_kind;  // parent output: 0 scalar, 1 unary, 2 edge
  uint64_t* pout;
  uint32_t Poutp, rsop;
  u64* scalars;         // [C]
  int* err;
  u64* updates;
};

#ifndef MB_HIST_WARPS
#define MB_HIST_WARPS 8
#endif
constexpr int kHistWarps = MB_HIST_WARPS;

// per-edge histogram row in u32 words: u16 counters in lane mode (lists are
// shorter than 65536 there), u32 in flat mode (shared-memory atomics); odd
// so the 32 rows of a warp fall in distinct banks
__host__ __device__ inline uint32_t hist_lane_words(int C, int k, int lane_mode) {
  const uint32_t n = static_cast<uint32_t>(C) * k;
  return lane_mode ? ((n + 1) / 2) | 1u : n + 1;
}

struct HistSmem {  // shared-memory carve-up (host computes the same sizes)
  uint32_t t1, i1, t2, i2, hist_per_warp, tbuf_per_warp, fst_per_warp;
};

__host__ __device__ inline HistSmem hist_smem_layout(int k, int C, uint32_t P2, int nterm, int out_kind,
                                                     uint32_t P2p, int ntermp, int pout_kind, uint32_t PF,
                                                     int lane_mode) {
  HistSmem L;
  const uint32_t kk = static_cast<uint32_t>(k) * k;
  L.t1 = kk * P2 * nterm;                                       // u32
  L.i1 = out_kind == 1 ? (kk * P2 + 1) / 2 : 0;                 // u16 pairs as u32
  L.t2 = out_kind == 3 ? kk * P2p * ntermp : 0;                 // u32
  L.i2 = (out_kind == 3 && pout_kind == 1) ? (kk * P2p + 1) / 2 : 0;
  L.hist_per_warp = 32u * hist_lane_words(C, k, lane_mode);    // u32, odd per-edge stride
  L.tbuf_per_warp = out_kind == 3 ? 32u * (2 * P2 + 1) * 2 : 0;  // u64 as 2 u32, odd per-lane stride
  L.fst_per_warp = PF ? 32u * (PF | 1u) * 2 : 0;                  // staged factor row (u64), odd stride
  return L;
}

__device__ __forceinline__ void build_terms(uint32_t* terms, uint16_t* idx1, int k, uint32_t P2, int s_out,
                                            int nterm, int fkind, bool want_idx1) {
  for (uint32_t e = threadIdx.x; e < static_cast<uint32_t>(k) * k * P2; e += blockDim.x) {
    const uint32_t i = e % P2, c1 = (e / P2) % k, c0 = e / (P2 * k);
    if (c0 == c1) continue;
    const uint32_t f2 = (1u << c0) | (1u << c1);
    const uint32_t S = sig_expand(sig_unrank(c_lut, s_out - 2, i), f2);
    if (want_idx1) idx1[e] = static_cast<uint16_t>(sig_index(c_lut, S, 1u << c0));
    uint32_t free = S & ~f2;
    for (int t = 0; t < nterm; ++t) {
      const int c = mb_ctz(free);
      free &= free - 1u;
      const uint32_t T = S & ~(1u << c);
      uint32_t j = 0;
      bool ok = true;
      switch (fkind) {
        case 0: ok = T == f2; break;
        case 1: j = sig_index(c_lut, T & ~(1u << c1), 1u << c0); break;
        case 2: j = sig_index(c_lut, T & ~(1u << c0), 1u << c1); break;
        default: j = sig_index(c_lut, T, f2); break;
      }
      terms[static_cast<size_t>(e) * nterm + t] = ok ? (static_cast<uint32_t>(c) << 16) | j : ~0u;
    }
  }
}

#ifndef MB_TRI_MINB
#define MB_TRI_MINB 2  // resident CTAs per SM the register budget is sized for (126 regs, no spill;
                       // measured: 3 -> 80 regs + spills, 13.4 ms vs 11.3 ms per 3 batches)
#endif
// LANE: lane-per-edge register histograms (k <= 8, lists < 65536).
// NARROW: the pivot factor is a narrow (u32) table on the unchecked path, so it
// is staged as u32 and each term is one 32x32->64 multiply-add.
template <bool LANE, bool NARROW>
__global__ void __launch_bounds__(32 * kHistWarps, MB_TRI_MINB) tri_hist_kernel(TriHistArgs A) {
  extern __shared__ uint32_t hsm[];
  const int k = A.k, C = A.C;
  const uint32_t PF = A.fkind ? A.PF : 0u;
  const HistSmem L = hist_smem_layout(k, C, A.P2, A.nterm, A.out_kind, A.P2p, A.ntermp, A.pout_kind, PF,
                                      LANE);
  uint32_t* terms = hsm;
  uint16_t* idx1 = reinterpret_cast<uint16_t*>(hsm + L.t1);
  uint32_t* termsp = hsm + L.t1 + L.i1;
  uint16_t* idx1p = reinterpret_cast<uint16_t*>(termsp + L.t2);
  uint32_t* wbase = hsm + ((L.t1 + L.i1 + L.t2 + L.i2 + 1) & ~1u);  // 8-byte aligned for tbuf
  build_terms(terms, idx1, k, A.P2, A.s_out, A.nterm, A.fkind, A.out_kind == 1);
  if (A.out_kind == 3) build_terms(termsp, idx1p, k, A.P2p, A.s_out + 1, A.ntermp, 3, A.pout_kind == 1);
  __syncthreads();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = wbase + static_cast<size_t>(wid) * (L.hist_per_warp + L.tbuf_per_warp + L.fst_per_warp);
  u64* tbuf = reinterpret_cast<u64*>(hist + L.hist_per_warp) + static_cast<size_t>(lane) * (2 * A.P2 + 1);
  u64* fst = reinterpret_cast<u64*>(hist + L.hist_per_warp + L.tbuf_per_warp) + static_cast<size_t>(lane) * (PF | 1u);
  uint32_t* fst32 = reinterpret_cast<uint32_t*>(fst);
  uint16_t* hist16 = reinterpret_cast<uint16_t*>(hist);
  uint32_t ovf = 0;  // overflow seen by this thread (one atomic at exit)
  uint64_t local[kChiStride];
#pragma unroll
  for (int c = 0; c < kChiStride; ++c) local[c] = 0;
  uint64_t upd = 0;
  const uint32_t LSW = hist_lane_words(C, k, LANE);
  const uint32_t LS = LANE ? 2 * LSW : LSW;  // per-edge row stride in counters
  const uint64_t nbatch = (A.nitems + 31) / 32;
  for (uint64_t bt = static_cast<uint64_t>(blockIdx.x) * kHistWarps + wid; bt < nbatch;
       bt += static_cast<uint64_t>(gridDim.x) * kHistWarps) {
    const uint64_t j0 = bt * 32;
    const bool live = j0 + lane < A.nitems;
    uint64_t j = j0 + lane;
    if (LANE) {
      // lane owns one oriented edge (edges visited in CN-length order, so the
      // 32 lists of a warp have similar lengths) and counts its common
      // neighbours' colours for all C colourings in registers: 4-bit fields
      // (k <= 8 colours in one word) flushed every 12 entries into 16-bit
      // fields (two colours per word).  No shared-memory atomics; the list is
      // read with 16-byte loads.
      if (live) j = A.eorder[j];
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
      if (live) {
        const uint64_t lo_ = A.cn_off[j], hi_ = A.cn_off[j + 1];
        int pend = 0;
        for (uint64_t p = lo_ & ~3ull; p < hi_; p += 4) {
          const uint4 q = __ldg(reinterpret_cast<const uint4*>(A.cn_w + p));
          const uint32_t ws[4] = {q.x, q.y, q.z, q.w};
          uint64_t cw[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool in = p + u >= lo_ && p + u < hi_;
            cw[u] = in ? load_colors(A.chi, ws[u]) : ~0ull;
          }
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
      }
      uint16_t* hrow = hist16 + lane * LS;
#pragma unroll
      for (int c = 0; c < kChiStride; ++c) {
        if (c < C) {
#pragma unroll
          for (int d = 0; d < 8; ++d)  // static indices keep H in registers
            if (d < k) hrow[c * k + d] = static_cast<uint16_t>(H[c][d >> 1] >> (16 * (d & 1)));
        }
      }
      __syncwarp();
    } else {
      for (uint32_t i = lane; i < L.hist_per_warp; i += 32) hist[i] = 0;
      const uint64_t myoff = A.cn_off[live ? j : A.nout];
      const uint64_t endoff = A.cn_off[min(j0 + 32, A.nout)];
      const uint64_t startoff = __shfl_sync(0xffffffffu, myoff, 0);
      __syncwarp();
      for (uint64_t e0 = startoff; e0 < endoff; e0 += 32) {
        const uint64_t e = e0 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const uint64_t o = __shfl_sync(0xffffffffu, myoff, lo + step);
          if (o <= e) lo += step;
        }
        if (e < endoff) {
          const uint32_t w = __ldg(A.cn_w + e);
          const uint64_t cw = load_colors(A.chi, w);
          uint32_t* h = hist + lo * LS;
          for (int c = 0; c < C; ++c) atomicAdd(h + c * k + color_of(cw, c), 1u);
        }
      }
      __syncwarp();
    }
    if (live) {
      uint32_t updl = 0;  // nonzero output-entry updates of this edge, folded into upd below
      const uint32_t a = A.out_src[j], b = A.out_nbr[j];
      const uint32_t sab = A.out_slot[j], sba = A.rev[sab];
      const uint64_t cas = load_colors(A.chi, a), cbs = load_colors(A.chi, b);
      for (int c = 0; c < C; ++c) {
        const uint32_t hb = lane * LS + c * k;
        auto hval = [&](uint32_t d) -> uint32_t { return LANE ? hist16[hb + d] : hist[hb + d]; };
        const uint32_t ca = color_of(cas, c), cb = color_of(cbs, c);
        uint64_t acc = 0, tmax = 0;
        for (int o = 0; o < 2; ++o) {
          const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
          const uint64_t orow = static_cast<uint64_t>(o ? sba : sab) * A.rso + c * A.Pout;
          if (c0 == c1) {
            if (A.out_kind == 2)
              for (uint32_t i = 0; i < A.Pout; ++i) A.out[orow + i] = 0;
            if (A.out_kind == 3)
              for (uint32_t i = 0; i < A.P2; ++i) tbuf[o * A.P2 + i] = 0;
            continue;
          }
          if (PF) {
            // stage this orientation's factor row: independent loads in
            // flight together instead of one dependent gather per term
            uint64_t fo;
            if (A.fkind == 1) fo = static_cast<uint64_t>(o ? b : a) * A.rsF + c * A.psF;
            else if (A.fkind == 2) fo = static_cast<uint64_t>(o ? a : b) * A.rsF + c * A.psF;
            else fo = static_cast<uint64_t>((o == 0) != (A.sw01 != 0) ? sab : sba) * A.rsF + c * A.psF;
            const uint64_t* F = A.F + fo;
            const uint32_t* F32 = reinterpret_cast<const uint32_t*>(A.F) + fo;
            if (NARROW) {
              for (uint32_t i0 = 0; i0 < PF; i0 += 8) {
                uint32_t r[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] = i0 + u < PF ? __ldg(F32 + i0 + u) : 0u;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                  if (i0 + u < PF) fst32[i0 + u] = r[u];
              }
            } else for (uint32_t i0 = 0; i0 < PF; i0 += 8) {
              uint64_t r[8];
              if (A.F_n) {
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] = i0 + u < PF ? __ldg(F32 + i0 + u) : 0u;
              } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] = i0 + u < PF ? __ldg(F + i0 + u) : 0ull;
              }
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (i0 + u < PF) fst[i0 + u] = r[u];
            }
          }
          const u64* Fs = PF ? fst : nullptr;
          // lane-mode counters are < 2^16 and there are <= 15 terms: with every
          // factor < 2^44 (host bound) no product or partial sum can reach 2^64
          const bool safe = LANE && A.f_safe;
          const uint32_t tb = (c0 * k + c1) * A.P2;
          for (uint32_t i = 0; i < A.P2; ++i) {
            const uint32_t* tt = terms + static_cast<size_t>(tb + i) * A.nterm;
            uint64_t v = 0;
            // branch-free multiply-add: lanes of a warp hold different
            // colour pairs, so per-term zero tests would only diverge
            if (NARROW) {
#pragma unroll 4
              for (int t = 0; t < A.nterm; ++t) {
                const uint32_t x = tt[t];
                const bool ok = x != ~0u;
                const uint32_t hc = ok ? hval(x >> 16) : 0u;
                const uint32_t f = ok ? fst32[x & 0xFFFFu] : 0u;
                v += static_cast<uint64_t>(f) * hc;
              }
            } else if (safe) {
#pragma unroll 4
              for (int t = 0; t < A.nterm; ++t) {
                const uint32_t x = tt[t];
                const bool ok = x != ~0u;
                const uint32_t hc = ok ? hval(x >> 16) : 0u;
                const uint64_t f = Fs ? (ok ? Fs[x & 0xFFFFu] : 0ull) : 1ull;
                v += f * hc;
              }
            } else {
#pragma unroll 4
              for (int t = 0; t < A.nterm; ++t) {
                const uint32_t x = tt[t];
                const bool ok = x != ~0u;
                const uint32_t hc = ok ? hval(x >> 16) : 0u;
                const uint64_t f = Fs ? (ok ? Fs[x & 0xFFFFu] : 0ull) : 1ull;
                ovf |= __umul64hi(f, hc) != 0;
                const uint64_t fh = f * hc;
                v += fh;
                ovf |= v < fh;
              }
            }
            updl += v != 0;
            if (A.out_kind == 2) {
              A.out[orow + i] = v;
            } else if (A.out_kind == 3) {
              tbuf[o * A.P2 + i] = v;
              tmax |= v;
            } else if (v) {
              if (A.out_kind == 0)
                {
                  acc += v;
                  ovf |= acc < v;
                }
              else
                atomic_add_ck(reinterpret_cast<u64*>(A.out) + static_cast<uint64_t>(o ? b : a) * A.rso + c * A.Pout +
                                  idx1[tb + i], v, A.err);
            }
          }
        }
        if (A.out_kind == 3 && ca != cb) {
          // parent stage on the same edge and histogram; its pivot factor is
          // this block's row for the orientation the parent reads
          for (int o = 0; o < 2; ++o) {
            const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
            const int osel = ((o == 0) != (A.sw01p != 0)) ? 0 : 1;
            const u64* T = tbuf + osel * A.P2;
            const uint32_t tb = (c0 * k + c1) * A.P2p;
            const bool safe = LANE && (tmax >> 44) == 0;
            for (uint32_t i = 0; i < A.P2p; ++i) {
              const uint32_t* tt = termsp + static_cast<size_t>(tb + i) * A.ntermp;
              uint64_t v = 0;
              if (safe) {
#pragma unroll 4
                for (int t = 0; t < A.ntermp; ++t) {
                  const uint32_t x = tt[t];
                  const bool ok = x != ~0u;
                  const uint32_t hc = ok ? hval(x >> 16) : 0u;
                  const uint64_t f = ok ? T[x & 0xFFFFu] : 0ull;
                  v += f * hc;
                }
              } else {
#pragma unroll 4
                for (int t = 0; t < A.ntermp; ++t) {
                  const uint32_t x = tt[t];
                  const bool ok = x != ~0u;
                  const uint32_t hc = ok ? hval(x >> 16) : 0u;
                  const uint64_t f = ok ? T[x & 0xFFFFu] : 0ull;
                  ovf |= __umul64hi(f, hc) != 0;
                  const uint64_t fh = f * hc;
                  v += fh;
                  ovf |= v < fh;
                }
              }
              updl += v != 0;
              if (A.pout_kind == 2) {
                A.pout[static_cast<uint64_t>(o ? sba : sab) * A.rsop + c * A.Poutp + i] = v;
              } else if (v) {
                if (A.pout_kind == 0)
                  {
                  acc += v;
                  ovf |= acc < v;
                }
                else
                  atomic_add_ck(reinterpret_cast<u64*>(A.pout) + static_cast<uint64_t>(o ? b : a) * A.rsop +
                                    c * A.Poutp + idx1p[tb + i], v, A.err);
              }
            }
          }
        } else if (A.out_kind == 3 && A.pout_kind == 2) {
          for (int o = 0; o < 2; ++o)
            for (uint32_t i = 0; i < A.P2p; ++i)
              A.pout[static_cast<uint64_t>(o ? sba : sab) * A.rsop + c * A.Poutp + i] = 0;
        }
#pragma unroll
        for (int cc = 0; cc < kChiStride; ++cc)
          if (cc == c) {
            local[cc] += acc;
            ovf |= local[cc] < acc;
          }
      }
      upd += updl;
    }
    __syncwarp();
  }
  const bool scalar_out = A.out_kind == 0 || (A.out_kind == 3 && A.pout_kind == 0);
  if (scalar_out) {
#pragma unroll
    for (int c = 0; c < kChiStride; ++c) {
      uint64_t v = local[c];
      for (int o = 16; o > 0; o >>= 1) v = add_ck(v, __shfl_down_sync(0xffffffffu, v, o), A.err);
      if (lane == 0 && v) atomic_add_ck(A.scalars + c, v, A.err);
    }
  }
  if (ovf) atomicOr(A.err, 1);
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if (lane == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

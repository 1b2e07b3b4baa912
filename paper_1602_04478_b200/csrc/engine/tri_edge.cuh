// Edge-centric 3-cycle blocks over per-edge common-neighbour (CN) lists.
// Included by engine.cu after its helpers.
//
// A labelled match of a 3-cycle block (positions P0, P1, P2) maps the pivot
// edge (P0, P1) onto an edge {a, b} of the graph and P2 onto a common
// neighbour w of a and b.  Every undirected edge is stored once, oriented from
// its (degree, id)-higher end a to the lower end b (the DB orientation of
// paper §5.1), together with the list of its common neighbours and the CSR
// slots (a->w, b->w) (structure of arrays).  One warp owns one oriented edge
// and evaluates both orientations (P0,P1) = (a,b) and (b,a), so every labelled
// match is produced exactly once, the pivot's rows are read once per edge, and
// a block keyed by the pivot (|B| = 2) writes each of its two output rows
// exactly once, without atomics.
//
// Colour-histogram fast path: when no factor depends on the third vertex
// (no annotation on P2 or on the edges P1-P2, P2-P0), a match's contribution
// depends on w only through chi(w).  The warp then reduces the CN list to a
// per-colour histogram with k ballots per 32 entries (reading 4 bytes per
// entry) and joins the histogram with the pivot's partial products — the
// disjoint-union join of paper Fig. 8 applied once per colour instead of once
// per common neighbour.
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
  const uint8_t* chi;
  int k;
  // factors (null when absent).  Edge factors carry `sw`: stored keyed in the
  // opposite direction of the walk named in the field.
  const uint64_t* n0; uint32_t Pn0; int sn0;   // node at P0
  const uint64_t* n1; uint32_t Pn1; int sn1;   // node at P1
  const uint64_t* n2; uint32_t Pn2; int sn2;   // node at P2 (per w)
  const uint64_t* e01; uint32_t Pe01; int se01; int sw01;  // keyed (P0,P1) unless sw
  const uint64_t* e12; uint32_t Pe12; int se12; int sw12;  // keyed (P1,P2) unless sw
  const uint64_t* e20; uint32_t Pe20; int se20; int sw20;  // keyed (P2,P0) unless sw
  int out_kind;  // 0 scalar, 1 unary keyed by img P0, 2 edge keyed (img P0, img P1)
  uint64_t* out;
  uint32_t Pout;
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
  // per warp: two orientation lists (mask, value) + two output rows + counts
  u64* base = tsm + static_cast<size_t>(wid) * (3 * kTriFixedCap + 2 * A.Pout + 2 + kMaxColors);
  uint32_t* lm = reinterpret_cast<uint32_t*>(base);            // [2][cap] masks
  u64* lv = base + kTriFixedCap;                               // [2][cap] values
  u64* orow = base + 3 * kTriFixedCap;                          // [2][Pout]
  int* lnum = reinterpret_cast<int*>(orow + 2 * A.Pout);       // [2]
  uint32_t* hist = reinterpret_cast<uint32_t*>(orow + 2 * A.Pout + 1);  // [k]
  const int nfixed = (A.n0 != nullptr) + (A.n1 != nullptr) + (A.e01 != nullptr);
  const bool per_w = A.n2 || A.e12 || A.e20;
  uint64_t local = 0, upd = 0;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kTriWarps + wid; j < A.nout;
       j += static_cast<uint64_t>(gridDim.x) * kTriWarps) {
    const uint32_t a = A.out_src[j], b = A.out_nbr[j];
    const uint32_t sab = A.out_slot[j], sba = A.rev[sab];
    const uint32_t ca = A.chi[a], cb = A.chi[b];
    for (uint32_t i = lane; i < 2 * A.Pout; i += 32) orow[i] = 0;
    // ---- pivot partial products for orientation o: (P0,P1) = (a,b) or (b,a)
    if (ca == cb) {
      if (lane < 2) lnum[lane] = 0;
    } else if (nfixed <= 1) {
      // cooperative: lane l handles entry l of the single pivot row per orientation
      const uint64_t* row[2] = {nullptr, nullptr};
      uint32_t P = 1, fx[2] = {(1u << ca) | (1u << cb), (1u << ca) | (1u << cb)};
      int s = 2;
      if (A.n0) {
        row[0] = A.n0 + static_cast<uint64_t>(a) * A.Pn0, row[1] = A.n0 + static_cast<uint64_t>(b) * A.Pn0;
        fx[0] = 1u << ca, fx[1] = 1u << cb, P = A.Pn0, s = A.sn0;
      } else if (A.n1) {
        row[0] = A.n1 + static_cast<uint64_t>(b) * A.Pn1, row[1] = A.n1 + static_cast<uint64_t>(a) * A.Pn1;
        fx[0] = 1u << cb, fx[1] = 1u << ca, P = A.Pn1, s = A.sn1;
      } else if (A.e01) {
        row[0] = A.e01 + static_cast<uint64_t>(A.sw01 ? sba : sab) * A.Pe01;
        row[1] = A.e01 + static_cast<uint64_t>(A.sw01 ? sab : sba) * A.Pe01;
        P = A.Pe01, s = A.se01;
      }
      const uint32_t bm = (1u << ca) | (1u << cb);
      for (int o = 0; o < 2; ++o) {
        int cnt = 0;
        for (uint32_t e0 = 0; e0 < P; e0 += 32) {
          const uint32_t e = e0 + lane;
          bool ok = false;
          uint32_t M = bm;
          uint64_t v = 1;
          if (e < P) {
            if (row[o]) {
              v = __ldg(row[o] + e);
              if (v) {
                M = row_mask(s - mb_popc(fx[o]), e, fx[o]);
                ok = (M & bm) == fx[o];
                M |= bm;
              }
            } else {
              ok = true;
            }
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, ok);
          if (ok) {
            const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
            lm[o * kTriFixedCap + pos] = M;
            lv[o * kTriFixedCap + pos] = v;
          }
          cnt += __popc(bal);
        }
        if (lane == 0) lnum[o] = cnt;
      }
    } else if (lane < 2) {
      const int o = lane;
      const uint32_t v0 = o ? b : a, v1 = o ? a : b;
      const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
      uint32_t m1[kTriFixedCap], m2[kTriFixedCap];
      uint64_t x1[kTriFixedCap], x2[kTriFixedCap];
      m1[0] = (1u << c0) | (1u << c1);
      x1[0] = 1;
      int nl = 1;
      if (A.n0) {
        nl = fold_row(A.n0 + static_cast<uint64_t>(v0) * A.Pn0, A.Pn0, A.sn0, 1u << c0, m1, x1, nl, m2, x2,
                      kTriFixedCap, A.err);
        for (int i = 0; i < nl; ++i) m1[i] = m2[i], x1[i] = x2[i];
      }
      if (A.n1) {
        nl = fold_row(A.n1 + static_cast<uint64_t>(v1) * A.Pn1, A.Pn1, A.sn1, 1u << c1, m1, x1, nl, m2, x2,
                      kTriFixedCap, A.err);
        for (int i = 0; i < nl; ++i) m1[i] = m2[i], x1[i] = x2[i];
      }
      if (A.e01) {
        const uint64_t s = (o == 0) != (A.sw01 != 0) ? sab : sba;
        nl = fold_row(A.e01 + s * A.Pe01, A.Pe01, A.se01, (1u << c0) | (1u << c1), m1, x1, nl, m2, x2,
                      kTriFixedCap, A.err);
        for (int i = 0; i < nl; ++i) m1[i] = m2[i], x1[i] = x2[i];
      }
      for (int i = 0; i < nl; ++i) lm[o * kTriFixedCap + i] = m1[i], lv[o * kTriFixedCap + i] = x1[i];
      lnum[o] = nl;
    }
    __syncwarp();
    const uint64_t c0 = A.cn_off[j], c1 = A.cn_off[j + 1];
    if (!per_w) {
      // ---- colour histogram of the common neighbours
      uint32_t my = 0;  // lane c < k holds the count of colour c
      if (lnum[0] | lnum[1]) {
        for (uint64_t i0 = c0; i0 < c1; i0 += 32) {
          const uint64_t i = i0 + lane;
          const int cw = i < c1 ? A.chi[__ldg(A.cn_w + i)] : -1;
          for (int c = 0; c < A.k; ++c) {
            const uint32_t n = __popc(__ballot_sync(0xffffffffu, cw == c));
            if (lane == c) my += n;
          }
        }
      }
      if (lane < kMaxColors) hist[lane] = my;
      __syncwarp();
      // ---- join: for each orientation, partial product e and colour c not in it
      const int n0 = lnum[0], n1 = lnum[1];
      const int items = (n0 + n1) * A.k;
      for (int it = lane; it < items; it += 32) {
        const int o = it >= n0 * A.k;
        const int r = o ? it - n0 * A.k : it;
        const int e = r / A.k, c = r - e * A.k;
        const uint32_t h = hist[c];
        if (!h) continue;
        const uint32_t m = lm[o * kTriFixedCap + e];
        if (m & (1u << c)) continue;
        const uint64_t v = mul_ck(lv[o * kTriFixedCap + e], h, A.err);
        ++upd;
        if (A.out_kind == 0) {
          local = add_ck(local, v, A.err);
        } else {
          const uint32_t cp0 = o ? cb : ca, cp1 = o ? ca : cb;
          const uint32_t fx = A.out_kind == 1 ? (1u << cp0) : ((1u << cp0) | (1u << cp1));
          atomic_add_ck(orow + o * A.Pout + sig_index(c_lut, m | (1u << c), fx), v, A.err);
        }
      }
    } else {
      // ---- general: factors on the third vertex, one (orientation, w) per item
      const uint64_t items = 2 * (c1 - c0);
      for (uint64_t it = lane; it < items; it += 32) {
        const int o = static_cast<int>(it & 1);
        const uint64_t ci = c0 + (it >> 1);
        const int nl = lnum[o];
        if (!nl) continue;
        const uint32_t w = __ldg(A.cn_w + ci), cw = A.chi[w], fw = 1u << cw;
        const uint32_t saw = __ldg(A.cn_sa + ci), sbw = __ldg(A.cn_sb + ci);
        const uint32_t cp0 = o ? cb : ca, cp1 = o ? ca : cb;
        const uint32_t s_p0w = o ? sbw : saw, s_p1w = o ? saw : sbw;
        const uint64_t* rn2 = A.n2 ? A.n2 + static_cast<uint64_t>(w) * A.Pn2 : nullptr;
        const uint64_t* r12 = nullptr;
        const uint64_t* r20 = nullptr;
        if (A.e12) r12 = A.e12 + static_cast<uint64_t>(A.sw12 ? A.rev[s_p1w] : s_p1w) * A.Pe12;
        if (A.e20) r20 = A.e20 + static_cast<uint64_t>(A.sw20 ? s_p0w : A.rev[s_p0w]) * A.Pe20;
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
    }
    __syncwarp();
    if (A.out_kind == 2) {
      // both rows of the pivot edge, written once
      for (uint32_t i = lane; i < 2 * A.Pout; i += 32) {
        const int o = i >= A.Pout;
        const uint64_t s = o ? sba : sab;
        A.out[s * A.Pout + (i - o * A.Pout)] = orow[i];
      }
    } else if (A.out_kind == 1) {
      for (uint32_t i = lane; i < 2 * A.Pout; i += 32) {
        const int o = i >= A.Pout;
        const uint64_t v = orow[i];
        if (v)
          atomic_add_ck(reinterpret_cast<u64*>(A.out) + static_cast<uint64_t>(o ? b : a) * A.Pout + (i - o * A.Pout),
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
// Histogram path, batched: one warp owns 32 consecutive oriented edges.
//
// (1) The warp scans the 32 edges' CN lists as one flat, coalesced range
//     (lane i reads entries i, i+32, ...), finds each entry's edge by a
//     5-step search over the 33 offsets and bumps hist[edge][chi(w)] in
//     shared memory.
// (2) Lane l then evaluates edge j0+l.  An output entry S (a colour set that
//     contains the pivot colours c0, c1) receives
//         sum over c in S \ {c0, c1} of hist[c] * F[S \ {c}]
//     where F is the single pivot factor (node row at P0 or P1, edge row of
//     the pivot, or the bare edge).  Which (c, F-index) pairs feed entry S
//     depends only on (c0, c1, S), so the CTA precomputes them once into a
//     shared table `terms[c0][c1][i][t]` and the lane does loads and
//     multiply-adds only.
// ---------------------------------------------------------------------------

struct TriHistArgs {
  uint64_t nout;
  const uint64_t* cn_off;
  const uint32_t* cn_w;
  const uint32_t* out_src;
  const uint32_t* out_nbr;
  const uint32_t* out_slot;
  const uint32_t* rev;
  const uint8_t* chi;
  int k;
  int s_out;      // popcount of the block's signatures
  uint32_t P2;    // C(k-2, s_out-2): entries of S containing both pivot colours
  int nterm;      // s_out - 2
  int fkind;      // pivot factor: 0 none, 1 node at P0, 2 node at P1, 3 edge (P0,P1)
  const uint64_t* F;
  uint32_t PF;
  int sw01;       // edge factor stored keyed (P1, P0)
  int out_kind;   // 0 scalar, 1 unary keyed by img P0, 2 edge keyed (img P0, img P1)
  uint64_t* out;
  uint32_t Pout;
  u64* scalar;
  int* err;
  u64* updates;
};

constexpr int kHistWarps = 8;

__global__ void __launch_bounds__(32 * kHistWarps) tri_hist_kernel(TriHistArgs A) {
  extern __shared__ uint32_t hsm[];
  const int k = A.k;
  const uint32_t tsize = static_cast<uint32_t>(k) * k * A.P2 * A.nterm;
  uint32_t* terms = hsm;                                   // [k][k][P2][nterm]  (c << 16) | j, or ~0
  uint16_t* idx1 = reinterpret_cast<uint16_t*>(hsm + tsize);  // [k][k][P2] unary output index
  const uint32_t isize = A.out_kind == 1 ? static_cast<uint32_t>(k) * k * A.P2 : 0;
  uint32_t* hist_all = hsm + tsize + (isize + 1) / 2;      // [warps][32][k]
  // ---- per-CTA term table
  for (uint32_t e = threadIdx.x; e < static_cast<uint32_t>(k) * k * A.P2; e += blockDim.x) {
    const uint32_t i = e % A.P2, c1 = (e / A.P2) % k, c0 = e / (A.P2 * k);
    if (c0 == c1) continue;
    const uint32_t f2 = (1u << c0) | (1u << c1);
    const uint32_t S = sig_expand(sig_unrank(c_lut, A.s_out - 2, i), f2);
    if (A.out_kind == 1) idx1[e] = static_cast<uint16_t>(sig_index(c_lut, S, 1u << c0));
    uint32_t free = S & ~f2;
    for (int t = 0; t < A.nterm; ++t) {
      const int c = mb_ctz(free);
      free &= free - 1u;
      const uint32_t T = S & ~(1u << c);
      uint32_t j = 0;
      bool ok = true;
      switch (A.fkind) {
        case 0: ok = T == f2; break;
        case 1: j = sig_index(c_lut, T & ~(1u << c1), 1u << c0); break;
        case 2: j = sig_index(c_lut, T & ~(1u << c0), 1u << c1); break;
        default: j = sig_index(c_lut, T, f2); break;
      }
      terms[static_cast<size_t>(e) * A.nterm + t] = ok ? (static_cast<uint32_t>(c) << 16) | j : ~0u;
    }
  }
  __syncthreads();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = hist_all + static_cast<size_t>(wid) * 32 * k;
  uint64_t local = 0, upd = 0;
  const uint64_t nbatch = (A.nout + 31) / 32;
  for (uint64_t bt = static_cast<uint64_t>(blockIdx.x) * kHistWarps + wid; bt < nbatch;
       bt += static_cast<uint64_t>(gridDim.x) * kHistWarps) {
    const uint64_t j0 = bt * 32;
    const uint64_t j = j0 + lane;
    const bool live = j < A.nout;
    for (int i = lane; i < 32 * k; i += 32) hist[i] = 0;
    // lane l holds offset of edge j0+l (and lane 31's end via shuffle)
    const uint64_t myoff = A.cn_off[live ? j : A.nout];
    const uint64_t endoff = A.cn_off[min(j0 + 32, A.nout)];
    const uint64_t startoff = __shfl_sync(0xffffffffu, myoff, 0);
    __syncwarp();
    for (uint64_t e0 = startoff; e0 < endoff; e0 += 32) {
      const uint64_t e = e0 + lane;
      // edge of entry e: last lane l with off(l) <= e (binary search over the
      // lanes' offsets; all lanes take part in every shuffle)
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint64_t o = __shfl_sync(0xffffffffu, myoff, lo + step);
        if (o <= e) lo += step;
      }
      if (e < endoff) atomicAdd(hist + lo * k + A.chi[__ldg(A.cn_w + e)], 1u);
    }
    __syncwarp();
    if (live) {
      const uint32_t a = A.out_src[j], b = A.out_nbr[j];
      const uint32_t sab = A.out_slot[j], sba = A.rev[sab];
      const uint32_t ca = A.chi[a], cb = A.chi[b];
      const uint32_t* h = hist + lane * k;
      for (int o = 0; o < 2; ++o) {
        const uint32_t c0 = o ? cb : ca, c1 = o ? ca : cb;
        const uint64_t orow = static_cast<uint64_t>(o ? sba : sab) * A.Pout;
        if (c0 == c1) {
          if (A.out_kind == 2)
            for (uint32_t i = 0; i < A.Pout; ++i) A.out[orow + i] = 0;
          continue;
        }
        const uint64_t* F = nullptr;
        if (A.fkind == 1) F = A.F + static_cast<uint64_t>(o ? b : a) * A.PF;
        else if (A.fkind == 2) F = A.F + static_cast<uint64_t>(o ? a : b) * A.PF;
        else if (A.fkind == 3) F = A.F + static_cast<uint64_t>((o == 0) != (A.sw01 != 0) ? sab : sba) * A.PF;
        const uint32_t tb = (c0 * k + c1) * A.P2;
        for (uint32_t i = 0; i < A.P2; ++i) {
          const uint32_t* tt = terms + static_cast<size_t>(tb + i) * A.nterm;
          uint64_t v = 0;
          for (int t = 0; t < A.nterm; ++t) {
            const uint32_t x = tt[t];
            if (x == ~0u) continue;
            const uint32_t hc = h[x >> 16];
            if (!hc) continue;
            const uint64_t f = F ? __ldg(F + (x & 0xFFFFu)) : 1ull;
            if (!f) continue;
            v = add_ck(v, mul_ck(f, hc, A.err), A.err);
            ++upd;
          }
          if (A.out_kind == 2) {
            A.out[orow + i] = v;
          } else if (v) {
            if (A.out_kind == 0)
              local = add_ck(local, v, A.err);
            else
              atomic_add_ck(reinterpret_cast<u64*>(A.out) + static_cast<uint64_t>(o ? b : a) * A.Pout +
                                idx1[tb + i], v, A.err);
          }
        }
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

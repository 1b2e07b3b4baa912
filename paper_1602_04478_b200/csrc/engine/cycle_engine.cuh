// General cycle-block solver (any length L >= 3, any node/edge annotations,
// 0/1/2 boundary nodes).  Included by engine.cu after its helpers.
//
// Degree-based (DB) evaluation, reference engine.cpp:212-241 and paper §5.1
// Eq. 1: every labelled match of the cycle has exactly one position h holding
// its (degree, id)-highest vertex x.  For each h the cycle is split into two
// half paths that start at x and meet at a position d; every other image must
// rank below x (the cap).  The reference splits at d = h + floor(L/2) and
// records interior boundary images in extra key slots; here d is chosen as a
// boundary position whenever h is not one (a valid split for Eq. 1 because
// both halves are rebuilt per h), so at most one boundary image is ever carried
// as a recorded key.
//
// The half-path tables of the reference (keys (x, v[, r]), hash maps) become
// level-synchronous frontiers on the device: sorted arrays of packed keys
// (x, v, r) with a dense colour-set row per key.  One hop expands every entry
// along the CSR row of v (relation = graph edges, optionally weighted by an
// edge-keyed child table), joins the node annotation of the new position,
// and aggregates equal keys by a radix sort + segmented add.  The two halves
// are then merged with the disjoint-union join (S+ n S- = {chi x, chi v}).
// Anchors are processed in batches so frontier memory stays bounded.

struct TabView {
  int kind = 0;  // 0 none, 1 scalar, 2 vertex, 3 edge, 4 pair
  int s = 0;
  uint32_t P = 0;
  uint32_t rs = 0;  // row stride (vertex/edge tables are [row][colouring][P]); pair tables: P
  uint64_t* data = nullptr;  // pre-offset to the colouring's slice
  uint64_t size = 0;         // readable elements from data (bounds checks)
  uint64_t size_t_ = 0;      // readable elements from data_t
  // pair tables: CSR by first key (off[n+1], cols) and its transpose
  const uint64_t* off = nullptr;
  const uint32_t* cols = nullptr;
  const uint64_t* off_t = nullptr;
  const uint32_t* cols_t = nullptr;
  const uint64_t* data_t = nullptr;
};

struct GraphView {
  uint32_t n;
  uint64_t m2;
  const uint64_t* off;
  const uint32_t* adj;
  const uint32_t* rev;
  const uint32_t* rank;
  const uint8_t* chi;  // pre-offset to the colouring; stride kChiStride
  int ordered;         // device ids descend with rank: rank(w) < rank(x) <=> w > x
};

__device__ __forceinline__ uint32_t vcol(const GraphView& G, uint32_t v) {
  return G.chi[static_cast<uint64_t>(v) * kChiStride];
}

struct HopArgs {
  GraphView G;
  // input frontier
  const uint64_t* key_in;
  const uint64_t* pay_in;
  uint64_t n_in;
  int s_in;
  uint32_t P_in;
  int first_hop;  // input keys are (x, x): fixed colours {chi x}
  int in_has_r;
  // work decomposition
  const uint64_t* woff;  // exclusive scan of per-entry work (n_in + 1)
  const uint64_t* sstart;  // per entry: first relation slot walked
  uint64_t W;
  const uint64_t* tstart;  // per tile of kHopTile items: the entry of its first item (k_tile_starts)
  // per-item results of the keys pass, read back by the accumulate pass: the
  // hash slot of the item's output key (~0u: the item was dropped) and the
  // colour of its new vertex
  uint32_t* item_slot;     // (k_slot_to_index turns the slots into dense row indices between the passes)
  uint16_t* item_col;      // colours of the item's (x, v, w), 4 bits each
  const uint8_t* ecol;     // per frontier entry: colours of (x, v), 4 bits each (k_hop_work)
  int unchecked;           // host bound: no output entry can reach 2^63 (plain adds, no return value)
  // hop relation: rows roff/radj (graph CSR or a pair table's CSR)
  const uint64_t* roff;
  const uint32_t* radj;
  const uint64_t* etab;  // relation payload (edge or pair table), may be null
  uint32_t Pe;
  int se;
  int e_rev;
  const uint64_t* ntab;  // node child at the new position, may be null
  uint32_t Pn;
  int sn;
  int record;            // the new position is the recorded boundary
  uint32_t rse, rsn;     // row strides of etab / ntab
  uint64_t n_etab, n_ntab;  // readable elements from etab / ntab (bounds checks)
  // output contributions
  int s_out;
  uint32_t P_out;
  int out_has_r;
  int bits;
  uint64_t* key_out;     // [distinct keys] (keys pass)
  uint64_t* row_out;     // [distinct keys][P_out] (accumulate pass)
  // open-addressing hash table of the output keys: slot -> dense index
  uint64_t* ht_key;
  uint32_t* ht_idx;
  uint64_t ht_mask;
  int ht_shift;
  unsigned long long* n_keys;
  int* err;
  u64* updates;
};

constexpr uint64_t kEmptyKey = ~0ull;

__device__ __forceinline__ uint64_t ht_slot(uint64_t key, int shift) {
  return (key * 0x9E3779B97F4A7C15ull) >> shift;
}

// Inserts `key` (keys pass): the first inserter takes the next dense index.
// Returns the key's slot.
__device__ __forceinline__ uint64_t ht_insert(uint64_t* ht_key, uint32_t* ht_idx, uint64_t mask, int shift,
                                              uint64_t key, unsigned long long* n_keys, uint64_t* key_out) {
  uint64_t h = ht_slot(key, shift);
  while (true) {
    const uint64_t cur = ht_key[h];
    if (cur == key) return h;
    if (cur == kEmptyKey) {
      const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(ht_key + h), kEmptyKey, key);
      if (prev == kEmptyKey) {
        const uint32_t idx = static_cast<uint32_t>(atomicAdd(n_keys, 1ull));
        ht_idx[h] = idx;
        key_out[idx] = key;
        return h;
      }
      if (prev == key) return h;
    }
    h = (h + 1) & mask;
  }
}

// Dense index of `key` in a table that is read and written by the same
// launch (the pair table of k_half_merge): inserts on first use; a thread
// that finds the key before its inserter has published the index waits for
// it (ht_idx starts as all ~0u).
__device__ __forceinline__ uint32_t ht_get(uint64_t* ht_key, uint32_t* ht_idx, uint64_t mask, int shift, uint64_t key,
                                           unsigned long long* n_keys, uint64_t* key_out, uint64_t* rows = nullptr,
                                           uint32_t P = 0) {
  uint64_t h = ht_slot(key, shift);
  while (true) {
    uint64_t cur = *reinterpret_cast<volatile uint64_t*>(ht_key + h);
    if (cur == kEmptyKey) {
      cur = atomicCAS(reinterpret_cast<unsigned long long*>(ht_key + h), kEmptyKey, key);
      if (cur == kEmptyKey) {
        const uint32_t idx = static_cast<uint32_t>(atomicAdd(n_keys, 1ull));
        key_out[idx] = key;
        if (rows)
          for (uint32_t j = 0; j < P; ++j) rows[static_cast<uint64_t>(idx) * P + j] = 0;
        __threadfence();
        atomicExch(ht_idx + h, idx);
        return idx;
      }
    }
    if (cur == key) {
      uint32_t idx;
      do {
        idx = *reinterpret_cast<volatile uint32_t*>(ht_idx + h);
      } while (idx == ~0u);
      return idx;
    }
    h = (h + 1) & mask;
  }
}

// Dense index of a key known to be present (after the keys pass), or ~0u.
__device__ __forceinline__ uint32_t ht_find(const uint64_t* __restrict__ ht_key, const uint32_t* __restrict__ ht_idx,
                                            uint64_t mask, int shift, uint64_t key) {
  uint64_t h = ht_slot(key, shift);
  while (true) {
    const uint64_t cur = ht_key[h];
    if (cur == key) return ht_idx[h];
    if (cur == kEmptyKey) return ~0u;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ uint64_t pack_key(uint64_t x, uint64_t v, uint64_t r, int has_r, int bits) {
  return has_r ? (((x << bits) | v) << bits) | r : (x << bits) | v;
}

__device__ __forceinline__ void unpack_key(uint64_t key, int has_r, int bits, uint32_t& x, uint32_t& v,
                                           uint32_t& r) {
  const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  if (has_r) {
    r = static_cast<uint32_t>(key & mask);
    key >>= bits;
  } else {
    r = 0xFFFFFFFFu;
  }
  v = static_cast<uint32_t>(key & mask);
  x = static_cast<uint32_t>(key >> bits);
}

// Per frontier entry (x, v): the relation row of v, restricted to neighbours
// ranked below the anchor x.  With degree-ordered device ids those are exactly
// the ids above x, i.e. a suffix of the sorted row (graph CSR and pair-table
// CSR rows are both sorted), so the work is counted and walked without the
// neighbours that would only be discarded.
__global__ void k_hop_work(const uint64_t* __restrict__ key_in, uint64_t n_in, int has_r, int bits,
                           const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj, int ordered,
                           uint64_t* __restrict__ work, uint64_t* __restrict__ sstart,
                           const uint8_t* __restrict__ chi, uint32_t n, uint8_t* __restrict__ ecol) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n_in) return;
  uint32_t x, v, r;
  unpack_key(key_in[i], has_r, bits, x, v, r);
  // the entry's key colours, read once here instead of once per work item
  ecol[i] = (x < n && v < n) ? static_cast<uint8_t>(chi[static_cast<uint64_t>(x) * kChiStride] |
                                                   (chi[static_cast<uint64_t>(v) * kChiStride] << 4))
                             : 0;
  uint64_t lo = off[v], hi = off[v + 1];
  if (ordered) {
    uint64_t a = lo, b = hi;  // first slot with adj > x
    while (a < b) {
      const uint64_t mid = (a + b) >> 1;
      if (adj[mid] <= x) a = mid + 1; else b = mid;
    }
    lo = a;
  }
  sstart[i] = lo;
  work[i] = hi - lo;
}

// S2[x] = sum of deg(v) over the suffix neighbours v of x (ids above x in the
// degree order): an upper bound of the second hop's work from anchor x.
__global__ void k_suffix_work(uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ adj,
                              uint64_t* __restrict__ s2) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  uint64_t lo = off[x], hi = off[x + 1];
  uint64_t a = lo, b = hi;
  while (a < b) {
    const uint64_t mid = (a + b) >> 1;
    if (adj[mid] <= x) a = mid + 1; else b = mid;
  }
  uint64_t t = 0;
  for (uint64_t e = a; e < hi; ++e) {
    const uint32_t v = adj[e];
    t += off[v + 1] - off[v];
  }
  s2[x] = t;
}

constexpr int kHopTile = 256;  // items per CTA of k_hop_expand

// tstart[t] = the frontier entry holding item t * kHopTile (the last i with
// woff[i] <= item), tstart[ntiles] = the entry of the last item: a thread per
// tile, so the binary searches of a hop run in parallel instead of one per
// CTA of k_hop_expand in front of a barrier (ncu: 25 % of that kernel's stall
// samples sat on the barrier).
__global__ void k_tile_starts(const uint64_t* __restrict__ woff, uint64_t n_in, uint64_t W, uint64_t ntiles,
                              uint64_t* __restrict__ tstart) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (t > ntiles) return;
  const uint64_t it = min(t * kHopTile, W - 1);
  uint64_t lo = 0, hi = n_in;
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (woff[mid] <= it) lo = mid; else hi = mid;
  }
  tstart[t] = lo;
}

// Between the passes: every live item's hash slot becomes the dense row index
// its key was given (one independent gather per thread, instead of a probe at
// the head of each accumulate thread's dependent chain).
__global__ void k_slot_to_index(uint32_t* __restrict__ item_slot, const uint32_t* __restrict__ ht_idx, uint64_t W) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= W) return;
  const uint32_t s = item_slot[i];
  if (s != ~0u) item_slot[i] = ht_idx[s];
}

// One thread per (frontier entry, neighbour) work item, two passes over the
// same items.  KEYS: the item's output key (x, w[, r]) is inserted into an
// open-addressing hash table that hands out dense indices.  ACCUMULATE: the
// item's contributions are added straight into the dense row of its key.
// This replaces the reference's hash-map accumulate (table.cpp:38-54) without
// materialising a row per item or sorting: aggregation costs one probe plus
// the row atomics of the nonzero contributions.  The CTA locates its items'
// entries once: the woff span of its tile is staged in shared memory.
// MODE 0: keys pass, 1: accumulate pass (find), 2: one fused pass (insert or
// find, the inserter zeroes the row before publishing its index).
template <int MODE>
__global__ void __launch_bounds__(kHopTile) k_hop_expand(HopArgs A) {
  constexpr bool KEYS = MODE == 0;
  __shared__ uint64_t s_woff[kHopTile + 1];
  __shared__ uint32_t s_binom[KEYS ? 1 : (kMaxColors + 1) * kBinomStride];
  if (!KEYS) stage_binom(c_lut, s_binom);
  const uint64_t item0 = static_cast<uint64_t>(blockIdx.x) * kHopTile;
  const uint64_t item = item0 + threadIdx.x;
  auto entry_of = [&](uint64_t it) {  // last i with woff[i] <= it
    uint64_t lo = 0, hi = A.n_in;
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (A.woff[mid] <= it) lo = mid; else hi = mid;
    }
    return lo;
  };
  // the tile's entries lie in [tstart[b], tstart[b + 1]] (k_tile_starts)
  const uint64_t e0 = A.tstart[blockIdx.x], cnt = A.tstart[blockIdx.x + 1] - e0 + 1;
  const bool staged = cnt <= kHopTile;
  if (staged)
    for (uint64_t j = threadIdx.x; j <= cnt && e0 + j <= A.n_in; j += kHopTile) s_woff[j] = A.woff[e0 + j];
  __syncthreads();
  if (item >= A.W) return;
  uint64_t i;
  if (staged) {
    uint64_t lo = 0, hi = cnt;
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (s_woff[mid] <= item) lo = mid; else hi = mid;
    }
    i = e0 + lo;
  } else {
    i = entry_of(item);
  }
  // Plain hops (no edge or node table joined at the new vertex): the keys
  // pass left each live item's row index (via k_slot_to_index) and colours, so
  // the accumulate pass reads neither the key, the neighbour nor the hash
  // table again; the input row is loaded four entries at a time (independent
  // loads) and, under the host's bound, added with plain reductions.
  if (MODE == 1 && !A.etab && !A.ntab) {
    const uint32_t oi = A.item_slot[item];
    if (oi == ~0u) return;
    const uint32_t col = A.item_col[item];
    const uint32_t cx = col & 15u, cv = (col >> 4) & 15u, cw = col >> 8;
    const uint32_t fin = A.first_hop ? (1u << cx) : ((1u << cx) | (1u << cv));
    const uint32_t fw = 1u << cw, fout = (1u << cx) | fw;
    u64* row = reinterpret_cast<u64*>(A.row_out + static_cast<uint64_t>(oi) * A.P_out);
    const uint64_t* prow = A.pay_in + i * A.P_in;
    const int t_in = A.s_in - mb_popc(fin);
    uint32_t nupd = 0;
    for (uint32_t b = 0; b < A.P_in; b += 4) {
      uint64_t pv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) pv[u] = b + u < A.P_in ? prow[b + u] : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!pv[u]) continue;
        const uint32_t Sin = sig_expand(sig_unrank(c_lut, t_in, b + u), fin);
        if (Sin & fw) continue;
        const uint32_t S2 = Sin | fw;
        const uint32_t o = sig_index_sm(s_binom, S2, fout);
        if (o >= A.P_out || mb_popc(S2) != A.s_out) {
          atomicOr(A.err, 16);
          continue;
        }
        if (A.unchecked) atomicAdd(row + o, static_cast<u64>(pv[u]));
        else atomic_add_ck(row + o, pv[u], A.err);
        ++nupd;
      }
    }
    const unsigned am = __activemask();
    const unsigned tot = __reduce_add_sync(am, nupd);
    if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(am) - 1) && tot) atomicAdd(A.updates, static_cast<u64>(tot));
    return;
  }
  // accumulate pass: items the keys pass dropped (no slot) are done; live ones
  // carry their row index and colours
  if (MODE == 1 && A.item_slot[item] == ~0u) return;
  uint32_t x, v, r;
  unpack_key(A.key_in[i], A.in_has_r, A.bits, x, v, r);
  if (MODE == 0) A.item_slot[item] = ~0u;  // until the item proves live below
  if (x >= A.G.n || v >= A.G.n) {
    if (MODE != 1) atomicOr(A.err, 32);
    return;
  }
  const uint64_t slot = A.sstart[i] + (item - A.woff[i]);
  if (slot >= A.roff[A.G.n]) {
    if (MODE != 1) atomicOr(A.err, 64);
    return;
  }
  const uint32_t w = A.radj[slot];
  if (w >= A.G.n) {
    if (MODE != 1) atomicOr(A.err, 128);
    return;
  }
  if (!(A.G.ordered || A.G.rank[w] < A.G.rank[x])) return;
  const uint32_t ec = A.ecol[i];
  // (the accumulate pass takes the neighbour's colour from the keys pass)
  const uint32_t cx = ec & 15u, cv = ec >> 4, cw = MODE == 1 ? A.item_col[item] >> 8 : vcol(A.G, w);
  const uint32_t fin = A.first_hop ? (1u << cx) : ((1u << cx) | (1u << cv));
  const uint32_t fw = 1u << cw, fv = 1u << cv;
  if (fin & fw) return;  // the new vertex repeats a key colour: no colourful extension
  const uint32_t rr = A.record ? w : r;
  const uint64_t key = pack_key(x, w, rr, A.out_has_r, A.bits);
  if (KEYS) {
    const uint64_t h = ht_insert(A.ht_key, A.ht_idx, A.ht_mask, A.ht_shift, key, A.n_keys, A.key_out);
    A.item_slot[item] = static_cast<uint32_t>(h);
    A.item_col[item] = static_cast<uint16_t>(cx | (cv << 4) | (cw << 8));
    return;
  }
  // accumulate pass: the row index the keys pass (and k_slot_to_index) left
  const uint32_t oi = MODE == 2 ? ht_get(A.ht_key, A.ht_idx, A.ht_mask, A.ht_shift, key, A.n_keys, A.key_out,
                                          A.row_out, A.P_out)
                                  : A.item_slot[item];
  if (oi == ~0u) {
    atomicOr(A.err, 64);
    return;
  }
  u64* row = reinterpret_cast<u64*>(A.row_out + static_cast<uint64_t>(oi) * A.P_out);
  const uint32_t fout = (1u << cx) | fw;
  const uint64_t* prow = A.pay_in + i * A.P_in;
  const int t_in = A.s_in - mb_popc(fin);
  const uint64_t erow = A.etab ? (A.e_rev ? A.G.rev[slot] : slot) * A.rse : 0;
  uint32_t nupd = 0;
  for (uint32_t ii = 0; ii < A.P_in; ++ii) {
    const uint64_t pv = prow[ii];
    if (!pv) continue;
    const uint32_t Sin = sig_expand(sig_unrank(c_lut, t_in, ii), fin);
    if (Sin & fw) continue;
    const uint32_t ne = A.etab ? A.Pe : 1u;
    for (uint32_t ie = 0; ie < ne; ++ie) {
      uint32_t S1;
      uint64_t v1;
      if (A.etab) {
        if (erow + ie >= A.n_etab) {
          atomicOr(A.err, 256);
          continue;
        }
        const uint64_t ev = A.etab[erow + ie];
        if (!ev) continue;
        const uint32_t E = sig_expand(sig_unrank(c_lut, A.se - 2, ie), fv | fw);
        if ((E & Sin) != fv) continue;
        S1 = Sin | E;
        v1 = mul_ck(pv, ev, A.err);
      } else {
        S1 = Sin | fw;
        v1 = pv;
      }
      const uint32_t nn = A.ntab ? A.Pn : 1u;
      for (uint32_t in = 0; in < nn; ++in) {
        uint32_t S2;
        uint64_t v2;
        if (A.ntab) {
          if (static_cast<uint64_t>(w) * A.rsn + in >= A.n_ntab) {
            atomicOr(A.err, 512);
            continue;
          }
          const uint64_t nv = A.ntab[static_cast<uint64_t>(w) * A.rsn + in];
          if (!nv) continue;
          const uint32_t Nn = sig_expand(sig_unrank(c_lut, A.sn - 1, in), fw);
          if ((Nn & S1) != fw) continue;
          S2 = S1 | Nn;
          v2 = mul_ck(v1, nv, A.err);
        } else {
          S2 = S1;
          v2 = v1;
        }
        const uint32_t o = sig_index_sm(s_binom, S2, fout);
        if (o >= A.P_out || mb_popc(S2) != A.s_out) {
          atomicOr(A.err, 16);  // signature outside the frontier row: plan/popcount bug
          continue;
        }
        atomic_add_ck(row + o, v2, A.err);
        ++nupd;
      }
    }
  }
  const unsigned am = __activemask();
  const unsigned tot = __reduce_add_sync(am, nupd);
  if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(am) - 1) && tot) atomicAdd(A.updates, static_cast<u64>(tot));
}

template <class T>
__global__ void k_iota(T* __restrict__ out, uint64_t W) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < W) out[i] = static_cast<T>(i);
}

__global__ void k_seg_heads(const uint64_t* __restrict__ keys, uint64_t W, uint64_t* __restrict__ head) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= W) return;
  head[i] = (keys[i] != ~0ull) && (i == 0 || keys[i] != keys[i - 1]);
}

// seg = inclusive-scan(head) - 1; accumulate the item's row into its segment.
__global__ void k_seg_accumulate(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                                 const uint64_t* __restrict__ segx, const uint64_t* __restrict__ head,
                                 const uint64_t* __restrict__ rows, uint32_t P, uint64_t W,
                                 uint64_t* __restrict__ key_out, uint64_t* __restrict__ pay_out, int* err) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= W || keys[i] == ~0ull) return;
  const uint64_t seg = segx[i] + head[i] - 1;  // exclusive scan + own head = inclusive
  if (head[i]) key_out[seg] = keys[i];
  const uint64_t* row = rows + static_cast<uint64_t>(idx[i]) * P;
  for (uint32_t j = 0; j < P; ++j)
    if (row[j]) atomic_add_ck(reinterpret_cast<u64*>(pay_out + seg * P + j), row[j], err);
}

// Frontier of the anchors x0, x0 + stride, ... (nx of them): stride > 1 when
// the anchors are dealt cyclically over ranks (vertex-sharded root block).
__global__ void k_init_frontier(uint32_t x0, uint32_t nx, uint32_t stride, int bits, const uint8_t* __restrict__ chi,
                                const uint64_t* __restrict__ utab, uint32_t Pu, uint32_t rsu,
                                uint64_t* __restrict__ key, uint64_t* __restrict__ pay) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nx) return;
  const uint64_t x = x0 + static_cast<uint64_t>(i) * stride;
  key[i] = (x << bits) | x;
  if (utab) {
    for (uint32_t j = 0; j < Pu; ++j) pay[static_cast<uint64_t>(i) * Pu + j] = utab[x * rsu + j];
  } else {
    pay[i] = 1;  // signature {chi x}
  }
}

struct MergeArgs {
  GraphView G;
  // side A (iterated; may carry r), side B (looked up by (x, v))
  const uint64_t* keyA;
  const uint64_t* payA;
  uint64_t nA;
  int sA;
  uint32_t PA;
  int A_has_r;
  const uint64_t* keyB;
  const uint64_t* payB;
  uint64_t nB;
  const uint64_t* htB_key;  // B's hash table (key -> entry)
  const uint32_t* htB_idx;
  uint64_t htB_mask;
  int htB_shift;
  int sB;
  uint32_t PB;
  int bits;
  // output
  int out_kind;  // 1 scalar, 2 vertex, 3 edge, 4 pair (contribution rows)
  // pair outputs: the running pair hash table (key -> dense row index)
  uint64_t* ph_key;
  uint32_t* ph_idx;
  uint64_t ph_mask;
  int ph_shift;
  unsigned long long* ph_n;
  uint64_t* ph_list;  // dense index -> key
  uint64_t* ph_rows;  // [dense index][Pout]
  int key_src0, key_src1;  // 0 = x, 1 = v, 2 = r
  uint64_t* out;
  uint32_t Pout, rso;
  u64* scalar;
  uint32_t scalar_mult;  // rotation-symmetric root cycle: the h = 0 count times L
  uint32_t t_mult;       // pair outputs: also add the contribution this many times at the swapped key
  int* err;
  u64* updates;
};

__device__ __forceinline__ uint64_t find_slot(const GraphView& G, uint32_t p, uint32_t q) {
  uint64_t lo = G.off[p], hi = G.off[p + 1];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (G.adj[mid] < q) lo = mid + 1; else hi = mid;
  }
  return (lo < G.off[p + 1] && G.adj[lo] == q) ? lo : ~0ull;
}

__global__ void __launch_bounds__(256) k_half_merge(MergeArgs A) {
  __shared__ uint32_t s_binom[(kMaxColors + 1) * kBinomStride];
  stage_binom(c_lut, s_binom);
  __syncthreads();
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  uint64_t local = 0, upd = 0;
  if (i < A.nA) {
    uint32_t x, v, r;
    unpack_key(A.keyA[i], A.A_has_r, A.bits, x, v, r);
    const uint64_t kb = (static_cast<uint64_t>(x) << A.bits) | v;
    const uint32_t bi = A.nB ? ht_find(A.htB_key, A.htB_idx, A.htB_mask, A.htB_shift, kb) : ~0u;
    const uint64_t lo = bi;
    bool found = bi != ~0u;
    uint64_t orow = 0, orow_t = 0;
    uint32_t ofix = 0;
    const uint32_t ids[3] = {x, v, r};
    if (found && A.out_kind == 3) {
      const uint32_t p = ids[A.key_src0], q = ids[A.key_src1];
      const uint64_t s = find_slot(A.G, p, q);
      if (s == ~0ull) {
        atomicOr(A.err, 4);  // pair not adjacent: plan/table kind mismatch
        found = false;
      }
      orow = s * A.rso;
      ofix = (1u << vcol(A.G, p)) | (1u << vcol(A.G, q));
    }
    if (found) {
      const uint32_t cx = vcol(A.G, x), cv = vcol(A.G, v);
      const uint32_t fx = 1u << cx, fv = 1u << cv, f2 = fx | fv;
      if (A.out_kind == 2) {
        const uint32_t y = ids[A.key_src0];
        orow = static_cast<uint64_t>(y) * A.rso;
        ofix = 1u << vcol(A.G, y);
      } else if (A.out_kind == 4) {
        // the reference's arity-2 merge output (table.cpp:225-275): rows of
        // the running pair hash table, inserted on first use; the host keeps
        // its capacity above the number of A entries of every launch
        const uint32_t p = ids[A.key_src0], q = ids[A.key_src1];
        const uint64_t key = (static_cast<uint64_t>(p) << A.bits) | q;
        const uint32_t di = ht_get(A.ph_key, A.ph_idx, A.ph_mask, A.ph_shift, key, A.ph_n, A.ph_list);
        orow = static_cast<uint64_t>(di) * A.Pout;
        if (A.t_mult) {
          const uint64_t kt = (static_cast<uint64_t>(q) << A.bits) | p;
          orow_t = static_cast<uint64_t>(ht_get(A.ph_key, A.ph_idx, A.ph_mask, A.ph_shift, kt, A.ph_n, A.ph_list)) *
                   A.Pout;
        }
        ofix = (1u << vcol(A.G, p)) | (1u << vcol(A.G, q));
      }
      const uint64_t* ra = A.payA + i * A.PA;
      const uint64_t* rb = A.payB + lo * A.PB;
      const int ta = A.sA - 2, tb = A.sB - 2;
      // B's nonzero entries with their colour sets, once per A entry (not once
      // per (A entry, A signature)); rows wider than kMergeB take the plain loop
      constexpr uint32_t kMergeB = 32;
      uint32_t sbl[kMergeB];
      uint64_t vbl[kMergeB];
      uint32_t nbl = 0;
      const bool listed = A.PB <= kMergeB;
      if (listed)
        for (uint32_t ib = 0; ib < A.PB; ++ib) {
          const uint64_t vb = rb[ib];
          if (!vb) continue;
          sbl[nbl] = sig_expand(sig_unrank(c_lut, tb, ib), f2);
          vbl[nbl++] = vb;
        }
      auto term = [&](uint32_t Sa, uint64_t va, uint32_t Sb, uint64_t vb) {
        if ((Sa & Sb) != f2) return;
        // a term standing for several equal Eq. 1 terms (reflection
        // symmetry, CycleRunner::solve) is counted that many times
        const uint64_t val = A.out_kind == 1 || A.scalar_mult == 1 ? mul_ck(va, vb, A.err)
                                                                   : mul_ck(mul_ck(va, vb, A.err), A.scalar_mult, A.err);
        ++upd;
        if (A.out_kind == 1) {
          local = add_ck(local, val, A.err);
        } else if (A.out_kind == 4) {
          const uint32_t o = sig_index_sm(s_binom, Sa | Sb, ofix);
          atomic_add_ck(reinterpret_cast<u64*>(A.ph_rows + orow + o), val, A.err);
          if (A.t_mult)
            atomic_add_ck(reinterpret_cast<u64*>(A.ph_rows + orow_t + o),
                          A.t_mult == A.scalar_mult ? val : mul_ck(mul_ck(va, vb, A.err), A.t_mult, A.err), A.err);
        } else {
          atomic_add_ck(reinterpret_cast<u64*>(A.out + orow + sig_index_sm(s_binom, Sa | Sb, ofix)), val, A.err);
        }
      };
      for (uint32_t ia = 0; ia < A.PA; ++ia) {
        const uint64_t va = ra[ia];
        if (!va) continue;
        const uint32_t Sa = sig_expand(sig_unrank(c_lut, ta, ia), f2);
        if (listed) {
          for (uint32_t j = 0; j < nbl; ++j) term(Sa, va, sbl[j], vbl[j]);
        } else {
          for (uint32_t ib = 0; ib < A.PB; ++ib) {
            const uint64_t vb = rb[ib];
            if (vb) term(Sa, va, sig_expand(sig_unrank(c_lut, tb, ib), f2), vb);
          }
        }
      }
    }
  }
  if (A.out_kind == 1) {
    for (int o = 16; o > 0; o >>= 1) local = add_ck(local, __shfl_down_sync(0xffffffffu, local, o), A.err);
    if ((threadIdx.x & 31) == 0 && local) atomic_add_ck(A.scalar, mul_ck(local, A.scalar_mult, A.err), A.err);
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(0xffffffffu, upd, o);
  if ((threadIdx.x & 31) == 0 && upd) atomicAdd(A.updates, static_cast<u64>(upd));
}

// Host side --------------------------------------------------------------------

struct CycleDesc {
  int L = 0;
  std::vector<TabView> node, edge;  // per position / per edge (edge i: i -> i+1)
  std::vector<char> edge_fwd;
  std::vector<int> bpos;
  TabView out;
  int s_out = 0;
};

struct Frontier {
  DBuf key, pay;  // entries in insertion order (not sorted)
  uint64_t n = 0;
  int s = 0;
  uint32_t P = 0;
  int has_r = 0;
  DBuf ht_key, ht_idx;  // hash table key -> entry (built by the hop that produced it)
  long double ub = 1e30L;  // host upper bound of any row entry (1e30: unknown)
  uint64_t ht_mask = 0;
  int ht_shift = 64;
};

// Rows of a relation as seen when walking from the first key to the second.
struct Relation {
  const uint64_t* off;
  const uint32_t* adj;
  const uint64_t* pay = nullptr;  // per-slot payload rows (null: plain graph edges)
  uint64_t size = 0;              // readable elements from pay
  uint32_t P = 0, rs = 0;         // entries per row, row stride
  int s = 0;
  int use_rev = 0;                // payload row = rev[slot] (edge tables walked backwards)
};

__global__ void k_pair_csr(uint32_t n, const uint64_t* __restrict__ keys, uint64_t nk, int bits,
                           uint64_t* __restrict__ off, uint32_t* __restrict__ cols) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < nk) cols[i] = static_cast<uint32_t>(keys[i] & ((1ull << bits) - 1));
  if (i <= n) {
    const uint64_t target = i << bits;
    uint64_t lo = 0, hi = nk;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    off[i] = lo;
  }
}

__global__ void k_swap_pair_keys(const uint64_t* __restrict__ in, uint64_t nk, int bits, uint64_t* __restrict__ out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nk) return;
  const uint64_t mask = (1ull << bits) - 1;
  out[i] = ((in[i] & mask) << bits) | (in[i] >> bits);
}

__global__ void k_gather_rows32(const uint32_t* __restrict__ idx, const uint64_t* __restrict__ in, uint32_t P,
                                uint64_t nk, uint64_t* __restrict__ out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nk * P) return;
  const uint64_t r = i / P, j = i - r * P;
  out[i] = in[static_cast<uint64_t>(idx[r]) * P + j];
}

// Re-inserts the dense keys 0..n-1 of a pair table into a larger hash table.
__global__ void k_pair_rehash(const uint64_t* __restrict__ list, uint64_t n, uint64_t* __restrict__ ht_key,
                              uint32_t* __restrict__ ht_idx, uint64_t mask, int shift) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint64_t key = list[i];
  uint64_t h = ht_slot(key, shift);
  while (atomicCAS(reinterpret_cast<unsigned long long*>(ht_key + h), kEmptyKey, key) != kEmptyKey) h = (h + 1) & mask;
  ht_idx[h] = static_cast<uint32_t>(i);
}

__global__ void k_gather_rows(const uint64_t* __restrict__ idx, const uint64_t* __restrict__ in, uint32_t P,
                              uint64_t nk, uint64_t* __restrict__ out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nk * P) return;
  const uint64_t r = i / P, j = i - r * P;
  out[i] = in[idx[r] * P + j];
}

struct PairHash {  // running pair-keyed output of a block (merge contributions)
  DBuf key, idx;     // open-addressing slots (2 x rows)
  DBuf list, rows;   // dense index -> key, [dense index][P] u64
  DBuf counter;      // number of keys (device)
  uint64_t cap_rows = 0, n = 0;  // row capacity, keys after the last merge (host)
  int shift = 64;
};

struct CycleRunner {
  GraphView G;
  int k = 0;
  int bits = 0;
  cudaStream_t stream;
  int* err;
  u64* scalar;
  u64* upd;
  std::function<void(const char*, const std::function<void()>&, uint64_t)> launch_b;
  void launch(const char* name, const std::function<void()>& f, uint64_t bytes = 0) { launch_b(name, f, bytes); }
  std::function<void(const uint64_t*, uint64_t*, uint64_t)> scan;  // exclusive scan of n+1
  DBuf sort_tmp;
  uint64_t mem_budget = 6ull << 30;  // bytes of per-hop scratch per batch
  uint64_t max_deg = 0;               // largest degree of the graph (host bounds of plain hops)
  bool force = false;                 // single-anchor batch: no further split
  uint32_t h_mult = 1;                // Eq. 1 terms represented by each evaluated h
  uint32_t h_mult_t = 0;              // ... and terms equal to it with the pair keys swapped
  static bool no_swap_sym() {
    static const bool off = std::getenv("MB_NO_SWAP_SYMMETRY") != nullptr;
    return off;
  }
  PairHash pairs;
  // pair-table streaming (engine_host.inc, streamed_root_of): called with a
  // full running table; it builds the partial table, evaluates the root on it
  // and drops it
  std::function<void()> pair_flush;
  uint64_t pair_flush_bytes = ~0ull;

  static uint64_t binom(int a, int b) { return binom_host(a, b); }

  double wait_s = 0;  // host time blocked in d2h (MB_DEBUG_BATCH)

  bool overflowed() {
    int e = 0;
    MB_CUDA(cudaMemcpyAsync(&e, err, sizeof(int), cudaMemcpyDeviceToHost, stream));
    MB_CUDA(cudaStreamSynchronize(stream));
    return (e & 1) != 0;
  }

  uint64_t d2h(const uint64_t* p) {
    uint64_t v = 0;
    const auto t0 = std::chrono::steady_clock::now();
    MB_CUDA(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, stream));
    MB_CUDA(cudaStreamSynchronize(stream));
    wait_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return v;
  }

  // Radix sort of (key, value) pairs on the low `end_bit` key bits only:
  // packed keys use 2 or 3 fields of `bits` bits, so most of the 64 are zero.
  template <class V>
  void sort_pairs(const uint64_t* kin, uint64_t* kout, const V* vin, V* vout, uint64_t W, int end_bit) {
    end_bit = std::min(64, std::max(1, end_bit));
    size_t tmp = 0;
    MB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, static_cast<int64_t>(W), 0, end_bit,
                                            stream));
    if (sort_tmp.bytes < tmp) sort_tmp.alloc(tmp);
    launch("cub_radix_sort", [&] {
      MB_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, tmp, kin, kout, vin, vout, static_cast<int64_t>(W), 0,
                                              end_bit, stream));
    });
  }

  // Sort contributions (keys[W], rows[W][P]) and add equal keys: the
  // reference's hash-map accumulate (table.cpp:38-54) as sort + segmented add.
  // Keys equal to UINT64_MAX are dropped.  Valid keys are below 2^key_bits;
  // sorting key_bits + 1 bits keeps the sentinel (that bit set) after them.
  void aggregate(const DBuf& keys, const DBuf& rows, uint64_t W, uint32_t P, DBuf& out_key, DBuf& out_pay,
                 uint64_t& out_n, int key_bits) {
    if (W >= 0xFFFFFFFFull) fail(kSpec, "cycle engine: more than 2^32 contributions in one aggregation");
    DBuf idx(W * 4), skeys(W * 8), sidx(W * 4);
    launch("cycle_iota", [&] { k_iota<uint32_t><<<grid_for(W, 256), 256, 0, stream>>>(idx.as<uint32_t>(), W); });
    sort_pairs(keys.as<uint64_t>(), skeys.as<uint64_t>(), idx.as<uint32_t>(), sidx.as<uint32_t>(), W, key_bits + 1);
    DBuf head((W + 1) * 8), segx((W + 1) * 8);
    MB_CUDA(cudaMemsetAsync(head.p, 0, (W + 1) * 8, stream));
    launch("cycle_seg_heads", [&] {
      k_seg_heads<<<grid_for(W, 256), 256, 0, stream>>>(skeys.as<uint64_t>(), W, head.as<uint64_t>());
    });
    scan(head.as<uint64_t>(), segx.as<uint64_t>(), W + 1);
    out_n = d2h(segx.as<uint64_t>() + W);
    out_key.alloc(std::max<uint64_t>(out_n, 1) * 8);
    out_pay.alloc(std::max<uint64_t>(out_n * P, 1) * 8);
    MB_CUDA(cudaMemsetAsync(out_pay.p, 0, out_pay.bytes, stream));
    if (out_n)
      launch("cycle_seg_accumulate", [&] {
        k_seg_accumulate<<<grid_for(W, 256), 256, 0, stream>>>(skeys.as<uint64_t>(), sidx.as<uint32_t>(),
                                                               segx.as<uint64_t>(), head.as<uint64_t>(),
                                                               rows.as<uint64_t>(), P, W, out_key.as<uint64_t>(),
                                                               out_pay.as<uint64_t>(), err);
      });
  }

  // Returns false when the hop exceeded the scratch budget (caller splits the batch).
  uint64_t last_over = 0;  // scratch bytes the last refused hop needed
  uint64_t batch_need = 0;  // largest hop scratch of the current batch
  std::function<const std::vector<double>&()> s2_prefix;  // prefix sums of S2 (host, per graph)

  bool hop(const Frontier& in, Frontier& out, const Relation& rel, const TabView& nt, bool record, bool first,
           bool force_hop) {
    out.has_r = in.has_r || record;
    out.s = in.s + 1 + (rel.pay ? rel.s - 2 : 0) + (nt.kind ? nt.s - 1 : 0);
    out.P = static_cast<uint32_t>(binom(k - 2, out.s - 2));
    out.n = 0;
    if (in.n == 0) return true;
    DBuf work((in.n + 1) * 8), woff((in.n + 1) * 8), sstart(std::max<uint64_t>(in.n, 1) * 8);
    DBuf ecol(std::max<uint64_t>(in.n, 1));
    MB_CUDA(cudaMemsetAsync(work.p, 0, (in.n + 1) * 8, stream));
    launch("cycle_hop_work", [&] {
      k_hop_work<<<grid_for(in.n, 256), 256, 0, stream>>>(in.key.as<uint64_t>(), in.n, in.has_r, bits, rel.off,
                                                          rel.adj, G.ordered, work.as<uint64_t>(),
                                                          sstart.as<uint64_t>(), G.chi, G.n, ecol.as<uint8_t>());
    });
    // an output entry sums at most max_deg items x P_in entries of the input
    // (plain hops; joined tables have no host bound: checked adds)
    out.ub = (rel.pay || nt.kind) ? 1e30L : in.ub * static_cast<long double>(std::max<uint64_t>(max_deg, 1)) * in.P;
    scan(work.as<uint64_t>(), woff.as<uint64_t>(), in.n + 1);
    const uint64_t W = d2h(woff.as<uint64_t>() + in.n);
    if (W == 0) return true;
    // scratch: 2W hash slots (12 B), W keys, and at most W rows
    // (+ 5 B per item: the keys pass's slot and colour, + the tile starts)
    batch_need = std::max<uint64_t>(batch_need, W * (out.P * 8ull + 47));
    if (W * (out.P * 8ull + 47) > mem_budget && !force_hop) {
      last_over = W * (out.P * 8ull + 47);
      return false;
    }
    // hash table: a power of two >= 2 W slots (load <= 1/2)
    int lg = 1;
    while ((1ull << lg) < 2 * W) ++lg;
    const uint64_t cap = 1ull << lg;
    if (cap > (1ull << 31)) fail(kBudget, "cycle engine: a single hop needs more than 2^31 hash slots");
    out.ht_key.alloc(cap * 8);
    out.ht_idx.alloc(cap * 4);
    out.ht_mask = cap - 1;
    out.ht_shift = 64 - lg;
    MB_CUDA(cudaMemsetAsync(out.ht_key.p, 0xFF, cap * 8, stream));
    out.key.alloc(W * 8);
    DBuf nk(8);
    MB_CUDA(cudaMemsetAsync(nk.p, 0, 8, stream));
    HopArgs A{};
    A.G = G;
    A.key_in = in.key.as<uint64_t>();
    A.pay_in = in.pay.as<uint64_t>();
    A.n_in = in.n;
    A.s_in = in.s;
    A.P_in = in.P;
    A.first_hop = first;
    A.in_has_r = in.has_r;
    A.woff = woff.as<uint64_t>();
    A.sstart = sstart.as<uint64_t>();
    A.W = W;
    A.roff = rel.off;
    A.radj = rel.adj;
    if (rel.pay) A.etab = rel.pay, A.Pe = rel.P, A.rse = rel.rs, A.se = rel.s, A.e_rev = rel.use_rev, A.n_etab = rel.size;
    if (nt.kind) A.ntab = nt.data, A.Pn = nt.P, A.rsn = nt.rs, A.sn = nt.s, A.n_ntab = nt.size;
    A.record = record;
    A.s_out = out.s;
    A.P_out = out.P;
    A.out_has_r = out.has_r;
    A.bits = bits;
    A.key_out = out.key.as<uint64_t>();
    A.ht_key = out.ht_key.as<uint64_t>();
    A.ht_idx = out.ht_idx.as<uint32_t>();
    A.ht_mask = out.ht_mask;
    A.ht_shift = out.ht_shift;
    A.n_keys = reinterpret_cast<unsigned long long*>(nk.p);
    A.err = err;
    A.updates = upd;
    const uint64_t ntiles = (W + kHopTile - 1) / kHopTile;
    DBuf tstart((ntiles + 1) * 8), item_slot(W * 4), item_col(W * 2);
    launch("cycle_tile_starts", [&] {
      k_tile_starts<<<grid_for(ntiles + 1, 256), 256, 0, stream>>>(woff.as<uint64_t>(), in.n, W, ntiles,
                                                                   tstart.as<uint64_t>());
    });
    A.tstart = tstart.as<uint64_t>();
    A.item_slot = item_slot.as<uint32_t>(), A.item_col = item_col.as<uint16_t>();
    A.ecol = ecol.as<uint8_t>();
    A.unchecked = out.ub < 9.0e18L ? 1 : 0;
    static const bool dbg = std::getenv("MB_DEBUG_HOPS") != nullptr;
    // compulsory bytes: per item its neighbour id, colour and one probe
    // (8-byte key) per pass; per input entry its key, work offsets and row;
    // per output key its slot and row
    const uint64_t hop_bytes = W * (4 + 1 + 2 * 8) + in.n * (8 + 16 + 8ull * in.P);
    // two passes (keys, then rows) by default: the fused pass measured 12 %
    // slower on the theta (n = 20k: 19.7 vs 17.1 s) and 30 % on R-MAT scale
    // 18 (7.0 vs 5.4 s), 6 % faster on config 4 (155 vs 165 s)
    static const bool fused = std::getenv("MB_FUSED_HOPS") != nullptr;
    if (!fused) {
      launch("cycle_hop_keys", [&] { k_hop_expand<0><<<grid_for(W, kHopTile), kHopTile, 0, stream>>>(A); },
             hop_bytes / 2);
      out.n = d2h(nk.as<uint64_t>());
      out.pay.alloc(std::max<uint64_t>(out.n * out.P, 1) * 8);
      if (out.n) MB_CUDA(cudaMemsetAsync(out.pay.p, 0, out.n * out.P * 8, stream));
      A.row_out = out.pay.as<uint64_t>();
      if (out.n)
        launch("cycle_slot_index", [&] {
          k_slot_to_index<<<grid_for(W, 256), 256, 0, stream>>>(A.item_slot, A.ht_idx, W);
        }, W * 12);
      if (out.n)
        launch("cycle_hop_expand", [&] { k_hop_expand<1><<<grid_for(W, kHopTile), kHopTile, 0, stream>>>(A); },
               hop_bytes / 2 + out.n * (8 + 8ull * out.P));
    } else {
      // one pass: rows for at most W keys (each item adds one key at most);
      // ht_idx starts all-ones so finders wait for the inserter's index
      MB_CUDA(cudaMemsetAsync(out.ht_idx.p, 0xFF, cap * 4, stream));
      out.pay.alloc(std::max<uint64_t>(W * out.P, 1) * 8);
      A.row_out = out.pay.as<uint64_t>();
      launch("cycle_hop_expand", [&] { k_hop_expand<2><<<grid_for(W, kHopTile), kHopTile, 0, stream>>>(A); },
             hop_bytes);
      out.n = d2h(nk.as<uint64_t>());
    }
    if (dbg)
      fprintf(stderr, "hop n_in=%llu W=%llu keys=%llu s_in=%d P_in=%u first=%d in_r=%d out_r=%d rec=%d s_out=%d "
              "P_out=%u etab=%p Pe=%u ntab=%p Pn=%u bits=%d\n",
              (unsigned long long)in.n, (unsigned long long)W, (unsigned long long)out.n, in.s, in.P, (int)first,
              in.has_r, out.has_r, (int)record, out.s, out.P, (const void*)A.etab, A.Pe, (const void*)A.ntab, A.Pn,
              bits);
    return true;
  }

  // Relation for the cycle edge e walked from position p to q.
  Relation relation(const CycleDesc& C, int e, bool walk_fwd_of_storage) const {
    Relation r;
    const TabView& t = C.edge[e];
    if (t.kind == 4) {
      r.off = walk_fwd_of_storage ? t.off : t.off_t;
      r.adj = walk_fwd_of_storage ? t.cols : t.cols_t;
      r.pay = walk_fwd_of_storage ? t.data : t.data_t;
      r.size = walk_fwd_of_storage ? t.size : t.size_t_;
      r.rs = t.P;
      r.P = t.P, r.s = t.s;
    } else {
      r.off = G.off, r.adj = G.adj;
      if (t.kind == 3)
        r.pay = t.data, r.P = t.P, r.rs = t.rs, r.s = t.s, r.use_rev = !walk_fwd_of_storage, r.size = t.size;
    }
    return r;
  }

  using Sink = std::function<void(Frontier&)>;

  // Copies entries [i0, i0 + cnt) of a frontier (the slice stays sorted).
  void slice(const Frontier& f, uint64_t i0, uint64_t cnt, Frontier& a) {
    a.s = f.s, a.P = f.P, a.has_r = f.has_r, a.n = cnt, a.ub = f.ub;
    a.key.alloc(std::max<uint64_t>(cnt, 1) * 8), a.pay.alloc(std::max<uint64_t>(cnt * f.P, 1) * 8);
    MB_CUDA(cudaMemcpyAsync(a.key.p, f.key.as<uint64_t>() + i0, cnt * 8, cudaMemcpyDeviceToDevice, stream));
    MB_CUDA(cudaMemcpyAsync(a.pay.p, f.pay.as<uint64_t>() + i0 * f.P, cnt * f.P * 8, cudaMemcpyDeviceToDevice,
                            stream));
  }

  // Walks a half path from position p (frontier cur) to d and hands every
  // finished frontier part to `sink`.  Over the scratch budget, a
  // multi-anchor batch returns false (the caller halves the anchor range; no
  // part has reached the sink then, since parts only arise below).  A
  // single-anchor batch instead splits the frontier into parts that continue
  // separately: hops and the final merge are linear in the frontier, so the
  // parts' contributions add up to the whole (hub anchors of the theta query
  // reach ~10^8 (v, r) keys in one hop).
  bool walk(const CycleDesc& C, Frontier& cur, int p, int d, bool cw, bool end_ann, int rec_pos, bool first,
            const Sink& sink) {
    const int L = C.L;
    const TabView none{};
    while (p != d) {
      const int q = cw ? (p + 1) % L : (p + L - 1) % L;
      const int e = cw ? p : q;  // cycle edge joining p and q
      // child keyed (nodes[e], nodes[e+1]) when edge_fwd; we walk p -> q
      const bool stored_pq = cw ? static_cast<bool>(C.edge_fwd[e]) : !C.edge_fwd[e];
      const Relation rel = relation(C, e, C.edge[e].kind ? stored_pq : true);
      const TabView& nt = (q != d || end_ann) ? C.node[q] : none;
      Frontier nxt;
      if (!hop(cur, nxt, rel, nt.kind ? nt : none, q == rec_pos, first, false)) {
        if (!force) return false;
        if (cur.n > 1) {
          // as many parts as the refused hop needs budgets (plus slack)
          const uint64_t parts = std::min<uint64_t>(cur.n, last_over / mem_budget + 2);
          const uint64_t per = (cur.n + parts - 1) / parts;
          Frontier whole = std::move(cur);
          for (uint64_t i0 = 0; i0 < whole.n; i0 += per) {
            Frontier a;
            slice(whole, i0, std::min(per, whole.n - i0), a);
            if (!walk(C, a, p, d, cw, end_ann, rec_pos, first, sink)) return false;
          }
          return true;
        }
        hop(cur, nxt, rel, nt.kind ? nt : none, q == rec_pos, first, true);  // one entry: no smaller unit
      }
      cur = std::move(nxt);
      first = false;
      p = q;
    }
    sink(cur);
    return true;
  }

  // Vertex sharding of a root block: this rank anchors the
  // device vertices x with x % shard_world == shard_rank.  Device ids follow
  // the degree order, so the cyclic deal gives every rank its share of hubs.
  uint32_t shard_rank = 0, shard_world = 1;

  // Builds the half path from h towards d for the owned anchors in [x0, x0 + nx).
  bool half(const CycleDesc& C, int h, int d, bool cw, bool start_ann, bool end_ann, int rec_pos, uint32_t x0,
            uint32_t nx, const Sink& sink) {
    {
      // first owned anchor at or after x0, and how many owned ones the range holds
      const uint32_t W = shard_world;
      const uint32_t first = x0 + ((shard_rank + W - x0 % W) % W);
      const uint64_t end = static_cast<uint64_t>(x0) + nx;
      nx = first < end ? static_cast<uint32_t>((end - 1 - first) / W + 1) : 0;
      x0 = first;
      if (nx == 0) return true;
    }
    Frontier cur;
    const TabView& hn = C.node[h];
    const bool use_start = start_ann && hn.kind;
    cur.s = use_start ? hn.s : 1;
    cur.P = use_start ? hn.P : 1;
    cur.n = nx;
    cur.has_r = 0;
    cur.ub = use_start ? 1e30L : 1.0L;  // unannotated anchors start with the entry 1
    cur.key.alloc(std::max<uint32_t>(nx, 1) * 8);
    cur.pay.alloc(std::max<uint64_t>(static_cast<uint64_t>(nx) * cur.P, 1) * 8);
    launch("cycle_init", [&] {
      k_init_frontier<<<grid_for(nx, 256), 256, 0, stream>>>(x0, nx, shard_world, bits, G.chi,
                                                             use_start ? hn.data : nullptr,
                                                             cur.P, hn.rs, cur.key.as<uint64_t>(),
                                                             cur.pay.as<uint64_t>());
    });
    return walk(C, cur, h, d, cw, end_ann, rec_pos, true, sink);
  }

  // Joins half-path parts: side A (iterated, may carry r) with side B (looked up by (x, v)).
  void merge(const CycleDesc& C, const Frontier& A, const Frontier& B, int ks0, int ks1) {
    MergeArgs M{};
    M.G = G;
    M.keyA = A.key.as<uint64_t>(), M.payA = A.pay.as<uint64_t>(), M.nA = A.n, M.sA = A.s, M.PA = A.P;
    M.A_has_r = A.has_r;
    M.keyB = B.key.as<uint64_t>(), M.payB = B.pay.as<uint64_t>(), M.nB = B.n, M.sB = B.s, M.PB = B.P;
    if (B.n && !B.ht_key.p) fail(kInternal, "half-path frontier without a hash table");
    M.htB_key = B.ht_key.as<uint64_t>(), M.htB_idx = B.ht_idx.as<uint32_t>();
    M.htB_mask = B.ht_mask, M.htB_shift = B.ht_shift;
    M.bits = bits;
    M.out_kind = C.out.kind == 1 ? 1 : (C.out.kind == 2 ? 2 : (C.out.kind == 3 ? 3 : 4));
    M.key_src0 = ks0, M.key_src1 = ks1;
    M.out = C.out.data, M.Pout = C.out.P, M.rso = C.out.rs;
    M.scalar = scalar, M.err = err, M.updates = upd;
    M.scalar_mult = h_mult;
    M.t_mult = h_mult_t;
    if (M.out_kind == 4) {
      ArenaScope no_arena(nullptr);  // the pair table outlives the anchor batch
      // streaming into the root: a full partial table is consumed first
      if (pair_flush && pairs.n && pairs.n * (C.out.P + 2) * 8ull > pair_flush_bytes) pair_flush();
      reserve_pairs(C.out.P, pairs.n + (h_mult_t ? 2 : 1) * A.n);
      M.ph_key = pairs.key.as<uint64_t>(), M.ph_idx = pairs.idx.as<uint32_t>();
      M.ph_mask = 2 * pairs.cap_rows - 1, M.ph_shift = pairs.shift;
      M.ph_n = reinterpret_cast<unsigned long long*>(pairs.counter.p);
      M.ph_list = pairs.list.as<uint64_t>(), M.ph_rows = pairs.rows.as<uint64_t>();
    }
    launch("cycle_merge", [&] { k_half_merge<<<grid_for(A.n, 256), 256, 0, stream>>>(M); });
    if (M.out_kind == 4) pairs.n = d2h(pairs.counter.as<uint64_t>());
  }

  // Makes room for `need` keys in the running pair table: a larger table is
  // rebuilt from the dense (key, row) list, whose indices stay valid.
  void reserve_pairs(uint32_t P, uint64_t need) {
    if (need <= pairs.cap_rows && pairs.key.p) return;
    uint64_t rows = std::max<uint64_t>(1ull << 16, pairs.cap_rows);
    while (rows < need) rows *= 2;
    if (need > 0xFFFFFFF0ull) fail(kBudget, "pair table exceeds 2^32 keys");
    int lg = 1;
    while ((1ull << lg) < 2 * rows) ++lg;
    PairHash nh;
    nh.cap_rows = rows;
    nh.shift = 64 - lg;
    nh.key.alloc((2 * rows) * 8);
    nh.idx.alloc((2 * rows) * 4);
    nh.list.alloc(rows * 8);
    nh.rows.alloc(rows * P * 8);
    nh.counter.alloc(8);
    MB_CUDA(cudaMemsetAsync(nh.key.p, 0xFF, 2 * rows * 8, stream));
    MB_CUDA(cudaMemsetAsync(nh.idx.p, 0xFF, 2 * rows * 4, stream));
    MB_CUDA(cudaMemsetAsync(nh.rows.p, 0, rows * P * 8, stream));
    nh.n = pairs.n;
    if (pairs.key.p && pairs.n) {
      MB_CUDA(cudaMemcpyAsync(nh.list.p, pairs.list.p, pairs.n * 8, cudaMemcpyDeviceToDevice, stream));
      MB_CUDA(cudaMemcpyAsync(nh.rows.p, pairs.rows.p, pairs.n * P * 8, cudaMemcpyDeviceToDevice, stream));
      launch("pair_rehash", [&] {
        k_pair_rehash<<<grid_for(pairs.n, 256), 256, 0, stream>>>(nh.list.as<uint64_t>(), pairs.n, nh.key.as<uint64_t>(),
                                                                  nh.idx.as<uint32_t>(), 2 * rows - 1, nh.shift);
      });
    }
    MB_CUDA(cudaMemcpyAsync(nh.counter.p, &nh.n, 8, cudaMemcpyHostToDevice, stream));
    MB_CUDA(cudaStreamSynchronize(stream));  // &nh.n is a host stack value
    pairs = std::move(nh);
  }

  // Evaluates position h of Eq. 1 for anchors [x0, x0+nx); false = split and
  // retry (nothing has been accumulated for this (h, batch) yet).
  Arena arena;  // per-batch scratch (reset at every batch)

  bool run_batch(const CycleDesc& C, int h, uint32_t x0, uint32_t nx) {
    arena.top = 0;  // the previous batch's buffers are all dead (stream order keeps reuse safe)
    ArenaScope scope(arena.base ? &arena : nullptr);
    const int L = C.L, nb = static_cast<int>(C.bpos.size());
    int d, rec = -1;
    int ks0 = 0, ks1 = 0;  // output key sources: 0 x, 1 v, 2 r
    if (nb == 0) {
      d = (h + L / 2) % L;
    } else if (nb == 1) {
      if (C.bpos[0] == h) {
        d = (h + L / 2) % L;
        ks0 = 0;
      } else {
        d = C.bpos[0];
        ks0 = 1;
      }
    } else {
      if (h == C.bpos[0]) {
        d = C.bpos[1], ks0 = 0, ks1 = 1;
      } else if (h == C.bpos[1]) {
        d = C.bpos[0], ks0 = 1, ks1 = 0;
      } else {
        d = C.bpos[0], rec = C.bpos[1], ks0 = 1, ks1 = 2;
      }
    }
    bool rec_cw = false;
    for (int p = h; p != d; p = (p + 1) % L)
      if (p == rec) rec_cw = true;
    // plus (clockwise) excludes the start annotation and includes the end (d);
    // minus (counter-clockwise) includes the start and excludes the end.  The
    // side that records r is iterated (A); the other is looked up (B), so B's
    // parts are built first and kept, and A's parts are merged as they come.
    const bool a_is_plus = rec >= 0 && rec_cw;
    std::vector<Frontier> bparts;
    const Sink keep = [&](Frontier& f) {
      if (f.n) bparts.push_back(std::move(f));
    };
    if (a_is_plus) {
      if (!half(C, h, d, false, true, false, -1, x0, nx, keep)) return false;
    } else {
      if (!half(C, h, d, true, false, true, -1, x0, nx, keep)) return false;
    }
    if (bparts.empty()) return true;
    const Sink join = [&](Frontier& a) {
      if (!a.n) return;
      for (const Frontier& b : bparts) merge(C, a, b, ks0, ks1);
    };
    if (a_is_plus) return half(C, h, d, true, false, true, rec, x0, nx, join);
    return half(C, h, d, false, true, false, rec >= 0 ? rec : -1, x0, nx, join);
  }

  // A root cycle with no boundary and no annotation on any node or edge: every
  // rotation maps the labelled matches whose highest vertex sits at position h
  // one-to-one onto those with it at h + 1, so all L terms of Eq. 1 are equal
  // and the h = 0 term times L is exact (configs 0 and 2).
  // A cycle block without annotations whose boundary positions are all fixed
  // by one reflection p -> c2 - p (mod L): one boundary node b (c2 = 2b), or
  // two opposite ones b0, b1 = b0 + L/2 (c2 = 2 b0; the theta's 6-cycle block
  // keyed by (0, 7)).  Returns c2, or -1.
  static int reflection_axis(const CycleDesc& C) {
    for (int q = 0; q < C.L; ++q)
      if (C.node[q].kind || C.edge[q].kind) return -1;
    if (C.bpos.size() == 1) return (2 * C.bpos[0]) % C.L;
    if (C.bpos.size() == 2 && C.L % 2 == 0 && ((C.bpos[1] - C.bpos[0] + C.L) % C.L) == C.L / 2)
      return (2 * C.bpos[0]) % C.L;
    return -1;
  }

  static bool rotation_symmetric(const CycleDesc& C) {
    if (!C.bpos.empty() || C.out.kind != 1) return false;
    for (int q = 0; q < C.L; ++q)
      if (C.node[q].kind || C.edge[q].kind) return false;
    return true;
  }

  void solve(const CycleDesc& C) {
    const uint32_t first_batch = std::max<uint32_t>(1, std::min<uint32_t>(G.n, 1u << 20));
    {
      // per-hop scratch: a quarter of what is free (a hop holds ~4x its rows
      // while it sorts), within [2, 48] GB
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
        // blocks the pool keeps mapped but does not use are available too
        int dev = 0;
        cudaMemPool_t pool;
        uint64_t reserved = 0, used = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        }
        const uint64_t avail = fr + (reserved > used ? reserved - used : 0) + dbuf_cache().cached;
        // a pair-keyed output also holds its pending contributions, the
        // running table and the compaction's sort buffers outside the arena
        const uint64_t div = C.out.kind == 4 ? 8 : 4;
        mem_budget = std::min<uint64_t>(48ull << 30, std::max<uint64_t>(2ull << 30, avail / div));
      }
      static const char* mb_env = std::getenv("MB_CYCLE_BUDGET_MB");
      if (mb_env) mem_budget = std::strtoull(mb_env, nullptr, 10) << 20;
    }
    // the per-batch arena: the per-hop budget (a hop's hash table, keys and
    // rows plus the frontiers and B parts that are still alive; a batch that
    // needs more spills into ordinary pool allocations)
    DBuf arena_mem;
    {
      static const bool no_arena = std::getenv("MB_NO_ARENA") != nullptr;
      ArenaScope off(nullptr);
      if (!no_arena) {
        size_t fr = 0, tot = 0;
        MB_CUDA(cudaMemGetInfo(&fr, &tot));
        // one budget: a batch that needs more spills to pool allocations
        const uint64_t want = std::min<uint64_t>(mem_budget, (static_cast<uint64_t>(fr) + dbuf_cache().cached) / 3);
        if (want >= (64ull << 20)) {
          arena_mem.alloc(want);
          arena.base = arena_mem.as<char>();
          arena.cap = want;
        }
      }
    }
    static const bool no_sym = std::getenv("MB_NO_CYCLE_SYMMETRY") != nullptr;
    // Eq. 1 positions to evaluate, each with the number of equal terms it stands for
    struct HTerm {
      int h;
      uint32_t a, b;  // the orbit's Eq. 1 terms: a x T_h + b x (T_h with its pair keys swapped)
    };
    std::vector<HTerm> hs;
    if (rotation_symmetric(C) && !no_sym) {
      hs.push_back({0, static_cast<uint32_t>(C.L), 0u});
    } else if (int c2 = reflection_axis(C); c2 >= 0 && !no_sym) {
      // a reflection s: p -> c2 - p (mod L) fixes the boundary positions and
      // maps the labelled matches whose highest vertex sits at h one-to-one
      // onto those with it at s(h), keys and colour sets unchanged.  With two
      // opposite boundary nodes and a pair-keyed output, the rotation r by
      // L/2 swaps them: T_r(h) is T_h with its keys swapped.  Each orbit of
      // {1, s, r, rs} is evaluated once (the theta's 6-cycle block: 2 of 6
      // positions).
      const int L = C.L;
      const bool swap_ok = C.bpos.size() == 2 && C.out.kind == 4 && !no_swap_sym();
      std::vector<char> seen(L, 0);
      auto refl = [&](int p) { return ((c2 - p) % L + L) % L; };
      auto rot = [&](int p) { return (p + L / 2) % L; };
      for (int h = 0; h < L; ++h) {
        if (seen[h]) continue;
        const int o1 = refl(h);
        uint32_t a = 1 + (o1 != h), b = 0;
        seen[h] = seen[o1] = 1;
        if (swap_ok) {
          const int o2 = rot(h), o3 = rot(o1);
          if (o2 != h && o2 != o1 && !seen[o2]) ++b, seen[o2] = 1;
          if (o3 != h && o3 != o1 && o3 != o2 && !seen[o3]) ++b, seen[o3] = 1;
        }
        hs.push_back({h, a, b});
      }
    } else {
      for (int h = 0; h < C.L; ++h) hs.push_back({h, 1u, 0u});
    }
    const int nh = static_cast<int>(hs.size());
    // Anchors are swept in device order (hubs first) with an adaptive batch:
    // halved when a hop would exceed the scratch budget (the attempt is
    // discarded), doubled after a success, so heavy anchors run in small
    // batches and the light tail in large ones.
    static const bool dbg = std::getenv("MB_DEBUG_BATCH") != nullptr;
    uint64_t ok = 0, failed = 0;
    const auto t_solve = std::chrono::steady_clock::now();
    wait_s = 0;
    t_dbuf_alloc_s = 0;
    // Per-anchor work estimate: S2[x] = sum of the degrees of x's suffix
    // neighbours bounds the second hop of x's half paths.  A batch is the
    // longest anchor range whose S2 sum times the learned ratio (bytes of the
    // largest hop per unit of S2, from the last batches) fits the budget.
    const std::vector<double>& pre = s2_prefix();
    auto pick = [&](uint32_t x0, double ratio) -> uint32_t {
      if (ratio <= 0) return std::min<uint32_t>(G.n - x0, 1024);
      const double lim = pre[x0] + static_cast<double>(mem_budget) / ratio;
      const uint32_t hi = static_cast<uint32_t>(std::min<uint64_t>(G.n, static_cast<uint64_t>(x0) + first_batch));
      const uint32_t e = static_cast<uint32_t>(std::upper_bound(pre.begin() + x0 + 1, pre.begin() + hi + 1, lim) -
                                               pre.begin()) - 1;
      return std::max<uint32_t>(1, e - x0);
    };
    static const bool old_batches = std::getenv("MB_HALVING_BATCHES") != nullptr;
    for (int hi = 0; hi < nh; ++hi) {
      const int h = hs[hi].h;
      h_mult = hs[hi].a;
      h_mult_t = hs[hi].b;
      uint32_t bs = first_batch, cap = first_batch;  // (MB_HALVING_BATCHES) cap: below the last size that failed
      double ratio = 0;  // 0: unknown yet (a first probe batch of 1024 anchors)
      for (uint32_t x0 = 0; x0 < G.n;) {
        const uint32_t nx = old_batches ? std::min(bs, G.n - x0) : pick(x0, ratio);
        force = nx == 1;
        batch_need = 0;
        const bool done = run_batch(C, h, x0, nx);
        const double s2 = std::max(1.0, pre[x0 + nx] - pre[x0]);
        if (!done) {
          ++failed;
          bs = std::max<uint32_t>(1, nx / 2);
          cap = bs;
          // the refused hop's need, with slack; a range that cannot shrink by
          // estimate any more is halved
          const double r = 1.25 * static_cast<double>(last_over) / s2;
          ratio = std::max(ratio * 2, r);
          if (!old_batches && pick(x0, ratio) >= nx) ratio = static_cast<double>(mem_budget) / std::max(1.0, pre[x0 + std::max<uint32_t>(1, nx / 2)] - pre[x0]);
          continue;
        }
        {
          ++ok;
          // learned ratio: this batch's largest hop per unit of S2 (decaying
          // towards the lighter anchors further along the sweep)
          const double r = 1.25 * static_cast<double>(batch_need) / s2;
          ratio = ratio <= 0 ? r : std::max(r, 0.7 * ratio);
          x0 += nx;
          // fail fast: every contribution is non-negative and the anchors run
          // hubs first, so once a checked add or multiply has overflowed the
          // count is >= 2^64 and the reference's checked arithmetic raises
          // OverflowError as well (errors.hpp:38-50, ProjectionTable::add at
          // table.cpp:38-54): stop here,
          // count() turns the flag into that error
          if (overflowed()) {
            if (dbg) fprintf(stderr, "cycle L=%d: overflow after anchor %u of %u\n", C.L, x0, G.n);
            return;
          }
          // anchors get lighter along the sweep: grow, but only slowly past a failure
          cap = static_cast<uint32_t>(std::min<uint64_t>(first_batch, cap + cap / 4 + 1));
          bs = static_cast<uint32_t>(std::min<uint64_t>(2ull * nx, cap));
        }
      }
    }
    if (dbg) {
      MB_CUDA(cudaStreamSynchronize(stream));
      const double tot = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_solve).count();
      fprintf(stderr, "cycle L=%d: %llu batches, %llu discarded attempts, budget %.1f GB, %.3f s (%.3f s in d2h, "
              "%.3f s in allocation)\n", C.L, (unsigned long long)ok, (unsigned long long)failed, mem_budget / 1e9, tot,
              wait_s, t_dbuf_alloc_s);
    }
  }

  // Concatenates the pair contributions of solve() and aggregates them into a
  // sorted pair table with CSR rows (and the transposed copy).
  void finish_pairs(uint32_t P, DBuf& key, DBuf& pay, uint64_t& nk, DBuf& off, DBuf& cols, DBuf& off_t,
                    DBuf& cols_t, DBuf& pay_t) {
    // the pair table in key order: sort the dense key list, gather the rows
    nk = pairs.n;
    key.alloc(std::max<uint64_t>(nk, 1) * 8);
    pay.alloc(std::max<uint64_t>(nk * P, 1) * 8);
    if (nk) {
      DBuf didx(nk * 4), sidx(nk * 4);
      launch("cycle_iota", [&] { k_iota<uint32_t><<<grid_for(nk, 256), 256, 0, stream>>>(didx.as<uint32_t>(), nk); });
      sort_pairs(pairs.list.as<uint64_t>(), key.as<uint64_t>(), didx.as<uint32_t>(), sidx.as<uint32_t>(), nk, 2 * bits);
      launch("pair_gather", [&] {
        k_gather_rows32<<<grid_for(nk * P, 256), 256, 0, stream>>>(sidx.as<uint32_t>(), pairs.rows.as<uint64_t>(), P, nk,
                                                                   pay.as<uint64_t>());
      });
    }
    {
      static const bool dbg = std::getenv("MB_DEBUG_PAIRS") != nullptr;
      if (dbg) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        fprintf(stderr, "pairs: table of %llu keys (capacity %llu; free %.1f GB, cached %.1f GB)\n",
                (unsigned long long)nk, (unsigned long long)pairs.cap_rows, fr / 1e9, dbuf_cache().cached / 1e9);
      }
    }
    pairs = PairHash{};
    build_csr(key, nk, off, cols);
    // transpose: swap the two keys, sort, gather rows
    DBuf tk(std::max<uint64_t>(nk, 1) * 8), idx(std::max<uint64_t>(nk, 1) * 8), sk(std::max<uint64_t>(nk, 1) * 8),
        sidx(std::max<uint64_t>(nk, 1) * 8);
    pay_t.alloc(std::max<uint64_t>(nk * P, 1) * 8);
    if (nk) {
      launch("pair_swap", [&] { k_swap_pair_keys<<<grid_for(nk, 256), 256, 0, stream>>>(key.as<uint64_t>(), nk, bits, tk.as<uint64_t>()); });
      launch("cycle_iota", [&] { k_iota<uint64_t><<<grid_for(nk, 256), 256, 0, stream>>>(idx.as<uint64_t>(), nk); });
      sort_pairs(tk.as<uint64_t>(), sk.as<uint64_t>(), idx.as<uint64_t>(), sidx.as<uint64_t>(), nk, 2 * bits);
      launch("pair_gather", [&] {
        k_gather_rows<<<grid_for(nk * P, 256), 256, 0, stream>>>(sidx.as<uint64_t>(), pay.as<uint64_t>(), P, nk,
                                                                 pay_t.as<uint64_t>());
      });
    }
    build_csr(sk, nk, off_t, cols_t);
  }

  void build_csr(const DBuf& keys, uint64_t nk, DBuf& off, DBuf& cols) {
    off.alloc((static_cast<uint64_t>(G.n) + 1) * 8);
    cols.alloc(std::max<uint64_t>(nk, 1) * 4);
    launch("pair_csr", [&] {
      k_pair_csr<<<grid_for(std::max<uint64_t>(nk, static_cast<uint64_t>(G.n) + 1), 256), 256, 0, stream>>>(
          G.n, keys.as<uint64_t>(), nk, bits, off.as<uint64_t>(), cols.as<uint32_t>());
    });
  }
};

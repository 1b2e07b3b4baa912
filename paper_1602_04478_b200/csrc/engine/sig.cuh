// Colour-set ("signature") indexing shared by every kernel.
//
// A projection table (reference: table.hpp:36-79, one hash entry per
// (key vertices, signature)) is stored densely on the device: one row per key
// (vertex, or CSR slot for vertex pairs) holding a count for every signature
// of the table's popcount s that contains the key vertices' colours.  The key
// colours are "fixed" and removed from the index, so a row has
//     P = C(k - f, s - f)      (f = number of key vertices)
// entries, addressed by the colex rank of the remaining colours after the
// fixed bit positions are squeezed out.  Colex order of t-subsets coincides
// with increasing bit-mask value, so unranking is a lookup into the list of
// t-bit masks in ascending order, valid for every k' <= kMaxColors at once.
#pragma once

#include <cstdint>

namespace mb {

constexpr int kMaxColors = 16;  // GPU engine limit (reference: 32, paper: <= 10)

struct SigLut {
  const uint16_t* unrank;  // concatenation over t of the t-bit masks < 2^16, ascending
  uint32_t off[kMaxColors + 2];
  uint32_t binom[kMaxColors + 1][kMaxColors + 2];  // binom[c][i] = C(c, i)
};

#ifdef __CUDACC__
#define MB_HD __host__ __device__ __forceinline__
#else
#define MB_HD inline
#endif

MB_HD int mb_clz(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __clz(x);
#else
  return __builtin_clz(x);
#endif
}

MB_HD int mb_ctz(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __ffs(x) - 1;
#else
  return __builtin_ctz(x);
#endif
}

MB_HD int mb_popc(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __popc(x);
#else
  return __builtin_popcount(x);
#endif
}

// Remove the bit positions of `fixed` from m (bits of m at fixed positions are dropped).
MB_HD uint32_t sig_compress(uint32_t m, uint32_t fixed) {
  while (fixed) {
    const int c = 31 - mb_clz(fixed);
    fixed &= ~(1u << c);
    m = (m & ((1u << c) - 1u)) | ((m >> (c + 1)) << c);
  }
  return m;
}

// Inverse of sig_compress, with the fixed bits set.
MB_HD uint32_t sig_expand(uint32_t t, uint32_t fixed) {
  uint32_t f = fixed;
  while (f) {
    const int c = mb_ctz(f);
    f &= f - 1u;
    t = (t & ((1u << c) - 1u)) | ((t >> c) << (c + 1));
  }
  return t | fixed;
}

// Colex rank of a mask among the masks of the same popcount.
MB_HD uint32_t sig_rank(const SigLut& L, uint32_t m) {
  uint32_t r = 0;
  int i = 1;
  while (m) {
    const int c = mb_ctz(m);
    m &= m - 1u;
    r += L.binom[c][i++];
  }
  return r;
}

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t sig_unrank(const SigLut& L, int t, uint32_t r) {
  return __ldg(L.unrank + L.off[t] + r);
}

// Shared-memory copy of the binomial table for kernels whose lanes rank
// different masks at once: indexing __constant__ memory with lane-divergent
// addresses serialises the warp, a shared-memory lookup does not.
constexpr int kBinomStride = kMaxColors + 2;
__device__ __forceinline__ void stage_binom(const SigLut& L, uint32_t* sb) {
  for (int i = threadIdx.x; i < (kMaxColors + 1) * kBinomStride; i += blockDim.x)
    sb[i] = L.binom[i / kBinomStride][i % kBinomStride];
}
__device__ __forceinline__ uint32_t sig_rank_sm(const uint32_t* sb, uint32_t m) {
  uint32_t r = 0;
  int i = 1;
  while (m) {
    const int c = __ffs(m) - 1;
    m &= m - 1u;
    r += sb[c * kBinomStride + i++];
  }
  return r;
}
__device__ __forceinline__ uint32_t sig_index_sm(const uint32_t* sb, uint32_t m, uint32_t fixed) {
  return sig_rank_sm(sb, sig_compress(m & ~fixed, fixed));
}
#endif

// Payload index of the full signature m in a row whose fixed colours are `fixed`.
MB_HD uint32_t sig_index(const SigLut& L, uint32_t m, uint32_t fixed) {
  return sig_rank(L, sig_compress(m & ~fixed, fixed));
}

}  // namespace mb

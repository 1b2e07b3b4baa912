#include "estimate.hpp"

#include "errors.hpp"

namespace mb {

namespace {

// Prefix-pruned permutation search: place node d at an image that keeps
// adjacency with every earlier placement.
void extend_perm(const uint32_t* adjm, int k, int* perm, uint32_t used, int d, uint64_t& count) {
  if (d == k) {
    ++count;
    return;
  }
  for (int img = 0; img < k; ++img) {
    if ((used >> img) & 1u) continue;
    bool ok = true;
    for (int j = 0; j < d && ok; ++j)
      ok = (((adjm[d] >> j) & 1u) == ((adjm[img] >> perm[j]) & 1u));
    if (!ok) continue;
    perm[d] = img;
    extend_perm(adjm, k, perm, used | (1u << img), d + 1, count);
  }
}

}  // namespace

uint64_t automorphism_count(const Query& q) {
  if (q.k > 10) fail(kSpec, "automorphism search supports k <= 10");
  uint32_t adjm[32] = {0};
  for (const auto& e : q.edges) {
    adjm[e.a] |= 1u << e.b;
    adjm[e.b] |= 1u << e.a;
  }
  int perm[32];
  uint64_t count = 0;
  extend_perm(adjm, q.k, perm, 0, 0, count);
  return count;
}

double normalization_factor(int k) {
  if (k < 1 || k > 32) fail(kSpec, "k out of range");
  // k^k/k! = prod_{i=1..k} k/i, kept as a reduced 128-bit fraction while it fits.
  unsigned __int128 num = 1, den = 1;
  auto gcd = [](unsigned __int128 a, unsigned __int128 b) {
    while (b) {
      const unsigned __int128 t = a % b;
      a = b;
      b = t;
    }
    return a;
  };
  for (int i = 1; i <= k; ++i) {
    unsigned __int128 a = static_cast<unsigned>(k), b = static_cast<unsigned>(i);
    const unsigned __int128 g1 = gcd(a, den);
    a /= g1;
    den /= g1;
    const unsigned __int128 g2 = gcd(num, b);
    num /= g2;
    b /= g2;
    if (num > (~static_cast<unsigned __int128>(0)) / a) {
      long double f = 1.0L;
      for (int j = 1; j <= k; ++j) f *= static_cast<long double>(k) / j;
      return static_cast<double>(f);
    }
    num *= a;
    den *= b;
  }
  return static_cast<double>(num) / static_cast<double>(den);
}

double coefficient_of_variation(const std::vector<uint64_t>& c) {
  if (c.size() <= 1) return 0.0;
  long double sum = 0, sq = 0;
  for (uint64_t x : c) {
    sum += static_cast<long double>(x);
    sq += static_cast<long double>(x) * static_cast<long double>(x);
  }
  if (sum == 0) return 0.0;
  const long double n = static_cast<long double>(c.size());
  const long double mean = sum / n;
  return static_cast<double>((sq / n - mean * mean) / mean);
}

}  // namespace mb

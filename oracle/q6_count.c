/*
 * TEST INFRASTRUCTURE ONLY — an independent CPU counter for BASELINE config 1's
 * query, used to pin the full-size (n = 1,000,000) counts the bench prints.
 * Only tests/ and tools/ load it; the product library never does.
 *
 * Query q6 (BASELINE.json configs[1]): edges 0-1, 1-2, 2-0, 1-3, 3-2, 2-4,
 * 4-5 — two triangles sharing the edge 1-2 and the path 2-4-5; k = 6.  A
 * colourful match is an injective image with six distinct colours, counted
 * labelled, as the reference's count_colorful counts them (engine.cpp:265-280;
 * C3 on K3 = 6 in tests/test_engine.cpp).  Derived from the reference's join
 * rules, not from the GPU kernels:
 *   - the two triangles are the common neighbours w0, w3 of the edge a -> b
 *     (images of 1 and 2): edge_join + node_join of table.cpp:135-223;
 *   - the path 2-4-5 hanging at b is the unary table Q[b][{c4, c5}] of
 *     2-paths b-x-y by their colour set: edge_table + to_unary
 *     (table.cpp:103-120, 306-317);
 *   - the disjoint-subset join of the pieces (merge_halves' S1 n S2 = 0 rule,
 *     table.cpp:225-275): with k = 6 every colour is used once, so the path's
 *     colour set is the complement of {chi a, chi b, chi w0, chi w3}.
 *   count = sum over oriented edges (a, b) of
 *           sum over ordered colour pairs (c0 != c3) of R(a, b) = [6] \ {chi a, chi b}:
 *               h_ab[c0] * h_ab[c3] * Q[b][R \ {c0, c3}]
 *   where h_ab[c] = number of common neighbours of a and b with colour c.
 * Common neighbours are listed once per undirected edge from its lower-degree
 * end (marks on the higher end's row), all colourings of a batch at once.
 * Arithmetic is 128-bit; a total >= 2^64 returns -1 (the reference's
 * OverflowError).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* index of the colour pair {a, b} (a != b, both < 6) in 0..14 */
static int pair_index(int a, int b) {
  if (a > b) { int t = a; a = b; b = t; }
  static const int base[6] = {0, 5, 9, 12, 14, 15};
  return base[a] + (b - a - 1);
}

/* chi: ncol colourings, n bytes each, colours 1..6.  out[c]: the count of
 * colouring c.  Returns 0, -1 on overflow, -2 on bad input. */
int or_q6_colorful(uint32_t n, const uint64_t* off, const uint32_t* adj, int ncol, const uint8_t* chi,
                   uint64_t* out) {
  if (ncol < 1) return -2;
  for (uint64_t i = 0; i < (uint64_t)ncol * n; ++i)
    if (chi[i] < 1 || chi[i] > 6) return -2;
  /* Q[c][v][15]: 2-paths v-x-y by colour pair; via N1[c][x][6] = neighbours of x by colour */
  uint32_t* N1 = calloc((size_t)ncol * n * 6, sizeof(uint32_t));
  uint64_t* Q = calloc((size_t)ncol * n * 15, sizeof(uint64_t));
  if (!N1 || !Q) { free(N1); free(Q); return -3; }
  #pragma omp parallel for schedule(dynamic, 1024)
  for (uint32_t x = 0; x < n; ++x)
    for (int c = 0; c < ncol; ++c) {
      const uint8_t* col = chi + (size_t)c * n;
      uint32_t* row = N1 + ((size_t)c * n + x) * 6;
      for (uint64_t e = off[x]; e < off[x + 1]; ++e) row[col[adj[e]] - 1]++;
    }
  #pragma omp parallel for schedule(dynamic, 1024)
  for (uint32_t v = 0; v < n; ++v)
    for (int c = 0; c < ncol; ++c) {
      const uint8_t* col = chi + (size_t)c * n;
      uint64_t* q = Q + ((size_t)c * n + v) * 15;
      for (uint64_t e = off[v]; e < off[v + 1]; ++e) {
        const uint32_t x = adj[e];
        const int cx = col[x] - 1;
        const uint32_t* r = N1 + ((size_t)c * n + x) * 6;
        for (int cy = 0; cy < 6; ++cy)
          if (cy != cx) q[pair_index(cx, cy)] += r[cy];
      }
    }
  int overflow = 0;
  u128* tot = calloc((size_t)ncol, sizeof(u128));
  #pragma omp parallel
  {
    uint32_t* mark = malloc((size_t)n * sizeof(uint32_t)); /* mark[w] = b + 1 when w in N(b) */
    u128* loc = calloc((size_t)ncol, sizeof(u128));
    uint32_t* h = malloc((size_t)ncol * 6 * sizeof(uint32_t));
    for (uint32_t i = 0; i < n; ++i) mark[i] = 0;
    #pragma omp for schedule(dynamic, 64)
    for (uint32_t b = 0; b < n; ++b) {
      const uint64_t db = off[b + 1] - off[b];
      for (uint64_t e = off[b]; e < off[b + 1]; ++e) mark[adj[e]] = b + 1;
      for (uint64_t e = off[b]; e < off[b + 1]; ++e) {
        const uint32_t a = adj[e];
        const uint64_t da = off[a + 1] - off[a];
        /* the undirected edge {a, b} is handled at its higher-(degree, id) end b */
        if (da > db || (da == db && a > b)) continue;
        memset(h, 0, (size_t)ncol * 6 * sizeof(uint32_t));
        int any = 0;
        for (uint64_t f = off[a]; f < off[a + 1]; ++f) {
          const uint32_t w = adj[f];
          if (mark[w] != b + 1) continue;
          any = 1;
          for (int c = 0; c < ncol; ++c) h[c * 6 + chi[(size_t)c * n + w] - 1]++;
        }
        if (!any) continue;
        for (int c = 0; c < ncol; ++c) {
          const uint8_t* col = chi + (size_t)c * n;
          const int ca = col[a] - 1, cb = col[b] - 1;
          if (ca == cb) continue;
          const uint32_t* hc = h + c * 6;
          /* both orientations: the pendant path hangs at the image of node 2 */
          for (int side = 0; side < 2; ++side) {
            const uint32_t at = side ? a : b;
            const uint64_t* q = Q + ((size_t)c * n + at) * 15;
            u128 s = 0;
            for (int c0 = 0; c0 < 6; ++c0) {
              if (c0 == ca || c0 == cb || !hc[c0]) continue;
              for (int c3 = 0; c3 < 6; ++c3) {
                if (c3 == ca || c3 == cb || c3 == c0 || !hc[c3]) continue;
                int p = -1, p2 = -1;
                for (int r = 0; r < 6; ++r)
                  if (r != ca && r != cb && r != c0 && r != c3) { if (p < 0) p = r; else p2 = r; }
                s += (u128)hc[c0] * hc[c3] * q[pair_index(p, p2)];
              }
            }
            loc[c] += s;
          }
        }
      }
    }
    #pragma omp critical
    for (int c = 0; c < ncol; ++c) tot[c] += loc[c];
    free(mark);
    free(loc);
    free(h);
  }
  for (int c = 0; c < ncol; ++c) {
    if (tot[c] >> 64) overflow = 1;
    out[c] = (uint64_t)tot[c];
  }
  free(tot);
  free(N1);
  free(Q);
  return overflow ? -1 : 0;
}

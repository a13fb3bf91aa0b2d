// lap_warp.cuh — warp-per-LAP shortest-augmenting-path Hungarian (sm_100a).
//
// Bit-exact re-design of LapSolver::solve (lap.cpp:24-84) for one warp:
// lane l owns columns j = s*32 + l (s < CPL), including the virtual start
// column m (lap.cpp:21-23).  Per Dijkstra step (lap.cpp:40-67) every lane
// relaxes its columns in parallel; the reference's ascending scan with a
// strict `<` ("first minimum wins", lap.cpp:53) becomes a warp argmin over an
// order-preserving 64-bit key with the lowest column on ties, done with
// `redux.sync` on the key halves (+ ballot / a third redux for the column).
// Every per-element update (lap.cpp:48-65) is order independent, so the
// result — assignment, duals, and the optimum summed in column order
// (lap.cpp:75-80) — is bitwise identical to the serial reference.
//
// Row duals are kept per *column* (w[j] == u[p[j]]): u[i0] for the row that
// just entered the tree is then read from the same lane as p[j1], so a step
// needs one round of shuffles instead of two dependent ones.
#pragma once

#include "common.cuh"

namespace qapb {

// Order-preserving map double -> u64.  x + 0.0 canonicalises -0.0 to +0.0:
// the serial scan's `<` treats them as equal, so they must share a key.
__device__ __forceinline__ unsigned long long ordkey(double x) {
  const long long b = __double_as_longlong(dadd(x, 0.0));
  return (unsigned long long)(b ^ ((b >> 63) | (long long)0x8000000000000000ull));
}

// The same key as two 32-bit halves in three integer ops (one shift, two
// 3-input LOPs): khi = hi ^ (s | 0x80000000), klo = lo ^ s, s = hi >> 31.
__device__ __forceinline__ void ordkey2(double x, unsigned& khi, unsigned& klo) {
  const double c = dadd(x, 0.0);
  asm("{\n\t.reg .b32 lo, hi, s, t;\n\t"
      "mov.b64 {lo, hi}, %2;\n\t"
      "shr.s32 s, hi, 31;\n\t"
      "or.b32 t, s, 0x80000000;\n\t"
      "xor.b32 %0, hi, t;\n\t"
      "xor.b32 %1, lo, s;\n\t}"
      : "=r"(khi), "=r"(klo)
      : "d"(c));
}

template <int CPL>
struct LapLane {
  int p[CPL];     // row matched to column s*32+lane, -1 when free   (lap.cpp:30)
  double w[CPL];  // dual of that row, u[p[j]]                       (lap.cpp:31 uu)
  double v[CPL];  // column dual                                     (lap.cpp:31 vv)
};

// a[s] for a warp-uniform runtime slot s, without spilling `a` to local memory
template <int CPL, class T>
__device__ __forceinline__ T pick(const T (&a)[CPL], int s) {
  T r = a[0];
#pragma unroll
  for (int k = 1; k < CPL; ++k)
    if (s == k) r = a[k];
  return r;
}

// One-column-per-lane form (m <= 31): the hot path of the Z stage at n <= 33.
// Same arithmetic as the generic form; minv of a used column is dead until
// the next row (lap.cpp:36-39 resets it), so it is shifted unconditionally.
__device__ __forceinline__ double warp_lap_solve_1(const double* __restrict__ cost, int m,
                                                   int lane, LapLane<1>& L) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  const bool real = lane < m;
  const double* __restrict__ colp = cost + (real ? lane : m - 1);
  // During the solve L.p holds the matched row's byte offset p*m*8 (-1 when
  // free): the next step's cost address is then one add away.
  L.p[0] = -1;
  L.w[0] = 0.0;
  L.v[0] = 0.0;
  int way = 0;
  // Non-finite (or overflow-prone) costs would let the search run forever
  // (the reference is undefined there too): check the tile once and bail out.
  bool ok = true;
  const int mm = m * m;
  if ((reinterpret_cast<uintptr_t>(cost) & 15) == 0) {  // Z tiles: 16-byte reads
    const double2* __restrict__ c2 = reinterpret_cast<const double2*>(cost);
    for (int e = lane; e < (mm >> 1); e += 32) {
      const double2 x = c2[e];
      ok = ok && (fabs(x.x) <= 1e300) && (fabs(x.y) <= 1e300);
    }
    if ((mm & 1) && lane == 0) ok = ok && (fabs(cost[mm - 1]) <= 1e300);
  } else {
    for (int e = lane; e < mm; e += 32) ok = ok && (fabs(cost[e]) <= 1e300);
  }
  const bool bad = !__all_sync(QAPB_FULL, ok);
  // A used column (and padding lanes, and the virtual column m) carries
  // minv = NaN: `cur < NaN` is false, so it never relaxes, and its order key
  // (0xfff8...) sorts above every finite and +inf key, so it is never the
  // argmin while an unused column remains (lap.cpp:47,58-64).  `used` is
  // therefore just isnan(minv).
  const double QNAN = __longlong_as_double(0x7ff8000000000000ll);
  const bool virt = lane == m;
  const double minv0 = real ? INF : QNAN;
  const int m8 = m * 8;
  int row8 = 0;  // i*m*8
  for (int i = 0; i < m && !bad; ++i, row8 += m8) {  // lap.cpp:33
    double minv = minv0;
    if (virt) {  // p[m] = i; u[i] is still 0
      L.p[0] = row8;
      L.w[0] = 0.0;
    }
    int j0 = m, i0 = row8;
    double ui0 = 0.0;
    while (true) {  // lap.cpp:40-67 (at most m+1 steps: finite costs, checked above)
      if (lane == j0) minv = QNAN;  // column j0 joins the tree
      const double cv = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(colp) + i0);
      const double cur = dsub(dsub(cv, ui0), L.v[0]);  // lap.cpp:48
      if (cur < minv) {                                 // lap.cpp:49-52 (false when used)
        minv = cur;
        way = j0;
      }
      unsigned hi, lo;  // order key of minv (NaN keys last: used / padding lanes)
      ordkey2(minv, hi, lo);
      const unsigned hmin = __reduce_min_sync(QAPB_FULL, hi);
      const unsigned lmin = __reduce_min_sync(QAPB_FULL, hi == hmin ? lo : 0xffffffffu);
      const int j1 = __ffs(__ballot_sync(QAPB_FULL, hi == hmin && lo == lmin)) - 1;
      const double delta = __shfl_sync(QAPB_FULL, minv, j1);
      const bool used = isnan(minv);
      minv = dsub(minv, delta);  // lap.cpp:63 (NaN stays NaN when used)
      // lap.cpp:60-61.  Adding +0.0 on unused columns is exact: u and v start
      // at +0.0 and only ever receive sums/differences that cannot produce
      // -0.0 from a non-negative-zero operand, so x + 0.0 == x bitwise here.
      const double du = used ? delta : 0.0;
      L.w[0] = dadd(L.w[0], du);
      L.v[0] = dsub(L.v[0], du);
      j0 = j1;
      const int pj = __shfl_sync(QAPB_FULL, L.p[0], j1);
      const double wj = __shfl_sync(QAPB_FULL, L.w[0], j1);
      if (pj == -1) break;
      i0 = pj;
      ui0 = wj;
    }
    while (j0 != m) {  // augment, lap.cpp:68-72
      const int jw = __shfl_sync(QAPB_FULL, way, j0);
      const int pw = __shfl_sync(QAPB_FULL, L.p[0], jw);
      const double ww = __shfl_sync(QAPB_FULL, L.w[0], jw);
      if (lane == j0) {
        L.p[0] = pw;
        L.w[0] = ww;
      }
      j0 = jw;
    }
  }
  if (bad) {  // non-finite input: leave a valid permutation for the writers
    L.p[0] = real ? lane : -1;
    L.w[0] = L.v[0] = __longlong_as_double(0x7ff8000000000000ll);
    return L.w[0];
  }
  const int prow = L.p[0] < 0 ? -1 : L.p[0] / (8 * m);  // back to row indices
  L.p[0] = prow;
  const double term = real ? cost[(size_t)prow * m + lane] : 0.0;
  double value = 0.0;  // lap.cpp:75-80
  for (int l = 0; l < m; ++l) value = dadd(value, __shfl_sync(QAPB_FULL, term, l));
  return value;
}

// Solve the m x m LAP whose row-major costs sit in shared memory `cost`.
// All 32 lanes must call it.  Returns the optimum (warp-uniform).
template <int CPL>
__device__ __forceinline__ double warp_lap_solve(const double* __restrict__ cost, int m,
                                                 int lane, LapLane<CPL>& L) {
  if constexpr (CPL == 1) {
    return warp_lap_solve_1(cost, m, lane, L);
  }
  // Same scheme as warp_lap_solve_1 with CPL columns per lane: used and
  // padding columns carry minv = NaN, rows travel as byte offsets, the dual
  // update adds `used ? delta : +0.0` unconditionally.
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  const double QNAN = __longlong_as_double(0x7ff8000000000000ll);
  double minv[CPL];
  int way[CPL];
  const char* colp[CPL];
  double minv0[CPL];
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = s * 32 + lane;
    L.p[s] = -1;
    L.w[s] = 0.0;
    L.v[s] = 0.0;
    way[s] = 0;
    colp[s] = reinterpret_cast<const char*>(cost + (j < m ? j : m - 1));
    minv0[s] = j < m ? INF : QNAN;
  }
  const int vs = m >> 5, vl = m & 31;  // owner of the virtual column m
  bool ok = true;  // finite costs bound every row to m+1 steps (see warp_lap_solve_1)
  for (int e = lane; e < m * m; e += 32) ok = ok && (fabs(cost[e]) <= 1e300);
  if (!__all_sync(QAPB_FULL, ok)) {
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      L.p[s] = (s * 32 + lane < m) ? s * 32 + lane : -1;
      L.w[s] = L.v[s] = QNAN;
    }
    return L.w[0];
  }
  const int m8 = m * 8;
  int row8 = 0;
  for (int i = 0; i < m; ++i, row8 += m8) {  // lap.cpp:33
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      minv[s] = minv0[s];
      if (s == vs && lane == vl) {  // p[m] = i; u[i] is still 0
        L.p[s] = row8;
        L.w[s] = 0.0;
      }
    }
    int j0 = m, i0 = row8;
    double ui0 = 0.0;
    while (true) {  // Dijkstra step, lap.cpp:40-67
      unsigned bhi = 0xffffffffu, blo = 0xffffffffu;
      int bcol = 0x7fffffff;
#pragma unroll
      for (int s = 0; s < CPL; ++s) {
        const int j = s * 32 + lane;
        if (j == j0) minv[s] = QNAN;  // column j0 joins the tree
        const double cv = *reinterpret_cast<const double*>(colp[s] + i0);
        const double cur = dsub(dsub(cv, ui0), L.v[s]);  // lap.cpp:48
        if (cur < minv[s]) {                             // lap.cpp:49-52 (false when used)
          minv[s] = cur;
          way[s] = j0;
        }
        unsigned hi, lo;
        ordkey2(minv[s], hi, lo);
        if (hi < bhi || (hi == bhi && lo < blo)) {  // lowest column of this lane on ties
          bhi = hi;
          blo = lo;
          bcol = j;
        }
      }
      // argmin over unused columns, lowest column on ties (lap.cpp:53-56)
      const unsigned hmin = __reduce_min_sync(QAPB_FULL, bhi);
      const unsigned lmin = __reduce_min_sync(QAPB_FULL, bhi == hmin ? blo : 0xffffffffu);
      const bool cand = (bhi == hmin) && (blo == lmin);
      const int j1 = (int)__reduce_min_sync(QAPB_FULL, cand ? (unsigned)bcol : 0xffffffffu);
      const int s1 = j1 >> 5, l1 = j1 & 31;
      const double delta = __shfl_sync(QAPB_FULL, pick<CPL>(minv, s1), l1);
#pragma unroll
      for (int s = 0; s < CPL; ++s) {  // dual update, lap.cpp:58-65 (see warp_lap_solve_1)
        const double du = isnan(minv[s]) ? delta : 0.0;
        minv[s] = dsub(minv[s], delta);
        L.w[s] = dadd(L.w[s], du);
        L.v[s] = dsub(L.v[s], du);
      }
      j0 = j1;
      const int pj = __shfl_sync(QAPB_FULL, pick<CPL>(L.p, s1), l1);
      const double wj = __shfl_sync(QAPB_FULL, pick<CPL>(L.w, s1), l1);
      if (pj == -1) break;  // lap.cpp:67
      i0 = pj;
      ui0 = wj;
    }
    while (j0 != m) {  // augment, lap.cpp:68-72
      const int s0 = j0 >> 5, l0 = j0 & 31;
      const int jw = __shfl_sync(QAPB_FULL, pick<CPL>(way, s0), l0);
      const int sw = jw >> 5, lw = jw & 31;
      const int pw = __shfl_sync(QAPB_FULL, pick<CPL>(L.p, sw), lw);
      const double ww = __shfl_sync(QAPB_FULL, pick<CPL>(L.w, sw), lw);
      if (lane == l0) {
#pragma unroll
        for (int s = 0; s < CPL; ++s)
          if (s == s0) {
            L.p[s] = pw;
            L.w[s] = ww;
          }
      }
      j0 = jw;
    }
  }
  // back to row indices; value = sum_j cost[p[j]][j] in column order (lap.cpp:75-80)
  double term[CPL];
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = s * 32 + lane;
    L.p[s] = L.p[s] < 0 ? -1 : L.p[s] / m8;
    term[s] = (j < m) ? cost[(size_t)L.p[s] * m + j] : 0.0;
  }
  double value = 0.0;
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int lim = m - s * 32 < 32 ? m - s * 32 : 32;
    for (int l = 0; l < lim; ++l) value = dadd(value, __shfl_sync(QAPB_FULL, term[s], l));
  }
  return value;
}

// pi[a][b] = (cost[a][b] - u[a]) - v[b]   (rlt2.cpp:320-322, :420-422, :439-440)
// `urow` is m doubles of per-warp shared scratch.  `out` may be global.
template <int CPL>
__device__ __forceinline__ void warp_lap_write_slack(const double* __restrict__ cost, int m,
                                                     int lane, const LapLane<CPL>& L,
                                                     double* urow, double* __restrict__ out) {
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = s * 32 + lane;
    if (j < m) urow[L.p[s]] = L.w[s];
  }
  __syncwarp();
  for (int a = 0; a < m; ++a) {
    const double ua = urow[a];
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int b = s * 32 + lane;
      if (b < m) out[(size_t)a * m + b] = dsub(dsub(cost[(size_t)a * m + b], ua), L.v[s]);
    }
  }
  __syncwarp();
}

// row_to_col / col_to_row / u / v outputs of LapSolver::solve (lap.cpp:76-82)
template <int CPL>
__device__ __forceinline__ void warp_lap_write_duals(int m, int lane, const LapLane<CPL>& L,
                                                     int* r2c, int* c2r, double* u, double* v) {
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = s * 32 + lane;
    if (j < m) {
      if (c2r) c2r[j] = L.p[s];
      if (r2c) r2c[L.p[s]] = j;
      if (u) u[L.p[s]] = L.w[s];
      if (v) v[j] = L.v[s];
    }
  }
}

}  // namespace qapb

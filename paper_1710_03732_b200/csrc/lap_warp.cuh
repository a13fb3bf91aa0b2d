// lap_warp.cuh — warp-per-LAP shortest-augmenting-path Hungarian (sm_100a).
//
// Bit-exact re-design of LapSolver::solve (lap.cpp:24-84) for one warp.  Each
// lane owns CPL columns (lap_col below), including the virtual start column m
// (lap.cpp:21-23).  Per Dijkstra step (lap.cpp:40-67) every lane relaxes its
// columns in parallel; the reference's ascending scan with a strict `<`
// ("first minimum wins", lap.cpp:53) becomes a warp argmin over an
// order-preserving 64-bit key with the lowest column on ties, done with
// `redux.sync` on the key halves.  Every per-element update (lap.cpp:48-65) is
// order independent, so the result — assignment, duals, and the optimum summed
// in column order (lap.cpp:75-80) — is bitwise identical to the serial
// reference.
//
// Row duals are kept per *column* (w[j] == u[p[j]]): u[i0] for the row that
// just entered the tree is then read from the same lane as p[j1], so a step
// needs one round of shuffles instead of two dependent ones.
//
// Three solvers share that scheme:
//  * warp_lap_solve_fast1 (m <= 31, the Z stage at n <= 33): lanes own
//    columns in REVERSE order (column 31 - lane), so the lowest tied column is
//    the highest ballot bit and a single FLO finds it; a used column carries
//    minv = NaN (its key sorts last, `cur < NaN` is false); the dual update is
//    three predicated DADDs; the augmenting path is shifted in one parallel
//    shuffle round.
//  * warp_lap_solve_fastN<CPL> (m <= 32*CPL-1): the same with CPL columns per
//    lane (column s*32 + lane) and a third redux for the lowest tied column.
//  * warp_lap_solve_safe<CPL>: explicit used flags and no NaN marking, for
//    tiles whose costs are not all finite with |c| <= 1e300 (the fast solvers'
//    NaN trick needs finite values).  It follows lap.cpp step for step, +inf
//    and huge costs included; where the reference's scan finds no column
//    (lap.cpp:53 never true: j1 = -1 and p[-1] is read — undefined behaviour)
//    it stops and reports the slot as undefined instead.
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
  int p[CPL];     // row matched to column lap_col(s, lane), -1 when free  (lap.cpp:30)
  double w[CPL];  // dual of that row, u[p[j]]                              (lap.cpp:31 uu)
  double v[CPL];  // column dual                                            (lap.cpp:31 vv)
};

// Column owned by slot s of `lane`.  One column per lane: reversed, so the
// lowest column of a tie is the highest set bit of a ballot.
template <int CPL>
__device__ __forceinline__ int lap_col(int s, int lane) {
  return CPL == 1 ? 31 - lane : s * 32 + lane;
}
template <int CPL>
__device__ __forceinline__ int lap_lane_of(int j) {
  return CPL == 1 ? 31 - j : (j & 31);
}

// a[s] for a warp-uniform runtime slot s, without spilling `a` to local memory
template <int CPL, class T>
__device__ __forceinline__ T pick(const T (&a)[CPL], int s) {
  T r = a[0];
#pragma unroll
  for (int k = 1; k < CPL; ++k)
    if (s == k) r = a[k];
  return r;
}

__device__ __forceinline__ double lds_f64(unsigned addr) {
  double x;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(addr));
  return x;
}

// lap.cpp:58-65 for one column: used (minv = NaN) -> u[p[j]] += delta,
// v[j] -= delta; unused -> minv[j] -= delta.  Branch-free: a used column's
// minv stays NaN under the subtraction, and an unused column adds +0.0 to u
// and v, which is exact because u and v never hold -0.0 (they start at +0.0
// and x + (+0.0) = x, x - (+0.0) = x for every other x; a sum or difference
// of non-negative-zero operands is -0.0 only from (-0.0) + (-0.0)).  ptxas
// turns predicated DADDs into compute-and-select, so this form (2 selects,
// 3 DADDs) is the cheaper one.
__device__ __forceinline__ void lap_dual_update(double& minv, double& w, double& v,
                                                double delta) {
  const double du = isnan(minv) ? delta : 0.0;
  minv = dsub(minv, delta);
  w = dadd(w, du);
  v = dsub(v, du);
}

// minv = NaN on the lane that owns column j1 (it joins the tree; lap.cpp:41)
__device__ __forceinline__ void lap_mark_used(double& minv, int lane, int j1lane) {
  asm("{\n\t.reg .pred q;\n\t.reg .b32 lo, hi;\n\t"
      "setp.eq.s32 q, %1, %2;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "@q mov.b32 hi, 0x7ff80000;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "+d"(minv)
      : "r"(lane), "r"(j1lane));
}

// highest set bit (FLO); the mask is never zero here
__device__ __forceinline__ int bfind_u32(unsigned x) {
  int r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

// True (warp-uniform) iff every cost is finite with |c| < 2^997 (~1.3e300):
// the fast solvers then never meet inf/NaN (|u|,|v| stay below 2m * 2^997).
// Which tiles take the safe solver does not change any result -- both do the
// same arithmetic when nothing overflows -- so the test only has to be
// sufficient: an integer max over the high words (sign dropped) of the
// exponent/mantissa, two integer ops per element.
__device__ __forceinline__ bool lap_tile_finite(const double* __restrict__ cost, int m, int lane) {
  constexpr unsigned kLimit = 0x7E400000u;  // high word of 2^997
  unsigned mx = 0;
  const int mm = m * m;
  if ((reinterpret_cast<uintptr_t>(cost) & 15) == 0) {  // Z tiles: 16-byte reads
    const uint4* __restrict__ c4 = reinterpret_cast<const uint4*>(cost);
    for (int e = lane; e < (mm >> 1); e += 32) {
      const uint4 x = c4[e];  // {lo0, hi0, lo1, hi1}
      mx = max(mx, max(x.y & 0x7fffffffu, x.w & 0x7fffffffu));
    }
    if ((mm & 1) && lane == 0)
      mx = max(mx, (unsigned)(__double_as_longlong(cost[mm - 1]) >> 32) & 0x7fffffffu);
  } else {
    for (int e = lane; e < mm; e += 32)
      mx = max(mx, (unsigned)(__double_as_longlong(cost[e]) >> 32) & 0x7fffffffu);
  }
  return __reduce_max_sync(QAPB_FULL, mx) < kLimit;
}

// value = sum_j cost[p[j]][j] in column order from 0.0 (lap.cpp:75-80).
// `term` is lane's cost[p[j]][j] for its column j (< m).  With a 16-byte
// aligned scratch of m doubles the sum runs over shared memory (two terms per
// load); otherwise over shuffles.
template <int CPL>
__device__ __forceinline__ double lap_value(const double (&term)[CPL], int m, int lane,
                                            double* scratch) {
  double value = 0.0;
  if (scratch) {
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int j = lap_col<CPL>(s, lane);
      if (j < m) scratch[j] = term[s];
    }
    __syncwarp();
    int c = 0;
#pragma unroll 4
    for (; c + 1 < m; c += 2) {
      const double2 t = *reinterpret_cast<const double2*>(scratch + c);
      value = dadd(dadd(value, t.x), t.y);
    }
    if (c < m) value = dadd(value, scratch[c]);
    __syncwarp();
    return value;
  }
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int lim = m - s * 32 < 32 ? m - s * 32 : 32;
    for (int l = 0; l < lim; ++l)
      value = dadd(value, __shfl_sync(QAPB_FULL, term[s], lap_lane_of<CPL>(s * 32 + l)));
  }
  return value;
}

// One column per lane (m <= 31), costs in shared memory, all finite.
__device__ __forceinline__ double warp_lap_solve_fast1(const double* __restrict__ cost, int m,
                                                       int lane, LapLane<1>& L,
                                                       double* scratch) {
  const double QNAN = __longlong_as_double(0x7ff8000000000000ll);
  const int col = 31 - lane;
  const bool real = col < m;
  const int vlane = 31 - m;  // owner of the virtual column m
  // shared-memory address of this lane's column in row 0; rows are byte offsets
  const unsigned colbase = smem_u32(cost) + (unsigned)((real ? col : 0) * 8);
  // During the solve L.p holds the matched row's byte offset p*m*8 (-1 when free)
  L.p[0] = -1;
  L.w[0] = 0.0;
  L.v[0] = 0.0;
  int way = vlane;
  const int m8 = m * 8;
  for (int row8 = 0; row8 < m * m8; row8 += m8) {  // lap.cpp:33
    if (lane == vlane) {  // p[m] = i; u[i] is still 0
      L.p[0] = row8;
      L.w[0] = 0.0;
    }
    // First step (j0 = m, u[i] = 0): every real column relaxes, cur - 0.0 is
    // cur bitwise, and cur < +inf holds for finite costs (lap.cpp:48-52).
    double minv = real ? dsub(lds_f64(colbase + row8), L.v[0]) : QNAN;
    way = vlane;
    int j1;
    while (true) {
      unsigned hi, lo;  // order key of minv (NaN keys last: used / padding lanes)
      ordkey2(minv, hi, lo);
      const unsigned hmin = __reduce_min_sync(QAPB_FULL, hi);
      const unsigned lmin = __reduce_min_sync(QAPB_FULL, hi == hmin ? lo : 0xffffffffu);
      j1 = bfind_u32(__ballot_sync(QAPB_FULL, hi == hmin && lo == lmin));  // lap.cpp:53-56
      const double delta = __shfl_sync(QAPB_FULL, minv, j1);
      lap_dual_update(minv, L.w[0], L.v[0], delta);  // lap.cpp:58-65
      lap_mark_used(minv, lane, j1);                 // next step's used[j0]
      const int pj = __shfl_sync(QAPB_FULL, L.p[0], j1);
      const double wj = __shfl_sync(QAPB_FULL, L.w[0], j1);
      if (pj == -1) break;  // lap.cpp:67
      // relax from the row of column j1 (lap.cpp:42-52)
      const double cur = dsub(dsub(lds_f64(colbase + (unsigned)pj), wj), L.v[0]);
      if (cur < minv) {  // false when used (NaN)
        minv = cur;
        way = j1;
      }
    }
    // augment (lap.cpp:68-72): p[j] = p[way[j]] along the path j1 -> ... -> m,
    // all reads before any write, so one parallel shuffle round does it
    bool onpath = false;
    for (int j = j1; j != vlane; j = __shfl_sync(QAPB_FULL, way, j)) onpath |= (lane == j);
    const int pw = __shfl_sync(QAPB_FULL, L.p[0], way);
    const double ww = __shfl_sync(QAPB_FULL, L.w[0], way);
    if (onpath) {
      L.p[0] = pw;
      L.w[0] = ww;
    }
  }
  double term[1];
  term[0] = real ? lds_f64(colbase + (unsigned)L.p[0]) : 0.0;
  L.p[0] = L.p[0] < 0 ? -1 : L.p[0] / m8;  // back to row indices
  return lap_value<1>(term, m, lane, scratch);
}

// CPL columns per lane (column s*32 + lane), costs in shared memory, all finite.
template <int CPL>
__device__ __forceinline__ double warp_lap_solve_fastN(const double* __restrict__ cost, int m,
                                                       int lane, LapLane<CPL>& L,
                                                       double* scratch) {
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
      for (int s = 0; s < CPL; ++s) lap_dual_update(minv[s], L.w[s], L.v[s], delta);
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
  double term[CPL];
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = s * 32 + lane;
    L.p[s] = L.p[s] < 0 ? -1 : L.p[s] / m8;  // back to row indices
    term[s] = (j < m) ? cost[(size_t)L.p[s] * m + j] : 0.0;
  }
  return lap_value<CPL>(term, m, lane, scratch);
}

// lap.cpp:24-84 with explicit used flags (any costs, +inf and huge included).
// Columns follow lap_col<CPL>.  Sets `undefined` (warp-uniform) where the
// reference's scan would find no column.
template <int CPL>
__device__ __forceinline__ double warp_lap_solve_safe(const double* __restrict__ cost, int m,
                                                   int lane, LapLane<CPL>& L, bool& undefined) {
  const double INF = __longlong_as_double(0x7ff0000000000000ll);
  double minv[CPL];
  int way[CPL];
  bool used[CPL];
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    L.p[s] = -1;
    L.w[s] = 0.0;
    L.v[s] = 0.0;
    way[s] = -1;
  }
  undefined = false;
  const int vown = lap_lane_of<CPL>(m), vslot = CPL == 1 ? 0 : (m >> 5);
  for (int i = 0; i < m && !undefined; ++i) {  // lap.cpp:33
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      minv[s] = INF;
      used[s] = false;
      if (s == vslot && lane == vown) {  // p[m] = i
        L.p[s] = i;
        L.w[s] = 0.0;
      }
    }
    int j0 = m;
    while (true) {
      const int o0 = lap_lane_of<CPL>(j0), s0 = CPL == 1 ? 0 : (j0 >> 5);
#pragma unroll
      for (int s = 0; s < CPL; ++s)
        if (s == s0 && lane == o0) used[s] = true;  // lap.cpp:41
      const int i0 = __shfl_sync(QAPB_FULL, pick<CPL>(L.p, s0), o0);
      const double ui0 = __shfl_sync(QAPB_FULL, pick<CPL>(L.w, s0), o0);
      unsigned bhi = 0xffffffffu, blo = 0xffffffffu;
      int bcol = 0x7fffffff;
#pragma unroll
      for (int s = 0; s < CPL; ++s) {
        const int j = lap_col<CPL>(s, lane);
        if (j >= m || used[s]) continue;
        const double cur = dsub(dsub(cost[(size_t)i0 * m + j], ui0), L.v[s]);  // lap.cpp:48
        if (cur < minv[s]) {
          minv[s] = cur;
          way[s] = j0;
        }
        if (minv[s] < INF) {  // a candidate of `minv[j] < delta` (delta starts at +inf)
          unsigned hi, lo;
          ordkey2(minv[s], hi, lo);
          if (hi < bhi || (hi == bhi && lo < blo) || (hi == bhi && lo == blo && j < bcol)) {
            bhi = hi;
            blo = lo;
            bcol = j;
          }
        }
      }
      const unsigned hmin = __reduce_min_sync(QAPB_FULL, bhi);
      const unsigned lmin = __reduce_min_sync(QAPB_FULL, bhi == hmin ? blo : 0xffffffffu);
      const bool cand = (bhi == hmin) && (blo == lmin) && bcol != 0x7fffffff;
      const unsigned jm = __reduce_min_sync(QAPB_FULL, cand ? (unsigned)bcol : 0xffffffffu);
      if (jm == 0xffffffffu) {  // j1 = -1 in lap.cpp:53: undefined there
        undefined = true;
        break;
      }
      const int j1 = (int)jm;
      const int o1 = lap_lane_of<CPL>(j1), s1 = CPL == 1 ? 0 : (j1 >> 5);
      const double delta = __shfl_sync(QAPB_FULL, pick<CPL>(minv, s1), o1);
#pragma unroll
      for (int s = 0; s < CPL; ++s) {  // lap.cpp:58-65 (columns 0..m)
        const int j = lap_col<CPL>(s, lane);
        if (j > m) continue;
        if (used[s]) {
          L.w[s] = dadd(L.w[s], delta);
          L.v[s] = dsub(L.v[s], delta);
        } else {
          minv[s] = dsub(minv[s], delta);
        }
      }
      j0 = j1;
      const int pj = __shfl_sync(QAPB_FULL, pick<CPL>(L.p, s1), o1);
      if (pj == -1) break;  // lap.cpp:67
    }
    if (undefined) break;
    while (j0 != m) {  // augment, lap.cpp:68-72
      const int o0 = lap_lane_of<CPL>(j0), s0 = CPL == 1 ? 0 : (j0 >> 5);
      const int jw = __shfl_sync(QAPB_FULL, pick<CPL>(way, s0), o0);
      const int ow = lap_lane_of<CPL>(jw), sw = CPL == 1 ? 0 : (jw >> 5);
      const int pw = __shfl_sync(QAPB_FULL, pick<CPL>(L.p, sw), ow);
      const double ww = __shfl_sync(QAPB_FULL, pick<CPL>(L.w, sw), ow);
      if (lane == o0) {
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
  double term[CPL];
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = lap_col<CPL>(s, lane);
    if (undefined && j < m) L.p[s] = j;  // a valid permutation for the writers
    term[s] = (j < m) ? cost[(size_t)L.p[s] * m + j] : 0.0;
  }
  return lap_value<CPL>(term, m, lane, nullptr);
}

// Solve the m x m LAP whose row-major costs sit in shared memory `cost`.
// All 32 lanes must call it.  Returns the optimum (warp-uniform).  `scratch`
// (optional): 16-byte aligned shared memory for m doubles.  `undefined`
// (optional) is set when the reference's behaviour is undefined (see top).
template <int CPL>
__device__ __forceinline__ double warp_lap_solve(const double* __restrict__ cost, int m,
                                                 int lane, LapLane<CPL>& L,
                                                 double* scratch = nullptr,
                                                 bool* undefined = nullptr) {
  if (!lap_tile_finite(cost, m, lane)) {
    bool und = false;
    const double v = warp_lap_solve_safe<CPL>(cost, m, lane, L, und);
    if (undefined) *undefined = und;
    return v;
  }
  if (undefined) *undefined = false;
  if constexpr (CPL == 1)
    return warp_lap_solve_fast1(cost, m, lane, L, scratch);
  else
    return warp_lap_solve_fastN<CPL>(cost, m, lane, L, scratch);
}

// pi[a][b] = (cost[a][b] - u[a]) - v[b]   (rlt2.cpp:320-322, :420-422, :439-440)
// `urow` is m doubles of per-warp shared scratch.  `out` may be global.
template <int CPL>
__device__ __forceinline__ void warp_lap_write_slack(const double* __restrict__ cost, int m,
                                                     int lane, const LapLane<CPL>& L,
                                                     double* urow, double* __restrict__ out) {
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = lap_col<CPL>(s, lane);
    if (j < m) urow[L.p[s]] = L.w[s];
  }
  __syncwarp();
  for (int a = 0; a < m; ++a) {
    const double ua = urow[a];
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
      const int b = lap_col<CPL>(s, lane);
      if (b < m) out[(size_t)a * m + b] = dsub(dsub(cost[(size_t)a * m + b], ua), L.v[s]);
    }
  }
  __syncwarp();
}

// The slack in place: cost[a][b] <- (cost[a][b] - u[a]) - v[b] over the whole
// tile in shared memory, element-parallel (two per lane and load when m is
// even).  urow / vrow: m doubles of shared scratch each, vrow 16-byte aligned.
template <int CPL>
__device__ __forceinline__ void warp_lap_slack_inplace(double* __restrict__ cost, int m, int lane,
                                                       const LapLane<CPL>& L, double* urow,
                                                       double* vrow) {
#pragma unroll
  for (int s = 0; s < CPL; ++s) {
    const int j = lap_col<CPL>(s, lane);
    if (j < m) {
      urow[L.p[s]] = L.w[s];
      vrow[j] = L.v[s];
    }
  }
  __syncwarp();
  const int esz = m * m;
  if ((m & 1) == 0 && m <= 64 && (reinterpret_cast<uintptr_t>(cost) & 15) == 0) {
    // lane -> (column pair cp, row phase g): it walks rows g, g + G, ... of
    // columns 2cp, 2cp+1, so the two column duals stay in registers
    const int pairs = m >> 1, G = small_udiv(32, pairs), g = small_udiv(lane, pairs),
              cp = lane - g * pairs;
    if (g < G) {
      const double2 vb = *reinterpret_cast<const double2*>(vrow + 2 * cp);
      double* c2 = cost + (size_t)g * m + 2 * cp;
      const double* ur = urow + g;
      for (int a = g; a < m; a += G, c2 += G * m, ur += G) {
        double2 c = *reinterpret_cast<double2*>(c2);
        const double ua = *ur;
        c.x = dsub(dsub(c.x, ua), vb.x);
        c.y = dsub(dsub(c.y, ua), vb.y);
        *reinterpret_cast<double2*>(c2) = c;
      }
    }
  } else {
    int a = lane / m, b = lane - a * m;  // element lane + 32k
    const int da = 32 / m, db = 32 - da * m;
    for (int e = lane; e < esz; e += 32) {
      cost[e] = dsub(dsub(cost[e], urow[a]), vrow[b]);
      a += da;
      b += db;
      if (b >= m) {
        b -= m;
        ++a;
      }
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
    const int j = lap_col<CPL>(s, lane);
    if (j < m) {
      if (c2r) c2r[j] = L.p[s];
      if (r2c) r2c[L.p[s]] = j;
      if (u) u[L.p[s]] = L.w[s];
      if (v) v[j] = L.v[s];
    }
  }
}

}  // namespace qapb

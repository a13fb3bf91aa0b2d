/*
 * oracle/rlt2_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference RLT2 dual-ascent path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg load it, and only
 * as the checker.  Every function cites the reference line it restates
 * (paths relative to /root/reference/proj).  Arithmetic is written in the
 * reference's evaluation order and compiled with -ffp-contract=off, so
 * results are bitwise identical to the reference's (SSE2 scalar, no FMA).
 * Parity is pinned against golden vectors produced by the compiled
 * reference (tests/golden/) — see tests/test_oracle.py.
 */
#include "rlt2_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int set_err(int code, const char* msg) {
  strncpy(g_err, msg, sizeof g_err - 1);
  return code;
}

/* ---------------- mt19937_64 + libstdc++ uniform_real_distribution ------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* std::uniform_real_distribution<double>(0,1) over mt19937_64 in libstdc++:
 * generate_canonical<double,53> (bits/random.tcc:3349-3381, one draw since
 * log2(range) = 64) then (u * (b - a)) + a. */
static double mt64_uniform01(mt64* g) {
  double sum = (double)mt64_next(g) * 1.0;
  double tmp = 18446744073709551616.0; /* 2^64 */
  double ret = sum / tmp;
  if (ret >= 1.0) ret = nextafter(1.0, 0.0);
  return (ret * (1.0 - 0.0)) + 0.0;
}

/* ---------------- instance generator, src/instance.cpp:131-150 ---------- */
int orc_generate_instance(int n, uint64_t seed, int max_entry, double* flow,
                          double* dist) {
  if (n < 2) return set_err(QAPB_EINVAL, "n must be >= 2");
  mt64 g;
  mt64_seed(&g, seed);
  memset(flow, 0, sizeof(double) * n * n);
  memset(dist, 0, sizeof(double) * n * n);
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      flow[i * n + j] = flow[j * n + i] =
          (double)(mt64_next(&g) % (uint64_t)(max_entry + 1));
  for (int p = 0; p < n; ++p)
    for (int q = p + 1; q < n; ++q)
      dist[p * n + q] = dist[q * n + p] =
          (double)(mt64_next(&g) % (uint64_t)(max_entry + 1));
  return 0;
}

/* ---------------- Hungarian LAP, src/lap.cpp:24-84 ---------------------- */
double orc_lap_solve(const double* cost, int m, int* r2c, int* c2r, double* u,
                     double* v) {
  const double INF = INFINITY;
  double* minv = malloc(sizeof(double) * (m + 1));
  double* uu = calloc(m, sizeof(double));
  double* vv = calloc(m + 1, sizeof(double));
  int* way = malloc(sizeof(int) * (m + 1));
  int* used = malloc(sizeof(int) * (m + 1));
  int* p = malloc(sizeof(int) * (m + 1));
  for (int j = 0; j <= m; ++j) p[j] = -1;
  for (int i = 0; i < m; ++i) { /* lap.cpp:33 */
    p[m] = i;
    int j0 = m;
    for (int j = 0; j <= m; ++j) {
      minv[j] = INF;
      used[j] = 0;
    }
    do { /* Dijkstra step, lap.cpp:40-67 */
      used[j0] = 1;
      const int i0 = p[j0];
      const double* row = cost + (size_t)i0 * m;
      int j1 = -1;
      double delta = INF;
      for (int j = 0; j < m; ++j) {
        if (used[j]) continue;
        const double cur = row[j] - uu[i0] - vv[j];
        if (cur < minv[j]) {
          minv[j] = cur;
          way[j] = j0;
        }
        if (minv[j] < delta) {
          delta = minv[j];
          j1 = j;
        }
      }
      for (int j = 0; j <= m; ++j) { /* lap.cpp:58-65 */
        if (used[j]) {
          uu[p[j]] += delta;
          vv[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      }
      j0 = j1;
    } while (p[j0] != -1);
    do { /* augment, lap.cpp:68-72 */
      const int j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    } while (j0 != m);
  }
  double value = 0; /* lap.cpp:75-80 */
  for (int j = 0; j < m; ++j) {
    if (c2r) c2r[j] = p[j];
    if (r2c) r2c[p[j]] = j;
    value += cost[(size_t)p[j] * m + j];
  }
  if (u) memcpy(u, uu, sizeof(double) * m);
  if (v) memcpy(v, vv, sizeof(double) * m);
  free(minv); free(uu); free(vv); free(way); free(used); free(p);
  return value;
}

/* ---------------- StoreIndex, include/qap/rlt2.hpp:25-69 ----------------- */
typedef struct {
  int m, fpairs, lpairs, tiles, esz;
  int *fp_i, *fp_j, *lp_p, *lp_q;
} sidx;

static inline int ix_fpair(const sidx* x, int i, int j) {
  return i * x->m - i * (i + 1) / 2 + (j - i - 1);
}
static inline int ix_lpair(const sidx* x, int p, int q) {
  return p * (x->m - 1) + q - (q > p);
}
static inline int ix_tile(const sidx* x, int i, int j, int p, int q) {
  return ix_fpair(x, i, j) * x->lpairs + ix_lpair(x, p, q);
}
static inline int ix_cell(const sidx* x, int i, int j, int p, int q, int k,
                          int r) {
  const int kl = k - (k > i) - (k > j);
  const int lo = p < q ? p : q, hi = p < q ? q : p;
  const int rl = r - (r > lo) - (r > hi);
  return kl * (x->m - 2) + rl;
}
static inline void ix_uncell(const sidx* x, int i, int j, int p, int q, int c,
                             int* k, int* r) {
  int kk = c / (x->m - 2), rr = c % (x->m - 2);
  if (kk >= i) ++kk;
  if (kk >= j) ++kk;
  const int lo = p < q ? p : q, hi = p < q ? q : p;
  if (rr >= lo) ++rr;
  if (rr >= hi) ++rr;
  *k = kk;
  *r = rr;
}
static inline size_t ix_cidx(const sidx* x, int i, int p, int j, int q) {
  const int m = x->m;
  return ((size_t)i * m + p) * (m - 1) * (m - 1) +
         (size_t)(j - (j > i)) * (m - 1) + (q - (q > p));
}

static void sidx_init(sidx* x, int m) { /* src/rlt2.cpp:44-64 */
  x->m = m;
  x->fpairs = m * (m - 1) / 2;
  x->lpairs = m * (m - 1);
  x->tiles = x->fpairs * x->lpairs;
  x->esz = (m - 2) * (m - 2);
  x->fp_i = malloc(sizeof(int) * (x->fpairs + 1));
  x->fp_j = malloc(sizeof(int) * (x->fpairs + 1));
  x->lp_p = malloc(sizeof(int) * (x->lpairs + 1));
  x->lp_q = malloc(sizeof(int) * (x->lpairs + 1));
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) {
      x->fp_i[ix_fpair(x, i, j)] = i;
      x->fp_j[ix_fpair(x, i, j)] = j;
    }
  for (int p = 0; p < m; ++p)
    for (int q = 0; q < m; ++q)
      if (p != q) {
        x->lp_p[ix_lpair(x, p, q)] = p;
        x->lp_q[ix_lpair(x, p, q)] = q;
      }
}
static void sidx_free(sidx* x) {
  free(x->fp_i); free(x->fp_j); free(x->lp_p); free(x->lp_q);
}

/* ---------------- init_coefficients, src/rlt2.cpp:66-89 ----------------- */
int orc_init_coefficients(int n, const double* flow, const double* dist,
                          const double* linear, double* b, double* c,
                          double* d) {
  if (n < 3)
    return set_err(QAPB_EINVAL, "init_coefficients: n >= 3 required by RLT2");
  const int m = n;
  sidx x;
  sidx_init(&x, m);
  for (int i = 0; i < m; ++i)
    for (int p = 0; p < m; ++p)
      b[i * m + p] = (linear ? linear[i * n + p] : 0.0) +
                     flow[i * n + i] * dist[p * n + p];
  memset(c, 0, sizeof(double) * (size_t)m * m * (m - 1) * (m - 1));
  for (int i = 0; i < m; ++i)
    for (int p = 0; p < m; ++p)
      for (int j = 0; j < m; ++j) {
        if (j == i) continue;
        for (int q = 0; q < m; ++q) {
          if (q == p) continue;
          c[ix_cidx(&x, i, p, j, q)] = flow[i * n + j] * dist[p * n + q];
        }
      }
  if (d) memset(d, 0, sizeof(double) * (size_t)x.tiles * x.esz);
  sidx_free(&x);
  return 0;
}

/* ---------------- redistribute_family, src/rlt2.cpp:184-205 ------------- */
int orc_redistribute_family(const double pi[3], double add[3],
                            int virtual_slots, double tol) {
  int nb = virtual_slots;
  double total = 0;
  for (int s = 0; s < 3; ++s) {
    if (pi[s] > tol)
      total += pi[s];
    else
      ++nb;
  }
  if (total <= 0) {
    add[0] = add[1] = add[2] = 0;
    return 1;
  }
  if (nb == 0) {
    add[0] = add[1] = add[2] = 0;
    return 0;
  }
  const double share = total / nb;
  for (int s = 0; s < 3; ++s) add[s] = (pi[s] > tol) ? -pi[s] : share;
  return 1;
}

/* ---------------- AscentEngine, src/rlt2.cpp:207-588 -------------------- */
struct orc_engine {
  int m;
  sidx ix;
  qapb_config cfg;
  double *b, *c, *d;
  double offset;
  size_t nb, nc, nd;
  int iter;
  double best, running, last_bound;
  double *theta, *delta, *piz, *piy, *pix, *ybar, *dx, *push, *incz, *ycost,
      *xcost;
  int *xrow, *xcol, *cert;
  int has_cert;
  double cert_val;
  mt64 rng;
  double temp;
  double *sa_fac, *sa_loc;
  qapb_record rec;
};

static int is_fast(const orc_engine* e) {
  return e->cfg.variant == QAPB_F1 || e->cfg.variant == QAPB_F2;
}
static int is_two_phase(const orc_engine* e) {
  return e->cfg.variant == QAPB_F2 || e->cfg.variant == QAPB_S2;
}

int orc_engine_create(int m, const double* b, const double* c, const double* d,
                      double offset, const qapb_config* cfg, orc_engine** out) {
  if (m < 3) return set_err(QAPB_EINVAL, "AscentEngine: m >= 3 required");
  orc_engine* e = calloc(1, sizeof *e);
  e->m = m;
  sidx_init(&e->ix, m);
  e->cfg = *cfg;
  e->nb = (size_t)m * m;
  e->nc = (size_t)m * m * (m - 1) * (m - 1);
  e->nd = (size_t)e->ix.tiles * e->ix.esz;
  e->b = malloc(sizeof(double) * e->nb);
  e->c = malloc(sizeof(double) * e->nc);
  e->d = calloc(e->nd, sizeof(double));
  memcpy(e->b, b, sizeof(double) * e->nb);
  memcpy(e->c, c, sizeof(double) * e->nc);
  if (d) memcpy(e->d, d, sizeof(double) * e->nd);
  e->offset = offset;
  e->best = -INFINITY;
  e->theta = calloc(e->ix.tiles, sizeof(double));
  e->delta = calloc(e->nb, sizeof(double));
  e->piz = calloc(e->nd, sizeof(double));
  e->piy = calloc(e->nc, sizeof(double));
  e->pix = calloc(e->nb, sizeof(double));
  e->ybar = calloc(e->ix.tiles, sizeof(double));
  e->dx = calloc(e->nb, sizeof(double));
  e->push = calloc(e->ix.tiles, sizeof(double));
  e->incz = is_fast(e) ? calloc(e->nd, sizeof(double)) : NULL;
  e->ycost = calloc(e->nc, sizeof(double));
  e->xcost = calloc(e->nb, sizeof(double));
  e->xrow = malloc(sizeof(int) * m);
  e->xcol = malloc(sizeof(int) * m);
  e->cert = malloc(sizeof(int) * m);
  for (int i = 0; i < m; ++i) e->xrow[i] = e->xcol[i] = -1;
  mt64_seed(&e->rng, cfg->seed);
  e->sa_fac = calloc(m, sizeof(double));
  e->sa_loc = calloc(m, sizeof(double));
  *out = e;
  return 0;
}

void orc_engine_destroy(orc_engine* e) {
  if (!e) return;
  free(e->b); free(e->c); free(e->d); free(e->theta); free(e->delta);
  free(e->piz); free(e->piy); free(e->pix); free(e->ybar); free(e->dx);
  free(e->push); free(e->incz); free(e->ycost); free(e->xcost);
  free(e->xrow); free(e->xcol); free(e->cert); free(e->sa_fac); free(e->sa_loc);
  sidx_free(&e->ix);
  free(e);
}

/* ascent_update, src/rlt2.cpp:237-299 */
static void ascent_update(orc_engine* e) {
  const sidx* ix = &e->ix;
  const int m = e->m;
  const double kz = e->cfg.kappa_z_upper, ky = e->cfg.kappa_y,
               kx = e->cfg.kappa_x;
  const double phi = e->cfg.phi_split, vph = e->cfg.varphi;
  for (int i = 0; i < m; ++i) /* x level, :244-249 */
    for (int p = 0; p < m; ++p) {
      const size_t ip = (size_t)i * m + p;
      e->dx[ip] = kx * e->pix[ip] + e->sa_fac[i] + e->sa_loc[p];
      e->b[ip] -= kx * e->pix[ip];
    }
  for (int t = 0; t < ix->tiles; ++t) { /* y level, :253-262 */
    const int i = ix->fp_i[t / ix->lpairs], j = ix->fp_j[t / ix->lpairs];
    const int p = ix->lp_p[t % ix->lpairs], q = ix->lp_q[t % ix->lpairs];
    const double up = e->piy[ix_cidx(ix, i, p, j, q)];
    const double lo = e->piy[ix_cidx(ix, j, q, i, p)];
    e->ybar[t] = 0.5 * (up + lo);
    e->c[ix_cidx(ix, i, p, j, q)] += vph * (lo - up) - ky * e->ybar[t];
    e->c[ix_cidx(ix, j, q, i, p)] +=
        vph * (up - lo) + e->dx[(size_t)j * m + q] / (m - 1);
    e->push[t] = (ky * e->ybar[t] + e->dx[(size_t)i * m + p] / (m - 1)) / (m - 2);
  }
  const int fast = is_fast(e);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < ix->tiles; ++t) { /* z level, :269-295 */
    const int i = ix->fp_i[t / ix->lpairs], j = ix->fp_j[t / ix->lpairs];
    const int p = ix->lp_p[t % ix->lpairs], q = ix->lp_q[t % ix->lpairs];
    double* dt = e->d + (size_t)t * ix->esz;
    double* it = fast ? e->incz + (size_t)t * ix->esz : NULL;
    const double* zt = e->piz + (size_t)t * ix->esz;
    for (int c = 0; c < ix->esz; ++c) {
      int k, r;
      ix_uncell(ix, i, j, p, q, c, &k, &r);
      int bf1, bf2, bl1, bl2;
      if (k > i) { bf1 = i; bf2 = k; bl1 = p; bl2 = r; }
      else       { bf1 = k; bf2 = i; bl1 = r; bl2 = p; }
      const int tB = ix_tile(ix, bf1, bf2, bl1, bl2);
      const int cB = ix_cell(ix, bf1, bf2, bl1, bl2, j, q);
      int cf1, cf2, cl1, cl2;
      if (k > j) { cf1 = j; cf2 = k; cl1 = q; cl2 = r; }
      else       { cf1 = k; cf2 = j; cl1 = r; cl2 = q; }
      const int tC = ix_tile(ix, cf1, cf2, cl1, cl2);
      const int cC = ix_cell(ix, cf1, cf2, cl1, cl2, i, p);
      const double sigB = kz * e->piz[(size_t)tB * ix->esz + cB] + e->push[tB];
      const double sigC = kz * e->piz[(size_t)tC * ix->esz + cC] + e->push[tC];
      const double gain = phi * sigB + phi * sigC;
      dt[c] += gain - kz * zt[c];
      if (fast) it[c] = (1.0 - kz) * zt[c] + gain;
    }
  }
  memset(e->sa_fac, 0, sizeof(double) * m);
  memset(e->sa_loc, 0, sizeof(double) * m);
}

/* solve_all lambda, src/rlt2.cpp:308-325 */
static void z_solve_all(orc_engine* e, const double* costs) {
  const sidx* ix = &e->ix;
  const int md = e->m - 2;
#pragma omp parallel
  {
    double* zu = malloc(sizeof(double) * md);
    double* zv = malloc(sizeof(double) * md);
#pragma omp for schedule(static)
    for (int t = 0; t < ix->tiles; ++t) {
      const double* tc = costs + (size_t)t * ix->esz;
      e->theta[t] = orc_lap_solve(tc, md, NULL, NULL, zu, zv);
      double* tz = e->piz + (size_t)t * ix->esz;
      for (int a = 0; a < md; ++a)
        for (int b = 0; b < md; ++b)
          tz[a * md + b] = tc[a * md + b] - zu[a] - zv[b];
    }
    free(zu);
    free(zv);
  }
}

/* stage_z_second_phase, src/rlt2.cpp:344-381 */
static void z_second_phase(orc_engine* e, double* costs) {
  const sidx* ix = &e->ix;
#pragma omp parallel for schedule(static)
  for (int t = 0; t < ix->tiles; ++t) {
    const int i = ix->fp_i[t / ix->lpairs], j = ix->fp_j[t / ix->lpairs];
    const int p = ix->lp_p[t % ix->lpairs], q = ix->lp_q[t % ix->lpairs];
    for (int c = 0; c < ix->esz; ++c) {
      int k, r;
      ix_uncell(ix, i, j, p, q, c, &k, &r);
      if (k < j) continue;
      const int tB = ix_tile(ix, i, k, p, r), cB = ix_cell(ix, i, k, p, r, j, q);
      const int tC = ix_tile(ix, j, k, q, r), cC = ix_cell(ix, j, k, q, r, i, p);
      const size_t iA = (size_t)t * ix->esz + c;
      const size_t iB = (size_t)tB * ix->esz + cB;
      const size_t iC = (size_t)tC * ix->esz + cC;
      const double pi[3] = {e->piz[iA], e->piz[iB], e->piz[iC]};
      double add[3];
      orc_redistribute_family(pi, add, 3, 1e-9);
      double total = 0;
      int nb = 3;
      for (int s = 0; s < 3; ++s)
        if (pi[s] > 1e-9)
          total += pi[s];
        else
          ++nb;
      const double share = total / nb;
      costs[iA] += add[0] + share;
      costs[iB] += add[1] + share;
      costs[iC] += add[2] + share;
    }
  }
}

/* stage_z, src/rlt2.cpp:301-338 */
static int stage_z(orc_engine* e) {
  double* costs = (is_fast(e) && e->iter > 0) ? e->incz : e->d;
  z_solve_all(e, costs);
  if (is_two_phase(e)) {
    double* th1 = malloc(sizeof(double) * e->ix.tiles);
    memcpy(th1, e->theta, sizeof(double) * e->ix.tiles);
    z_second_phase(e, costs);
    z_solve_all(e, costs);
    for (int t = 0; t < e->ix.tiles; ++t)
      if (e->theta[t] < th1[t] - 1e-7) {
        free(th1);
        return set_err(QAPB_ELOGIC, "phase-2 theta regressed");
      }
    free(th1);
  }
  return 0;
}

/* stage_y, src/rlt2.cpp:383-426 */
static void stage_y(orc_engine* e) {
  const sidx* ix = &e->ix;
  const int m = e->m, my = m - 1;
  const int inc = is_fast(e) && e->iter > 0;
  for (int ipf = 0; ipf < m * m; ++ipf) {
    const int i = ipf / m, p = ipf % m;
    for (int j = 0; j < m; ++j) {
      if (j == i) continue;
      for (int q = 0; q < m; ++q) {
        if (q == p) continue;
        const size_t cix = ix_cidx(ix, i, p, j, q);
        const int t = (i < j) ? ix_tile(ix, i, j, p, q) : ix_tile(ix, j, i, q, p);
        if (!inc)
          e->ycost[cix] = e->c[cix] + ((i < j) ? e->theta[t] : 0.0);
        else if (i < j)
          e->ycost[cix] = e->theta[t];
        else
          e->ycost[cix] = e->ybar[t] + e->dx[(size_t)i * m + p] / (m - 1);
      }
    }
  }
#pragma omp parallel
  {
    double* u = malloc(sizeof(double) * my);
    double* v = malloc(sizeof(double) * my);
#pragma omp for schedule(static)
    for (int ipf = 0; ipf < m * m; ++ipf) {
      const double* cost = e->ycost + (size_t)ipf * my * my;
      e->delta[ipf] = orc_lap_solve(cost, my, NULL, NULL, u, v);
      double* py = e->piy + (size_t)ipf * my * my;
      for (int a = 0; a < my; ++a)
        for (int b = 0; b < my; ++b) py[a * my + b] = cost[a * my + b] - u[a] - v[b];
    }
    free(u);
    free(v);
  }
}

/* stage_x, src/rlt2.cpp:428-449 */
static void stage_x(orc_engine* e) {
  const int m = e->m;
  const int inc = is_fast(e) && e->iter > 0;
  for (size_t ip = 0; ip < (size_t)m * m; ++ip)
    e->xcost[ip] = e->delta[ip] + (inc ? 0.0 : e->b[ip]);
  double* u = malloc(sizeof(double) * m);
  double* v = malloc(sizeof(double) * m);
  const double nu = orc_lap_solve(e->xcost, m, e->xrow, e->xcol, u, v);
  for (size_t ip = 0; ip < (size_t)m * m; ++ip)
    e->pix[ip] = e->xcost[ip] - u[ip / m] - v[ip % m];
  free(u);
  free(v);
  if (is_fast(e)) {
    e->running += nu;
    e->last_bound = e->running + e->offset;
  } else {
    e->last_bound = nu + e->offset;
  }
  if (e->last_bound > e->best) e->best = e->last_bound;
}

/* feasibility_check, src/rlt2.cpp:453-473 */
static int feasibility_check(orc_engine* e) {
  const double tol = 1e-7;
  const sidx* ix = &e->ix;
  const int m = e->m;
  const int* s = e->xrow;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      if (j != i && e->piy[ix_cidx(ix, i, s[i], j, s[j])] > tol) return 0;
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) {
      const int t = ix_tile(ix, i, j, s[i], s[j]);
      const double* tz = e->piz + (size_t)t * ix->esz;
      for (int k = 0; k < m; ++k)
        if (k != i && k != j && tz[ix_cell(ix, i, j, s[i], s[j], k, s[k])] > tol)
          return 0;
    }
  memcpy(e->cert, s, sizeof(int) * m);
  e->has_cert = 1;
  e->cert_val = e->last_bound;
  return 1;
}

/* sa_perturb, src/rlt2.cpp:477-513 */
static void sa_perturb(orc_engine* e) {
  const double nu = e->best;
  if (nu <= 0) return;
  if (e->temp <= 0) {
    const double ub = isfinite(e->cfg.upper_bound) ? e->cfg.upper_bound
                                                   : 1.05 * nu + 1.0;
    e->temp = e->cfg.sa_t0_fraction * ub;
  }
  const double cap = e->cfg.sa_kappa_lb_cap * nu;
  const int m = e->m;
  double* amt = calloc(2 * m, sizeof(double));
  double total = 0;
  for (int s = 0; s < 2 * m; ++s) {
    const double kap = mt64_uniform01(&e->rng) * cap;
    const int accept = mt64_uniform01(&e->rng) < exp(-kap / e->temp);
    if (accept) {
      amt[s] = kap;
      total += kap;
    }
  }
  if (total > cap)
    for (int s = 0; s < 2 * m; ++s) amt[s] *= cap / total;
  for (int i = 0; i < m; ++i) e->sa_fac[i] = amt[i] / m;
  for (int p = 0; p < m; ++p) e->sa_loc[p] = amt[m + p] / m;
  double drained = 0;
  for (int i = 0; i < m; ++i) {
    drained += e->sa_fac[i] + e->sa_loc[i];
    for (int p = 0; p < m; ++p) e->b[(size_t)i * m + p] -= e->sa_fac[i] + e->sa_loc[p];
  }
  if (is_fast(e)) e->running -= drained;
  if ((e->iter + 1) % e->cfg.sa_cool_period == 0) e->temp *= e->cfg.sa_cool_factor;
  free(amt);
}

static double orc_gap(const orc_engine* e) { /* src/rlt2.cpp:532-535 */
  if (!isfinite(e->cfg.upper_bound) || e->cfg.upper_bound == 0) return INFINITY;
  return (e->cfg.upper_bound - e->best) / e->cfg.upper_bound;
}

/* iterate, src/rlt2.cpp:515-530 */
int orc_engine_iterate(orc_engine* e, double* bound) {
  memset(&e->rec, 0, sizeof e->rec);
  if (e->iter > 0) ascent_update(e);
  int rc = stage_z(e);
  if (rc) return rc;
  stage_y(e);
  stage_x(e);
  if (!e->has_cert) {
    const int feas = feasibility_check(e);
    if (!feas && e->cfg.sa_enabled) sa_perturb(e);
  }
  ++e->iter;
  e->rec.iteration = e->iter;
  e->rec.bound = e->last_bound;
  e->rec.gap = orc_gap(e);
  if (bound) *bound = e->last_bound;
  return 0;
}

/* run, src/rlt2.cpp:544-588 */
int orc_engine_run(orc_engine* e, qapb_report* rep, qapb_record* recs,
                   int max_records, int* cert) {
  rep->termination = QAPB_TERM_ITERATION_LIMIT;
  rep->n_records = 0;
  int cap = 1024, nh = 0;
  double* hist = malloc(sizeof(double) * cap);
  while (e->iter < e->cfg.iter_limit) {
    int rc = orc_engine_iterate(e, NULL);
    if (rc) {
      free(hist);
      return rc;
    }
    if (e->cfg.record_history && recs && rep->n_records < max_records)
      recs[rep->n_records++] = e->rec;
    if (nh == cap) hist = realloc(hist, sizeof(double) * (cap *= 2));
    hist[nh++] = e->best;
    if (e->has_cert) {
      rep->termination = QAPB_TERM_FEASIBLE_FOUND;
      break;
    }
    if (e->cfg.min_gap > 0 && orc_gap(e) <= e->cfg.min_gap) {
      rep->termination = QAPB_TERM_GAP_CLOSED;
      break;
    }
    if (e->best >= e->cfg.fathom_threshold) {
      rep->termination = QAPB_TERM_EARLY_STOP;
      break;
    }
    if (e->cfg.early_stop_window > 0 && nh > e->cfg.early_stop_window) {
      const double prev = hist[nh - 1 - e->cfg.early_stop_window];
      const double scale = fabs(e->best) > 1.0 ? fabs(e->best) : 1.0;
      if (e->best - prev < e->cfg.early_stop_delta * scale) {
        rep->termination = QAPB_TERM_EARLY_STOP;
        break;
      }
    }
  }
  free(hist);
  rep->best_bound = e->best;
  rep->upper_bound = e->cfg.upper_bound;
  rep->gap = orc_gap(e);
  rep->iterations = e->iter;
  rep->has_certificate = e->has_cert;
  rep->certificate_value = e->has_cert ? e->cert_val : 0.0;
  rep->wall_ms = 0;
  if (e->has_cert && cert) memcpy(cert, e->cert, sizeof(int) * e->m);
  return 0;
}

static const double* arr(orc_engine* e, int which, size_t* n) {
  switch (which) {
    case QAPB_ARR_PI_Z: *n = e->nd; return e->piz;
    case QAPB_ARR_PI_Y: *n = e->nc; return e->piy;
    case QAPB_ARR_PI_X: *n = e->nb; return e->pix;
    case QAPB_ARR_STORE_B: *n = e->nb; return e->b;
    case QAPB_ARR_STORE_C: *n = e->nc; return e->c;
    case QAPB_ARR_STORE_D: *n = e->nd; return e->d;
    case QAPB_ARR_THETA: *n = e->ix.tiles; return e->theta;
    case QAPB_ARR_DELTA: *n = e->nb; return e->delta;
    case QAPB_ARR_INCZ: *n = e->incz ? e->nd : 0; return e->incz;
  }
  *n = 0;
  return NULL;
}

int orc_engine_array_size(orc_engine* e, int which, size_t* count) {
  arr(e, which, count);
  return 0;
}

int orc_engine_get_array(orc_engine* e, int which, double* dst, size_t count) {
  size_t n;
  const double* a = arr(e, which, &n);
  if (!a || n != count) return set_err(QAPB_EINVAL, "bad array request");
  memcpy(dst, a, sizeof(double) * n);
  return 0;
}

int orc_engine_scalars(orc_engine* e, double* best, double* gap, int* iteration,
                       double* last_bound, double* running) {
  if (best) *best = e->best;
  if (gap) *gap = orc_gap(e);
  if (iteration) *iteration = e->iter;
  if (last_bound) *last_bound = e->last_bound;
  if (running) *running = e->running;
  return 0;
}

int orc_engine_certificate(orc_engine* e, int* has, int* perm, double* value) {
  *has = e->has_cert;
  if (e->has_cert && perm) memcpy(perm, e->cert, sizeof(int) * e->m);
  if (value) *value = e->cert_val;
  return 0;
}

int orc_engine_x_assignment(orc_engine* e, int* xrow) {
  memcpy(xrow, e->xrow, sizeof(int) * e->m);
  return 0;
}

void orc_exp_batch(const double* x, double* y, size_t n) {
  double (*volatile libm_exp)(double) = exp;  /* a real libm call per element */
  for (size_t i = 0; i < n; ++i) y[i] = libm_exp(x[i]);
}

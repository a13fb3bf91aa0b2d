// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin C wrapper around the *unmodified* reference library
// (/root/reference/proj/src/{instance,lap,rlt2}.cpp, compiled by
// oracle/Makefile into oracle/_ref/libqapref.so).  It lets the pytest parity
// suite, tests/golden/make_golden.py and bench.py's cpu_baseline / reference
// arm call the reference implementation through ctypes.  Nothing in the
// product (paper_1710_03732_b200/) links or loads this file.
//
// The reference's private engine arrays (theta_, delta_, incz_) are exposed
// for parity checks by compiling this translation unit with `private` mapped
// to `public`; the class layout is unchanged.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#define private public
#include "qap/rlt2.hpp"
#undef private
#include "qap/instance.hpp"
#include "qap/lap.hpp"

#include "../include/qapb200.h"

#define QREF extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return QAPB_OK;
  } catch (const std::invalid_argument& e) {
    return fail(e, QAPB_EINVAL);
  } catch (const std::logic_error& e) {
    return fail(e, QAPB_ELOGIC);
  } catch (const std::runtime_error& e) {
    return fail(e, QAPB_ERUNTIME);
  } catch (const std::exception& e) {
    return fail(e, QAPB_ERUNTIME);
  }
}

qap::AscentConfig to_cfg(const qapb_config* c) {
  qap::AscentConfig a;
  if (!c) return a;
  a.variant = static_cast<qap::Variant>(c->variant);
  a.sa_enabled = c->sa_enabled != 0;
  a.iter_limit = c->iter_limit;
  a.min_gap = c->min_gap;
  a.kappa_z_upper = c->kappa_z_upper;
  a.phi_split = c->phi_split;
  a.kappa_y = c->kappa_y;
  a.kappa_x = c->kappa_x;
  a.varphi = c->varphi;
  a.sa_t0_fraction = c->sa_t0_fraction;
  a.sa_kappa_lb_cap = c->sa_kappa_lb_cap;
  a.sa_cool_factor = c->sa_cool_factor;
  a.sa_cool_period = c->sa_cool_period;
  a.workers = c->workers;
  a.seed = c->seed;
  a.upper_bound = c->upper_bound;
  a.fathom_threshold = c->fathom_threshold;
  a.early_stop_window = c->early_stop_window;
  a.early_stop_delta = c->early_stop_delta;
  a.record_history = c->record_history != 0;
  return a;
}

int term_code(const std::string& s) {
  if (s == "gap-closed") return QAPB_TERM_GAP_CLOSED;
  if (s == "feasible-found") return QAPB_TERM_FEASIBLE_FOUND;
  if (s == "early-stop") return QAPB_TERM_EARLY_STOP;
  return QAPB_TERM_ITERATION_LIMIT;
}

void fill_report(const qap::BoundReport& r, qapb_report* rep,
                 qapb_record* recs, int max_records, int* cert) {
  if (rep) {
    rep->best_bound = r.best_bound;
    rep->upper_bound = r.upper_bound;
    rep->gap = r.gap;
    rep->termination = term_code(r.termination);
    rep->iterations = r.iterations;
    rep->has_certificate = !r.certificate.empty();
    rep->certificate_value = r.certificate_value;
    rep->wall_ms = r.wall_ms;
    rep->n_records = 0;
  }
  if (recs) {
    int k = std::min<int>(max_records, (int)r.records.size());
    for (int i = 0; i < k; ++i) {
      recs[i].iteration = r.records[i].iteration;
      recs[i].bound = r.records[i].bound;
      recs[i].gap = r.records[i].gap;
      recs[i].z_ms = r.records[i].z_ms;
      recs[i].y_ms = r.records[i].y_ms;
      recs[i].x_ms = r.records[i].x_ms;
    }
    if (rep) rep->n_records = k;
  }
  if (cert && !r.certificate.empty())
    std::copy(r.certificate.begin(), r.certificate.end(), cert);
}

qap::QapInstance make_inst(int n, const double* flow, const double* dist,
                           const double* linear) {
  qap::QapInstance inst;
  inst.n = n;
  inst.flow.assign(flow, flow + (size_t)n * n);
  inst.dist.assign(dist, dist + (size_t)n * n);
  if (linear)
    inst.linear.assign(linear, linear + (size_t)n * n);
  else
    inst.linear.assign((size_t)n * n, 0.0);
  inst.name = "ffi";
  return inst;
}

qap::CoefficientStore make_store(int m, const double* b, const double* c,
                                 const double* d, double offset) {
  qap::CoefficientStore st;
  st.m = m;
  st.idx = qap::StoreIndex(m);
  st.b.assign(b, b + (size_t)m * m);
  st.c.assign(c, c + (size_t)m * m * (m - 1) * (m - 1));
  const size_t nd = (size_t)st.idx.tiles * st.idx.esz;
  if (d)
    st.d.assign(d, d + nd);
  else
    st.d.assign(nd, 0.0);
  st.offset = offset;
  return st;
}
}  // namespace

struct qref_engine {
  qap::AscentEngine eng;
};

QREF const char* qref_last_error() { return g_err.c_str(); }

QREF int qref_lap_solve(const double* cost, int m, int* r2c, int* c2r,
                        double* u, double* v, double* value) {
  return guard([&] {
    qap::LapSolver s(m);
    *value = s.solve(cost, m, r2c, c2r, u, v);
  });
}

QREF int qref_lap_solve_batch(const double* costs, int m, int count,
                              int workers, double* values, int* r2c, int* c2r,
                              double* u, double* v) {
  return guard([&] {
    qap::LapBatch b;
    b.resize(count, m);
    std::memcpy(b.costs.data(), costs, sizeof(double) * (size_t)count * m * m);
    qap::solve_batch(b, workers);
    if (values) std::copy(b.values.begin(), b.values.end(), values);
    if (r2c) std::copy(b.row_to_col.begin(), b.row_to_col.end(), r2c);
    if (c2r) std::copy(b.col_to_row.begin(), b.col_to_row.end(), c2r);
    if (u) std::copy(b.u.begin(), b.u.end(), u);
    if (v) std::copy(b.v.begin(), b.v.end(), v);
  });
}

QREF int qref_generate_instance(int n, unsigned long long seed, int max_entry,
                                double* flow, double* dist) {
  return guard([&] {
    auto inst = qap::generate_instance(n, seed, max_entry);
    std::copy(inst.flow.begin(), inst.flow.end(), flow);
    std::copy(inst.dist.begin(), inst.dist.end(), dist);
  });
}

QREF int qref_evaluate_objective(int n, const double* flow, const double* dist,
                                 const double* linear, const int* perm,
                                 double* value) {
  return guard([&] {
    auto inst = make_inst(n, flow, dist, linear);
    *value = qap::evaluate_objective(inst, std::vector<int>(perm, perm + n));
  });
}

QREF int qref_init_coefficients(int n, const double* flow, const double* dist,
                                const double* linear, double* b, double* c,
                                double* d) {
  return guard([&] {
    auto st = qap::init_coefficients(make_inst(n, flow, dist, linear));
    std::copy(st.b.begin(), st.b.end(), b);
    std::copy(st.c.begin(), st.c.end(), c);
    if (d) std::copy(st.d.begin(), st.d.end(), d);
  });
}

QREF int qref_store_evaluate(int m, const double* b, const double* c,
                             const double* d, double offset, const int* perm,
                             double* value) {
  return guard([&] {
    auto st = make_store(m, b, c, d, offset);
    *value = qap::store_evaluate(st, std::vector<int>(perm, perm + m));
  });
}

QREF int qref_collapse_store(int m, const double* b, const double* c,
                             const double* d, double offset, int fac, int loc,
                             double* ob, double* oc, double* od,
                             double* ooffset) {
  return guard([&] {
    auto st = make_store(m, b, c, d, offset);
    auto out = qap::collapse_store(st, fac, loc);
    std::copy(out.b.begin(), out.b.end(), ob);
    std::copy(out.c.begin(), out.c.end(), oc);
    if (od) std::copy(out.d.begin(), out.d.end(), od);
    *ooffset = out.offset;
  });
}

QREF int qref_redistribute_family(const double pi[3], double add[3],
                                  int virtual_slots, double tol, int* ok) {
  return guard([&] { *ok = qap::redistribute_family(pi, add, virtual_slots, tol); });
}

QREF int qref_engine_create(int m, const double* b, const double* c,
                            const double* d, double offset,
                            const qapb_config* cfg, qref_engine** out) {
  return guard([&] {
    *out = new qref_engine{qap::AscentEngine(make_store(m, b, c, d, offset),
                                             to_cfg(cfg))};
  });
}

QREF int qref_engine_create_instance(int n, const double* flow,
                                     const double* dist, const double* linear,
                                     const qapb_config* cfg,
                                     qref_engine** out) {
  return guard([&] {
    *out = new qref_engine{qap::AscentEngine(
        qap::init_coefficients(make_inst(n, flow, dist, linear)), to_cfg(cfg))};
  });
}

QREF int qref_engine_destroy(qref_engine* e) {
  delete e;
  return QAPB_OK;
}

QREF int qref_engine_iterate(qref_engine* e, double* bound) {
  return guard([&] {
    double b = e->eng.iterate();
    if (bound) *bound = b;
  });
}

QREF int qref_engine_run(qref_engine* e, qapb_report* rep, qapb_record* recs,
                         int max_records, int* cert) {
  return guard([&] { fill_report(e->eng.run(), rep, recs, max_records, cert); });
}

QREF int qref_engine_scalars(qref_engine* e, double* best, double* gap,
                             int* iteration, double* last_bound,
                             double* running) {
  if (best) *best = e->eng.best_bound();
  if (gap) *gap = e->eng.gap();
  if (iteration) *iteration = e->eng.iteration();
  if (last_bound) *last_bound = e->eng.last_bound_;
  if (running) *running = e->eng.running_;
  return QAPB_OK;
}

QREF int qref_engine_certificate(qref_engine* e, int* has, int* perm,
                                 double* value) {
  *has = e->eng.has_certificate();
  if (*has && perm)
    std::copy(e->eng.certificate().begin(), e->eng.certificate().end(), perm);
  if (value) *value = e->eng.certificate_value();
  return QAPB_OK;
}

QREF int qref_engine_x_assignment(qref_engine* e, int* xrow) {
  std::copy(e->eng.x_assignment().begin(), e->eng.x_assignment().end(), xrow);
  return QAPB_OK;
}

static const std::vector<double>* ref_array(qref_engine* e, int which) {
  auto& g = e->eng;
  switch (which) {
    case QAPB_ARR_PI_Z: return &g.piz_;
    case QAPB_ARR_PI_Y: return &g.piy_;
    case QAPB_ARR_PI_X: return &g.pix_;
    case QAPB_ARR_STORE_B: return &g.st_.b;
    case QAPB_ARR_STORE_C: return &g.st_.c;
    case QAPB_ARR_STORE_D: return &g.st_.d;
    case QAPB_ARR_THETA: return &g.theta_;
    case QAPB_ARR_DELTA: return &g.delta_;
    case QAPB_ARR_INCZ: return &g.incz_;
  }
  return nullptr;
}

QREF int qref_engine_array_size(qref_engine* e, int which, size_t* count) {
  auto* a = ref_array(e, which);
  if (!a) {
    g_err = "unknown array";
    return QAPB_EINVAL;
  }
  *count = a->size();
  return QAPB_OK;
}

QREF int qref_engine_get_array(qref_engine* e, int which, double* dst,
                               size_t count) {
  auto* a = ref_array(e, which);
  if (!a || count != a->size()) {
    g_err = "bad array request";
    return QAPB_EINVAL;
  }
  std::copy(a->begin(), a->end(), dst);
  return QAPB_OK;
}

QREF int qref_engine_snapshot(qref_engine* e, double* b, double* c, double* d,
                              double* offset) {
  return guard([&] {
    auto st = e->eng.snapshot();
    std::copy(st.b.begin(), st.b.end(), b);
    std::copy(st.c.begin(), st.c.end(), c);
    std::copy(st.d.begin(), st.d.end(), d);
    *offset = st.offset;
  });
}

QREF int qref_run_ascent(int n, const double* flow, const double* dist,
                         const double* linear, const qapb_config* cfg,
                         qapb_report* rep, qapb_record* recs, int max_records,
                         int* cert) {
  return guard([&] {
    fill_report(qap::run_ascent(make_inst(n, flow, dist, linear), to_cfg(cfg)),
                rep, recs, max_records, cert);
  });
}

// BoundReport::to_json of the reference (nlohmann dump(2), rlt2.cpp:604-630),
// same argument convention as qapb_report_json (include/qapb200.h)
QREF int qref_report_json(const char* instance, const char* variant, int sa_enabled,
                          double best_bound, double upper_bound, double gap,
                          const char* termination, int iterations, double wall_ms,
                          const int* cert, int ncert, double cert_value, const double* recs,
                          int nrec, char* out, size_t cap, size_t* len) {
  return guard([&] {
    qap::BoundReport r;
    r.instance = instance ? instance : "";
    r.variant = variant ? variant : "";
    r.sa_enabled = sa_enabled != 0;
    r.best_bound = best_bound;
    r.upper_bound = upper_bound;
    r.gap = gap;
    r.termination = termination ? termination : "";
    r.iterations = iterations;
    r.wall_ms = wall_ms;
    if (cert) r.certificate.assign(cert, cert + ncert);
    r.certificate_value = cert_value;
    for (int k = 0; k < nrec; ++k) {
      qap::IterationRecord x;
      x.iteration = (int)recs[6 * k];
      x.bound = recs[6 * k + 1];
      x.gap = recs[6 * k + 2];
      x.z_ms = recs[6 * k + 3];
      x.y_ms = recs[6 * k + 4];
      x.x_ms = recs[6 * k + 5];
      r.records.push_back(x);
    }
    const std::string j = r.to_json();
    if (len) *len = j.size();
    if (!out || cap <= j.size()) throw std::invalid_argument("buffer too small");
    std::memcpy(out, j.c_str(), j.size() + 1);
  });
}

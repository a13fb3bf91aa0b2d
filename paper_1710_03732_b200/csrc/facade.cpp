// facade.cpp — the reference's C++ API (include/qap/{instance,lap,rlt2}.hpp)
// implemented over the C-ABI (include/qapb200.h).  This is the binding a
// maintainer swaps in for proj/src/{lap,rlt2}.cpp: callers (bnb.cpp,
// qap_cli.cpp, the reference's unit tests) compile unchanged against these
// headers and link libqapb200.so.  Status codes become the reference's
// exception types again.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <random>
#include <sstream>
#include <stdexcept>

#include "qap/instance.hpp"
#include "qap/lap.hpp"
#include "qap/rlt2.hpp"
#include "qapb200.h"

#define QAP_API __attribute__((visibility("default")))

namespace qap {
namespace {

void check(qapb_status rc) {
  if (rc == QAPB_OK) return;
  const std::string msg = qapb_last_error();
  switch (rc) {
    case QAPB_EINVAL: throw std::invalid_argument(msg);
    case QAPB_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

qapb_config to_c(const AscentConfig& a) {
  qapb_config c;
  qapb_config_init(&c);
  c.variant = static_cast<int>(a.variant);
  c.sa_enabled = a.sa_enabled;
  c.iter_limit = a.iter_limit;
  c.min_gap = a.min_gap;
  c.kappa_z_upper = a.kappa_z_upper;
  c.phi_split = a.phi_split;
  c.kappa_y = a.kappa_y;
  c.kappa_x = a.kappa_x;
  c.varphi = a.varphi;
  c.sa_t0_fraction = a.sa_t0_fraction;
  c.sa_kappa_lb_cap = a.sa_kappa_lb_cap;
  c.sa_cool_factor = a.sa_cool_factor;
  c.sa_cool_period = a.sa_cool_period;
  c.workers = a.workers;
  c.seed = a.seed;
  c.upper_bound = a.upper_bound;
  c.fathom_threshold = a.fathom_threshold;
  c.early_stop_window = a.early_stop_window;
  c.early_stop_delta = a.early_stop_delta;
  c.record_history = a.record_history;
  c.device = a.device;
  return c;
}

const char* term_name(int t) {
  switch (t) {
    case QAPB_TERM_GAP_CLOSED: return "gap-closed";
    case QAPB_TERM_FEASIBLE_FOUND: return "feasible-found";
    case QAPB_TERM_EARLY_STOP: return "early-stop";
  }
  return "iteration-limit";
}

size_t nc_of(int m) { return (size_t)m * m * (m - 1) * (m - 1); }
size_t nd_of(int m) {
  if (m < 3) return 0;
  return (size_t)(m * (m - 1) / 2) * (m * (m - 1)) * (m - 2) * (m - 2);
}

std::string slurp(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("cannot open " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

BoundReport report_from(const qapb_report& r, std::vector<qapb_record>& recs,
                        const std::vector<int>& cert, const AscentConfig& cfg) {
  BoundReport rep;
  rep.variant = variant_name(cfg.variant);
  rep.sa_enabled = cfg.sa_enabled;
  rep.best_bound = r.best_bound;
  rep.upper_bound = r.upper_bound;
  rep.gap = r.gap;
  rep.termination = term_name(r.termination);
  rep.iterations = r.iterations;
  rep.wall_ms = r.wall_ms;
  if (r.has_certificate) {
    rep.certificate = cert;
    rep.certificate_value = r.certificate_value;
  }
  for (int k = 0; k < r.n_records; ++k)
    rep.records.push_back(IterationRecord{recs[k].iteration, recs[k].bound, recs[k].gap,
                                          recs[k].z_ms, recs[k].y_ms, recs[k].x_ms});
  return rep;
}
}  // namespace

// ---------------------------------------------------------------- instance
QAP_API double evaluate_objective(const QapInstance& inst, const std::vector<int>& perm) {
  const int n = inst.n;
  if ((int)perm.size() != n) throw std::invalid_argument("perm size != n");
  std::vector<char> seen(n, 0);
  for (int i = 0; i < n; ++i) {
    if (perm[i] < 0 || perm[i] >= n || seen[perm[i]])
      throw std::invalid_argument("not a permutation");
    seen[perm[i]] = 1;
  }
  double v = 0;
  for (int i = 0; i < n; ++i) {
    v += inst.b(i, perm[i]);
    for (int j = 0; j < n; ++j) v += inst.f(i, j) * inst.d(perm[i], perm[j]);
  }
  return v;
}

QAP_API QapInstance parse_qaplib(const std::string& text, bool swap_order,
                                 const std::string& name) {
  std::istringstream in(text);
  QapInstance inst;
  inst.name = name;
  if (!(in >> inst.n) || inst.n <= 0) throw std::runtime_error("bad instance size");
  const int nn = inst.n * inst.n;
  auto block = [&](const char* what) {
    std::vector<double> out(nn);
    for (double& x : out)
      if (!(in >> x)) throw std::runtime_error(std::string("truncated input reading ") + what);
    return out;
  };
  std::vector<double> a = block("first matrix");
  std::vector<double> b = block("second matrix");
  inst.flow = swap_order ? b : a;
  inst.dist = swap_order ? a : b;
  double probe;
  if (in >> probe) {
    inst.linear.resize(nn);
    inst.linear[0] = probe;
    for (int i = 1; i < nn; ++i)
      if (!(in >> inst.linear[i])) throw std::runtime_error("truncated linear-cost matrix");
  } else {
    inst.linear.assign(nn, 0.0);
  }
  return inst;
}

QAP_API QapInstance load_qaplib_file(const std::string& path, bool swap_order) {
  std::string base = path.substr(path.find_last_of('/') == std::string::npos
                                     ? 0
                                     : path.find_last_of('/') + 1);
  const size_t dot = base.find_last_of('.');
  if (dot != std::string::npos) base = base.substr(0, dot);
  return parse_qaplib(slurp(path), swap_order, base);
}

QAP_API std::vector<int> parse_solution(const std::string& text, int expect_n, double* value) {
  std::istringstream in(text);
  int n;
  double v;
  if (!(in >> n >> v)) throw std::runtime_error("bad solution header");
  if (n != expect_n) throw std::runtime_error("solution size mismatch");
  std::vector<int> perm(n);
  for (int& p : perm) {
    if (!(in >> p)) throw std::runtime_error("truncated permutation");
    p -= 1;
  }
  std::vector<char> seen(n, 0);
  for (int p : perm) {
    if (p < 0 || p >= n || seen[p]) throw std::runtime_error("solution is not a permutation");
    seen[p] = 1;
  }
  if (value) *value = v;
  return perm;
}

QAP_API std::vector<int> load_solution_file(const std::string& path, int expect_n,
                                            double* value) {
  return parse_solution(slurp(path), expect_n, value);
}

QAP_API std::string format_qaplib(const QapInstance& inst) {
  std::ostringstream out;
  out << inst.n << "\n\n";
  for (const auto* mtx : {&inst.flow, &inst.dist}) {
    for (int i = 0; i < inst.n; ++i) {
      for (int j = 0; j < inst.n; ++j) {
        const double v = (*mtx)[(size_t)i * inst.n + j];
        if (j) out << ' ';
        if (v == std::floor(v))
          out << (long long)v;
        else
          out << v;
      }
      out << "\n";
    }
    out << "\n";
  }
  return out.str();
}

QAP_API QapInstance generate_instance(int n, std::uint64_t seed, int max_entry) {
  if (n < 2) throw std::invalid_argument("n must be >= 2");
  QapInstance inst;
  inst.n = n;
  inst.flow.assign((size_t)n * n, 0.0);
  inst.dist.assign((size_t)n * n, 0.0);
  inst.linear.assign((size_t)n * n, 0.0);
  inst.name = "rand" + std::to_string(n) + "-" + std::to_string(seed);
  std::mt19937_64 rng(seed);
  auto draw = [&]() { return (double)(rng() % (std::uint64_t)(max_entry + 1)); };
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) inst.flow[(size_t)i * n + j] = inst.flow[(size_t)j * n + i] = draw();
  for (int p = 0; p < n; ++p)
    for (int q = p + 1; q < n; ++q) inst.dist[(size_t)p * n + q] = inst.dist[(size_t)q * n + p] = draw();
  return inst;
}

QAP_API std::vector<ManifestEntry> parse_manifest(const std::string& text) {
  std::vector<ManifestEntry> out;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    const size_t h = line.find('#');
    if (h != std::string::npos) line.erase(h);
    std::istringstream ls(line);
    ManifestEntry e;
    if (!(ls >> e.path)) continue;
    std::string tok;
    while (ls >> tok) {
      if (tok == "swap")
        e.swap_order = true;
      else if (tok.rfind("opt=", 0) == 0)
        e.best_known = std::stod(tok.substr(4));
      else if (tok.rfind("sln=", 0) == 0)
        e.sln_path = tok.substr(4);
      else
        throw std::runtime_error("unknown manifest token: " + tok);
    }
    out.push_back(e);
  }
  return out;
}

QAP_API std::vector<ManifestEntry> load_manifest_file(const std::string& path) {
  auto entries = parse_manifest(slurp(path));
  const size_t slash = path.find_last_of('/');
  const std::string dir = slash == std::string::npos ? "" : path.substr(0, slash + 1);
  for (auto& e : entries) {
    if (!e.path.empty() && e.path[0] != '/') e.path = dir + e.path;
    if (!e.sln_path.empty() && e.sln_path[0] != '/') e.sln_path = dir + e.sln_path;
  }
  return entries;
}

// ---------------------------------------------------------------- LAP
QAP_API void LapSolver::reserve(int m) { max_m_ = std::max(max_m_, m); }

QAP_API double LapSolver::solve(const double* cost, int m, int* row_to_col, int* col_to_row,
                                double* u, double* v) {
  if (m <= 0) throw std::invalid_argument("lap: m must be positive");
  double value = 0;
  check(qapb_lap_solve(cost, m, row_to_col, col_to_row, u, v, &value));
  return value;
}

QAP_API LapResult solve_lap(const double* cost, int m) {
  LapResult r;
  r.row_to_col.resize(m);
  r.col_to_row.resize(m);
  r.u.resize(m);
  r.v.resize(m);
  LapSolver s(m);
  r.value = s.solve(cost, m, r.row_to_col.data(), r.col_to_row.data(), r.u.data(), r.v.data());
  return r;
}

QAP_API LapResult solve_lap(const std::vector<double>& cost, int m) {
  if ((int)cost.size() != m * m) throw std::invalid_argument("lap: cost size != m*m");
  return solve_lap(cost.data(), m);
}

QAP_API void LapBatch::resize(int count_, int m_) {
  m = m_;
  count = count_;
  costs.assign((size_t)count * m * m, 0.0);
  values.assign(count, 0.0);
  row_to_col.assign((size_t)count * m, -1);
  col_to_row.assign((size_t)count * m, -1);
  u.assign((size_t)count * m, 0.0);
  v.assign((size_t)count * m, 0.0);
}

QAP_API void solve_batch(LapBatch& b, int) {
  if (b.count == 0) return;
  if (b.m <= 0) throw std::invalid_argument("lap: m must be positive");
  check(qapb_lap_solve_batch(b.costs.data(), b.m, b.count, b.values.data(), b.row_to_col.data(),
                             b.col_to_row.data(), b.u.data(), b.v.data()));
}

QAP_API void solve_batch_serial(LapBatch& b) { solve_batch(b, 1); }

// ---------------------------------------------------------------- RLT2
QAP_API const char* variant_name(Variant v) { return qapb_variant_name(static_cast<int>(v)); }

QAP_API Variant parse_variant(const std::string& s) {
  int v = 0;
  check(qapb_parse_variant(s.c_str(), &v));
  return static_cast<Variant>(v);
}

QAP_API StoreIndex::StoreIndex(int m_) : m(m_) {
  fpairs = m * (m - 1) / 2;
  lpairs = m * (m - 1);
  tiles = fpairs * lpairs;
  esz = (m - 2) * (m - 2);
  fp_i.resize(fpairs);
  fp_j.resize(fpairs);
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) {
      fp_i[fpair(i, j)] = i;
      fp_j[fpair(i, j)] = j;
    }
  lp_p.resize(lpairs);
  lp_q.resize(lpairs);
  for (int p = 0; p < m; ++p)
    for (int q = 0; q < m; ++q)
      if (p != q) {
        lp_p[lpair(p, q)] = p;
        lp_q[lpair(p, q)] = q;
      }
}

QAP_API CoefficientStore init_coefficients(const QapInstance& inst) {
  if (inst.n < 3) throw std::invalid_argument("init_coefficients: n >= 3 required by RLT2");
  const int m = inst.n;
  CoefficientStore st;
  st.m = m;
  st.idx = StoreIndex(m);
  st.b.resize((size_t)m * m);
  st.c.resize(nc_of(m));
  st.d.assign(nd_of(m), 0.0);
  const double* lin = inst.linear.empty() ? nullptr : inst.linear.data();
  check(qapb_init_coefficients(m, inst.flow.data(), inst.dist.data(), lin, st.b.data(),
                               st.c.data(), nullptr));
  return st;
}

QAP_API double store_evaluate(const CoefficientStore& st, const std::vector<int>& perm) {
  double v = 0;
  check(qapb_store_evaluate(st.m, st.b.data(), st.c.data(), st.d.data(), st.offset, perm.data(),
                            &v));
  return v;
}

QAP_API CoefficientStore collapse_store(const CoefficientStore& st, int fac, int loc) {
  const int mc = st.m - 1;
  if (mc < 2) throw std::invalid_argument("collapse_store: store too small");
  CoefficientStore out;
  out.m = mc;
  out.idx = StoreIndex(mc);
  out.b.resize((size_t)mc * mc);
  out.c.resize(nc_of(mc));
  out.d.assign(nd_of(mc), 0.0);
  check(qapb_collapse_store(st.m, st.b.data(), st.c.data(), st.d.data(), st.offset, fac, loc,
                            out.b.data(), out.c.data(), out.d.data(), &out.offset));
  return out;
}

QAP_API bool redistribute_family(const double pi[3], double add[3], int virtual_slots,
                                 double tol) {
  int ok = 0;
  check(qapb_redistribute_family(pi, add, virtual_slots, tol, &ok));
  return ok != 0;
}

QAP_API AscentEngine::AscentEngine(CoefficientStore store, const AscentConfig& cfg)
    : cfg_(cfg), m_(store.m) {
  if (m_ < 3) throw std::invalid_argument("AscentEngine: m >= 3 required");
  const qapb_config c = to_c(cfg);
  check(qapb_engine_create(store.m, store.b.data(), store.c.data(), store.d.data(), store.offset,
                           &c, &h_));
}

QAP_API AscentEngine::~AscentEngine() {
  if (h_) qapb_engine_destroy(h_);
}

QAP_API AscentEngine::AscentEngine(AscentEngine&& o) noexcept
    : h_(o.h_), cfg_(o.cfg_), m_(o.m_) {
  o.h_ = nullptr;
}

QAP_API AscentEngine& AscentEngine::operator=(AscentEngine&& o) noexcept {
  if (this != &o) {
    if (h_) qapb_engine_destroy(h_);
    h_ = o.h_;
    cfg_ = o.cfg_;
    m_ = o.m_;
    o.h_ = nullptr;
    invalidate();
  }
  return *this;
}

void AscentEngine::invalidate() {
  st_ok_ = piz_ok_ = piy_ok_ = pix_ok_ = cert_ok_ = x_ok_ = false;
}

QAP_API double AscentEngine::iterate() {
  double b = 0;
  invalidate();
  check(qapb_engine_iterate(h_, &b));
  return b;
}

QAP_API BoundReport AscentEngine::run() {
  invalidate();
  std::vector<qapb_record> recs(std::max(1, cfg_.iter_limit));
  std::vector<int> cert(m_, -1);
  qapb_report r{};
  check(qapb_engine_run(h_, &r, recs.data(), (int)recs.size(), cert.data()));
  return report_from(r, recs, cert, cfg_);
}

QAP_API double AscentEngine::best_bound() const {
  double v = 0;
  check(qapb_engine_best_bound(h_, &v));
  return v;
}

QAP_API double AscentEngine::gap() const {
  double v = 0;
  check(qapb_engine_gap(h_, &v));
  return v;
}

QAP_API int AscentEngine::iteration() const {
  int v = 0;
  check(qapb_engine_iteration(h_, &v));
  return v;
}

QAP_API const CoefficientStore& AscentEngine::store() const {
  if (!st_ok_) {
    st_.m = m_;
    if (st_.idx.m != m_) st_.idx = StoreIndex(m_);
    st_.b.resize((size_t)m_ * m_);
    st_.c.resize(nc_of(m_));
    st_.d.resize(nd_of(m_));
    check(qapb_engine_get_array(h_, QAPB_ARR_STORE_B, st_.b.data(), st_.b.size()));
    check(qapb_engine_get_array(h_, QAPB_ARR_STORE_C, st_.c.data(), st_.c.size()));
    check(qapb_engine_get_array(h_, QAPB_ARR_STORE_D, st_.d.data(), st_.d.size()));
    check(qapb_engine_store_offset(h_, &st_.offset));
    st_ok_ = true;
  }
  return st_;
}

QAP_API CoefficientStore AscentEngine::snapshot() const {
  CoefficientStore s;
  s.m = m_;
  s.idx = StoreIndex(m_);
  s.b.resize((size_t)m_ * m_);
  s.c.resize(nc_of(m_));
  s.d.resize(nd_of(m_));
  check(qapb_engine_snapshot(h_, s.b.data(), s.c.data(), s.d.data(), &s.offset));
  return s;
}

QAP_API bool AscentEngine::has_certificate() const { return !certificate().empty(); }

QAP_API const std::vector<int>& AscentEngine::certificate() const {
  if (!cert_ok_) {
    int has = 0;
    double v = 0;
    std::vector<int> p(m_, -1);
    check(qapb_engine_certificate(h_, &has, p.data(), &v));
    cert_ = has ? p : std::vector<int>{};
    cert_ok_ = true;
  }
  return cert_;
}

QAP_API double AscentEngine::certificate_value() const {
  int has = 0;
  double v = 0;
  check(qapb_engine_certificate(h_, &has, nullptr, &v));
  return v;
}

QAP_API const std::vector<int>& AscentEngine::x_assignment() const {
  if (!x_ok_) {
    xrow_.assign(m_, -1);
    check(qapb_engine_x_assignment(h_, xrow_.data()));
    x_ok_ = true;
  }
  return xrow_;
}

namespace {
const std::vector<double>& fetch(qapb_engine* h, int which, std::vector<double>& dst, bool& ok) {
  if (!ok) {
    size_t n = 0;
    check(qapb_engine_array_size(h, which, &n));
    dst.resize(n);
    if (n) check(qapb_engine_get_array(h, which, dst.data(), n));
    ok = true;
  }
  return dst;
}
}  // namespace

QAP_API const std::vector<double>& AscentEngine::pi_z() const {
  return fetch(h_, QAPB_ARR_PI_Z, piz_, piz_ok_);
}
QAP_API const std::vector<double>& AscentEngine::pi_y() const {
  return fetch(h_, QAPB_ARR_PI_Y, piy_, piy_ok_);
}
QAP_API const std::vector<double>& AscentEngine::pi_x() const {
  return fetch(h_, QAPB_ARR_PI_X, pix_, pix_ok_);
}

QAP_API BoundReport run_ascent(const QapInstance& inst, const AscentConfig& cfg) {
  if (inst.n < 3) throw std::invalid_argument("init_coefficients: n >= 3 required by RLT2");
  const qapb_config c = to_c(cfg);
  std::vector<qapb_record> recs(std::max(1, cfg.iter_limit));
  std::vector<int> cert(inst.n, -1);
  qapb_report r{};
  const double* lin = inst.linear.empty() ? nullptr : inst.linear.data();
  check(qapb_run_ascent(inst.n, inst.flow.data(), inst.dist.data(), lin, &c, &r, recs.data(),
                        (int)recs.size(), cert.data()));
  BoundReport rep = report_from(r, recs, cert, cfg);
  rep.instance = inst.name;
  if (!rep.certificate.empty()) rep.certificate_value = evaluate_objective(inst, rep.certificate);
  return rep;
}

QAP_API BoundReport run_ascent_warm(CoefficientStore warm, const AscentConfig& cfg) {
  AscentEngine eng(std::move(warm), cfg);
  return eng.run();
}

QAP_API std::string BoundReport::to_json() const {
  std::ostringstream o;
  o.precision(17);
  auto num = [&](double v) {
    std::ostringstream t;
    t.precision(17);
    t << v;
    return t.str();
  };
  o << "{\n  \"instance\": \"" << instance << "\",\n  \"variant\": \"" << variant
    << "\",\n  \"sa_enabled\": " << (sa_enabled ? "true" : "false")
    << ",\n  \"best_bound\": " << num(best_bound);
  if (std::isfinite(upper_bound)) o << ",\n  \"upper_bound\": " << num(upper_bound);
  if (std::isfinite(gap)) o << ",\n  \"gap\": " << num(gap);
  o << ",\n  \"termination\": \"" << termination << "\",\n  \"iterations\": " << iterations
    << ",\n  \"wall_ms\": " << num(wall_ms);
  if (!certificate.empty()) {
    o << ",\n  \"certificate\": [";
    for (size_t i = 0; i < certificate.size(); ++i) o << (i ? ", " : "") << certificate[i];
    o << "],\n  \"certificate_value\": " << num(certificate_value);
  }
  o << ",\n  \"records\": [";
  for (size_t k = 0; k < records.size(); ++k) {
    const auto& r = records[k];
    o << (k ? "," : "") << "\n    {\"m\": " << r.iteration << ", \"bound\": " << num(r.bound)
      << ", \"gap\": " << num(std::isfinite(r.gap) ? r.gap : -1.0) << ", \"z_ms\": " << num(r.z_ms)
      << ", \"y_ms\": " << num(r.y_ms) << ", \"x_ms\": " << num(r.x_ms) << "}";
  }
  o << (records.empty() ? "]" : "\n  ]") << "\n}";
  return o.str();
}

QAP_API std::string BoundReport::to_csv() const {
  std::ostringstream out;
  out << "iteration,bound,gap,z_ms,y_ms,x_ms\n";
  for (const auto& r : records)
    out << r.iteration << ',' << r.bound << ',' << (std::isfinite(r.gap) ? r.gap : -1.0) << ','
        << r.z_ms << ',' << r.y_ms << ',' << r.x_ms << "\n";
  return out.str();
}

}  // namespace qap

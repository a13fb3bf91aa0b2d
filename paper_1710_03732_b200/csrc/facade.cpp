// facade.cpp — the reference's C++ API (include/qap/{instance,lap,rlt2}.hpp)
// implemented over the C-ABI (include/qapb200.h).  This is the binding a
// maintainer swaps in for proj/src/{lap,rlt2}.cpp: callers (bnb.cpp,
// qap_cli.cpp, the reference's unit tests) compile unchanged against these
// headers and link libqapb200.so.  Status codes become the reference's
// exception types again.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
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
// QAPB_FACADE_STATS=1: wall time spent per facade call kind, summed over
// all threads, printed to stderr at exit (where a branch-and-bound spends its
// node time).  Off: one getenv per process.
namespace {
enum StatKind { kStCollapse, kStEngine, kStRun, kStSnapshot, kStInit, kStKinds };
struct FacadeStats {
  std::atomic<long long> ns[kStKinds]{};
  std::atomic<long long> calls[kStKinds]{};
  std::atomic<long long> iterations{0};
  bool on = std::getenv("QAPB_FACADE_STATS") != nullptr;
  ~FacadeStats() {
    if (!on) return;
    static const char* names[kStKinds] = {"collapse_store", "AscentEngine()", "run()",
                                          "snapshot()", "init_coefficients"};
    for (int k = 0; k < kStKinds; ++k)
      std::fprintf(stderr, "qapb facade: %-18s calls %8lld  total %9.3f s  mean %8.3f ms\n",
                   names[k], calls[k].load(), ns[k].load() * 1e-9,
                   calls[k] ? ns[k].load() * 1e-6 / calls[k].load() : 0.0);
    std::fprintf(stderr, "qapb facade: iterations %lld\n", iterations.load());
  }
};
FacadeStats g_stats;
struct StatTimer {
  StatKind k;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit StatTimer(StatKind kind) : k(kind) {}
  ~StatTimer() {
    if (!g_stats.on) return;
    g_stats.ns[k] += std::chrono::duration_cast<std::chrono::nanoseconds>(
                         std::chrono::steady_clock::now() - t0).count();
    ++g_stats.calls[k];
  }
};
}  // namespace

namespace {

void check(qapb_status rc) {
  if (rc == QAPB_OK) return;
  const std::string msg = qapb_last_error();
  // bnb.cpp's bank threads do not catch: QAPB_LOG_ERRORS=1 names the error
  // before std::terminate hides it
  if (std::getenv("QAPB_LOG_ERRORS")) std::fprintf(stderr, "qapb error %d: %s\n", (int)rc, msg.c_str());
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
// QAPLIB I/O, generators and manifests (instance.hpp) are outside the
// drop-in boundary: they stay the reference's own
// src/instance.cpp, linked next to this library.  The
// engine needs only the objective of a certificate (run_ascent,
// rlt2.cpp:594-595), summed in the reference's order (instance.cpp:11-26:
// per facility, the linear term, then its row of flow x distance products).
namespace {
double certificate_objective(const QapInstance& inst, const std::vector<int>& perm) {
  const int n = inst.n;
  const bool lin = !inst.linear.empty();
  double sum = 0;
  for (int i = 0; i < n; ++i) {
    const int pi = perm[i];
    sum += lin ? inst.linear[(size_t)i * n + pi] : 0.0;
    const double* frow = inst.flow.data() + (size_t)i * n;
    const double* drow = inst.dist.data() + (size_t)pi * n;
    for (int j = 0; j < n; ++j) sum += frow[j] * drow[perm[j]];
  }
  return sum;
}
}  // namespace

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

namespace {
int bank_device(int requested);

std::shared_ptr<qapb_store> own_store(qapb_store* p) {
  return std::shared_ptr<qapb_store>(p, [](qapb_store* q) { qapb_store_destroy(q); });
}

// A store in HBM with host-empty b, c, d (rlt2.hpp CoefficientStore::device)
CoefficientStore device_store(qapb_store* p, int m, double offset) {
  CoefficientStore st;
  st.m = m;
  st.idx = StoreIndex(m);
  st.offset = offset;
  st.device = own_store(p);
  return st;
}

// the store as a device store (uploads a host store)
std::shared_ptr<qapb_store> on_device(const CoefficientStore& st, int device) {
  if (st.device) return st.device;
  qapb_store* p = nullptr;
  check(qapb_store_upload(st.m, st.b.data(), st.c.data(), st.m >= 3 ? st.d.data() : nullptr,
                          st.offset, device, &p));
  return own_store(p);
}
}  // namespace

// rlt2.cpp:66-89: built in HBM by the init kernel (D' = 0), kept there
QAP_API CoefficientStore init_coefficients(const QapInstance& inst) {
  StatTimer timer(kStInit);
  if (inst.n < 3) throw std::invalid_argument("init_coefficients: n >= 3 required by RLT2");
  const double* lin = inst.linear.empty() ? nullptr : inst.linear.data();
  qapb_store* p = nullptr;
  check(qapb_store_init(inst.n, inst.flow.data(), inst.dist.data(), lin, bank_device(0), &p));
  return device_store(p, inst.n, 0.0);
}

QAP_API CoefficientStore& host_view(CoefficientStore& st) {
  if (!st.device) return st;
  st.b.resize((size_t)st.m * st.m);
  st.c.resize(nc_of(st.m));
  st.d.resize(nd_of(st.m));
  double off = 0;
  check(qapb_store_download(st.device.get(), st.b.data(), st.c.data(), st.d.data(), &off));
  return st;
}

// rlt2.cpp:91-107, on the device (terms in the reference's order)
QAP_API double store_evaluate(const CoefficientStore& st, const std::vector<int>& perm) {
  double v = 0;
  if (st.device) {
    check(qapb_store_evaluate_device(st.device.get(), st.offset, perm.data(), &v));
  } else {
    check(qapb_store_evaluate(st.m, st.b.data(), st.c.data(), st.d.data(), st.offset,
                              perm.data(), &v));
  }
  return v;
}

// rlt2.cpp:109-182, device to device; the child stays in HBM
QAP_API CoefficientStore collapse_store(const CoefficientStore& st, int fac, int loc) {
  StatTimer timer(kStCollapse);
  const int mc = st.m - 1;
  if (mc < 2) throw std::invalid_argument("collapse_store: store too small");
  std::shared_ptr<qapb_store> src = on_device(st, bank_device(0));
  qapb_store* p = nullptr;
  check(qapb_store_collapse_offset(src.get(), st.offset, fac, loc, &p));
  int m = 0;
  double off = 0;
  check(qapb_store_info(p, &m, &off));  // st.offset + b[fac, loc] (rlt2.cpp:116)
  return device_store(p, mc, off);
}

QAP_API bool redistribute_family(const double pi[3], double add[3], int virtual_slots,
                                 double tol) {
  int ok = 0;
  check(qapb_redistribute_family(pi, add, virtual_slots, tol, &ok));
  return ok != 0;
}

// Bank-per-GPU placement (the reference's banks are threads,
// bnb.cpp:549-556).  With QAPB_BANK_GPUS=N (N > 1, or "all"), every thread that
// builds engines on the default device 0 is pinned to one of the first N visible
// GPUs, round-robin in order of first use, so the reference's branch-and-bound
// spreads its banks over the node without a source change.  Unset: device 0.
namespace {
int bank_device(int requested) {
  if (requested != 0) return requested;
  const char* e = std::getenv("QAPB_BANK_GPUS");
  if (!e || !*e) return 0;
  int visible = 0;
  if (qapb_device_count(&visible) != QAPB_OK || visible < 1) return 0;
  const int want = std::strcmp(e, "all") == 0 ? visible : std::atoi(e);
  const int n = std::max(1, std::min(want, visible));
  static std::atomic<int> next{0};
  thread_local int dev = -1;
  if (dev < 0) {
    dev = next.fetch_add(1) % n;
    if (std::getenv("QAPB_BANK_GPUS_VERBOSE"))
      std::fprintf(stderr, "qapb: engine thread placed on device %d of %d\n", dev, n);
  }
  return dev;
}
}  // namespace

QAP_API AscentEngine::AscentEngine(CoefficientStore store, const AscentConfig& cfg)
    : cfg_(cfg), m_(store.m) {
  StatTimer timer(kStEngine);
  if (m_ < 3) throw std::invalid_argument("AscentEngine: m >= 3 required");
  cfg_.device = bank_device(cfg.device);
  const qapb_config c = to_c(cfg_);
  if (store.device) {  // device-to-device (snapshots, collapsed children, init_coefficients)
    int dev = -1;
    check(qapb_store_device(store.device.get(), &dev));
    if (dev == cfg_.device) {
      check(qapb_engine_create_from_store_offset(store.device.get(), store.offset, &c, &h_));
      return;
    }
    host_view(store);  // another GPU: through the host
  }
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
  StatTimer timer(kStRun);
  invalidate();
  std::vector<qapb_record> recs(std::max(1, cfg_.iter_limit));
  std::vector<int> cert(m_, -1);
  qapb_report r{};
  check(qapb_engine_run(h_, &r, recs.data(), (int)recs.size(), cert.data()));
  if (g_stats.on) g_stats.iterations += r.iterations;
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

// rlt2.cpp:537-542, kept in HBM (std::logic_error for F variants).  A search
// tree can hold many snapshots at once (bnb.cpp keeps each branching node's
// store for its children, also while they wait in the master heap): when the
// device has less than a quarter of its memory free, the snapshot goes to the
// host instead (host-resident store; collapse_store uploads it again).
QAP_API CoefficientStore AscentEngine::snapshot() const {
  StatTimer timer(kStSnapshot);
  size_t free_b = 0, total_b = 0;
  check(qapb_device_memory(cfg_.device, &free_b, &total_b));
  const size_t need = (nc_of(m_) + nd_of(m_) + (size_t)m_ * m_) * sizeof(double);
  if (free_b < total_b / 4 + need || std::getenv("QAPB_SNAPSHOT_HOST")) {
    CoefficientStore s;
    s.m = m_;
    s.idx = StoreIndex(m_);
    s.b.resize((size_t)m_ * m_);
    s.c.resize(nc_of(m_));
    s.d.resize(nd_of(m_));
    check(qapb_engine_snapshot(h_, s.b.data(), s.c.data(), s.d.data(), &s.offset));
    return s;
  }
  qapb_store* p = nullptr;
  check(qapb_store_from_engine(h_, &p));
  int m = 0;
  double off = 0;
  check(qapb_store_info(p, &m, &off));
  return device_store(p, m, off);
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
  if (!rep.certificate.empty())
    rep.certificate_value = certificate_objective(inst, rep.certificate);
  return rep;
}

QAP_API BoundReport run_ascent_warm(CoefficientStore warm, const AscentConfig& cfg) {
  AscentEngine eng(std::move(warm), cfg);
  return eng.run();
}

// ---- BoundReport::to_json, byte-identical to the reference's (rlt2.cpp:604-630,
// nlohmann::json::dump(2)): object keys in sorted order (std::map), 2-space
// indent, integers as integers, doubles as nlohmann's Grisu2 digits in its
// layout (digits[.0] up to 10^15, 0.000ddd down to 1e-4, d.ddde+XX
// otherwise), non-finite as null, strings escaped as nlohmann does.
namespace {

// Shortest-digit conversion of nlohmann/json (the reference's vendored
// serializer, absent from /root/reference): Grisu2 (F. Loitsch, "Printing
// Floating-Point Numbers Quickly and Accurately with Integers", PLDI 2010)
// with alpha = -60, gamma = -32, cached powers 10^(-300 + 8i) and the
// "round toward w" step, then nlohmann's layout rules.  Grisu2 is not always
// the shortest or the closest representation, so std::to_chars would differ
// from the reference in ~0.5% of values.
struct DiyFp {
  std::uint64_t f;
  int e;
};

DiyFp diy_mul(DiyFp x, DiyFp y) {  // upper 64 bits of the 128-bit product, rounded
  const std::uint64_t u_lo = x.f & 0xFFFFFFFFu, u_hi = x.f >> 32;
  const std::uint64_t v_lo = y.f & 0xFFFFFFFFu, v_hi = y.f >> 32;
  const std::uint64_t p0 = u_lo * v_lo, p1 = u_lo * v_hi, p2 = u_hi * v_lo, p3 = u_hi * v_hi;
  std::uint64_t q = (p0 >> 32) + (p1 & 0xFFFFFFFFu) + (p2 & 0xFFFFFFFFu);
  q += std::uint64_t{1} << 31;
  return {p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32), x.e + y.e + 64};
}

DiyFp diy_normalize(DiyFp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

struct CachedPow {
  std::uint64_t f;
  int e, k;
};

const CachedPow kCachedPows[79] = {
    {0xAB70FE17C79AC6CAull, -1060, -300},
    {0xFF77B1FCBEBCDC4Full, -1034, -292},
    {0xBE5691EF416BD60Cull, -1007, -284},
    {0x8DD01FAD907FFC3Cull, -980, -276},
    {0xD3515C2831559A83ull, -954, -268},
    {0x9D71AC8FADA6C9B5ull, -927, -260},
    {0xEA9C227723EE8BCBull, -901, -252},
    {0xAECC49914078536Dull, -874, -244},
    {0x823C12795DB6CE57ull, -847, -236},
    {0xC21094364DFB5637ull, -821, -228},
    {0x9096EA6F3848984Full, -794, -220},
    {0xD77485CB25823AC7ull, -768, -212},
    {0xA086CFCD97BF97F4ull, -741, -204},
    {0xEF340A98172AACE5ull, -715, -196},
    {0xB23867FB2A35B28Eull, -688, -188},
    {0x84C8D4DFD2C63F3Bull, -661, -180},
    {0xC5DD44271AD3CDBAull, -635, -172},
    {0x936B9FCEBB25C996ull, -608, -164},
    {0xDBAC6C247D62A584ull, -582, -156},
    {0xA3AB66580D5FDAF6ull, -555, -148},
    {0xF3E2F893DEC3F126ull, -529, -140},
    {0xB5B5ADA8AAFF80B8ull, -502, -132},
    {0x87625F056C7C4A8Bull, -475, -124},
    {0xC9BCFF6034C13053ull, -449, -116},
    {0x964E858C91BA2655ull, -422, -108},
    {0xDFF9772470297EBDull, -396, -100},
    {0xA6DFBD9FB8E5B88Full, -369, -92},
    {0xF8A95FCF88747D94ull, -343, -84},
    {0xB94470938FA89BCFull, -316, -76},
    {0x8A08F0F8BF0F156Bull, -289, -68},
    {0xCDB02555653131B6ull, -263, -60},
    {0x993FE2C6D07B7FACull, -236, -52},
    {0xE45C10C42A2B3B06ull, -210, -44},
    {0xAA242499697392D3ull, -183, -36},
    {0xFD87B5F28300CA0Eull, -157, -28},
    {0xBCE5086492111AEBull, -130, -20},
    {0x8CBCCC096F5088CCull, -103, -12},
    {0xD1B71758E219652Cull, -77, -4},
    {0x9C40000000000000ull, -50, 4},
    {0xE8D4A51000000000ull, -24, 12},
    {0xAD78EBC5AC620000ull, 3, 20},
    {0x813F3978F8940984ull, 30, 28},
    {0xC097CE7BC90715B3ull, 56, 36},
    {0x8F7E32CE7BEA5C70ull, 83, 44},
    {0xD5D238A4ABE98068ull, 109, 52},
    {0x9F4F2726179A2245ull, 136, 60},
    {0xED63A231D4C4FB27ull, 162, 68},
    {0xB0DE65388CC8ADA8ull, 189, 76},
    {0x83C7088E1AAB65DBull, 216, 84},
    {0xC45D1DF942711D9Aull, 242, 92},
    {0x924D692CA61BE758ull, 269, 100},
    {0xDA01EE641A708DEAull, 295, 108},
    {0xA26DA3999AEF774Aull, 322, 116},
    {0xF209787BB47D6B85ull, 348, 124},
    {0xB454E4A179DD1877ull, 375, 132},
    {0x865B86925B9BC5C2ull, 402, 140},
    {0xC83553C5C8965D3Dull, 428, 148},
    {0x952AB45CFA97A0B3ull, 455, 156},
    {0xDE469FBD99A05FE3ull, 481, 164},
    {0xA59BC234DB398C25ull, 508, 172},
    {0xF6C69A72A3989F5Cull, 534, 180},
    {0xB7DCBF5354E9BECEull, 561, 188},
    {0x88FCF317F22241E2ull, 588, 196},
    {0xCC20CE9BD35C78A5ull, 614, 204},
    {0x98165AF37B2153DFull, 641, 212},
    {0xE2A0B5DC971F303Aull, 667, 220},
    {0xA8D9D1535CE3B396ull, 694, 228},
    {0xFB9B7CD9A4A7443Cull, 720, 236},
    {0xBB764C4CA7A44410ull, 747, 244},
    {0x8BAB8EEFB6409C1Aull, 774, 252},
    {0xD01FEF10A657842Cull, 800, 260},
    {0x9B10A4E5E9913129ull, 827, 268},
    {0xE7109BFBA19C0C9Dull, 853, 276},
    {0xAC2820D9623BF429ull, 880, 284},
    {0x80444B5E7AA7CF85ull, 907, 292},
    {0xBF21E44003ACDD2Dull, 933, 300},
    {0x8E679C2F5E44FF8Full, 960, 308},
    {0xD433179D9C8CB841ull, 986, 316},
    {0x9E19DB92B4E31BA9ull, 1013, 324},
};

int find_largest_pow10(std::uint32_t n, std::uint32_t& pow10) {
  static const std::uint32_t p[10] = {1,      10,      100,      1000,      10000,
                                      100000, 1000000, 10000000, 100000000, 1000000000};
  int k = 10;
  while (k > 1 && n < p[k - 1]) --k;
  pow10 = p[k - 1];
  return k;
}

void grisu2_round(char* buf, int len, std::uint64_t dist, std::uint64_t delta, std::uint64_t rest,
                  std::uint64_t ten_k) {
  // move the last digit down while that brings the value closer to w
  while (rest < dist && delta - rest >= ten_k &&
         (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf[len - 1]--;
    rest += ten_k;
  }
}

// digits of some V in [M-, M+] (all three share the exponent e, -60 <= e <= -32)
void grisu2_digits(char* buf, int& len, int& dexp, DiyFp Mm, DiyFp w, DiyFp Mp) {
  std::uint64_t delta = Mp.f - Mm.f;
  std::uint64_t dist = Mp.f - w.f;
  const int sh = -Mp.e;
  const std::uint64_t one = std::uint64_t{1} << sh;
  auto p1 = static_cast<std::uint32_t>(Mp.f >> sh);
  std::uint64_t p2 = Mp.f & (one - 1);
  std::uint32_t pow10 = 0;
  int n = find_largest_pow10(p1, pow10);
  while (n > 0) {
    const std::uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[len++] = static_cast<char>('0' + d);
    p1 = r;
    --n;
    const std::uint64_t rest = (std::uint64_t{p1} << sh) + p2;
    if (rest <= delta) {
      dexp += n;
      grisu2_round(buf, len, dist, delta, rest, std::uint64_t{pow10} << sh);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    const std::uint64_t d = p2 >> sh, r = p2 & (one - 1);
    buf[len++] = static_cast<char>('0' + d);
    p2 = r;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dexp -= m;
  grisu2_round(buf, len, dist, delta, p2, one);
}

// v > 0 finite -> digits in buf, value = digits * 10^dexp
void grisu2(char* buf, int& len, int& dexp, double v) {
  std::uint64_t bits;
  std::memcpy(&bits, &v, sizeof bits);
  const std::uint64_t E = bits >> 52, F = bits & ((std::uint64_t{1} << 52) - 1);
  const DiyFp x = E == 0 ? DiyFp{F, 1 - 1075} : DiyFp{F + (std::uint64_t{1} << 52), (int)E - 1075};
  const bool lower_closer = F == 0 && E > 1;
  const DiyFp mp = diy_normalize(DiyFp{2 * x.f + 1, x.e - 1});
  DiyFp mm = lower_closer ? DiyFp{4 * x.f - 1, x.e - 2} : DiyFp{2 * x.f - 1, x.e - 1};
  mm = DiyFp{mm.f << (mm.e - mp.e), mp.e};
  const DiyFp w = diy_normalize(x);
  // cached power c = 10^-k with -60 <= e_c + mp.e + 64 <= -32
  const int f = -60 - mp.e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
  const CachedPow& c = kCachedPows[(300 + k + 7) / 8];
  const DiyFp ck{c.f, c.e};
  const DiyFp W = diy_mul(w, ck), Wm = diy_mul(mm, ck), Wp = diy_mul(mp, ck);
  dexp = -c.k;
  len = 0;
  grisu2_digits(buf, len, dexp, DiyFp{Wm.f + 1, Wm.e}, W, DiyFp{Wp.f - 1, Wp.e});
}

std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  std::string out;
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0) return out + "0.0";
  char dig[32];
  int k = 0, dexp = 0;
  grisu2(dig, k, dexp, v);
  const std::string digits(dig, dig + k);
  const int n = k + dexp;  // value = 0.d1d2... x 10^n
  if (k <= n && n <= 15) {
    out += digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int x = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
    out += eb;
  }
  return out;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char ch : s) {
    switch (ch) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (ch < 0x20) {
          char u[8];
          std::snprintf(u, sizeof u, "\\u%04x", ch);
          o += u;
        } else {
          o += (char)ch;
        }
    }
  }
  return o + "\"";
}

// one "key": value member per line at the given indent, keys sorted
std::string json_object(const std::vector<std::pair<std::string, std::string>>& kv, int ind) {
  if (kv.empty()) return "{}";
  auto sorted = kv;
  std::sort(sorted.begin(), sorted.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  const std::string pad(ind + 2, ' ');
  std::string o = "{\n";
  for (size_t i = 0; i < sorted.size(); ++i)
    o += pad + json_string(sorted[i].first) + ": " + sorted[i].second +
         (i + 1 < sorted.size() ? ",\n" : "\n");
  return o + std::string(ind, ' ') + "}";
}

std::string json_array(const std::vector<std::string>& items, int ind) {
  if (items.empty()) return "[]";
  const std::string pad(ind + 2, ' ');
  std::string o = "[\n";
  for (size_t i = 0; i < items.size(); ++i)
    o += pad + items[i] + (i + 1 < items.size() ? ",\n" : "\n");
  return o + std::string(ind, ' ') + "]";
}

}  // namespace

QAP_API std::string BoundReport::to_json() const {
  std::vector<std::pair<std::string, std::string>> kv;
  kv.emplace_back("instance", json_string(instance));
  kv.emplace_back("variant", json_string(variant));
  kv.emplace_back("sa_enabled", sa_enabled ? "true" : "false");
  kv.emplace_back("best_bound", json_double(best_bound));
  if (std::isfinite(upper_bound)) kv.emplace_back("upper_bound", json_double(upper_bound));
  if (std::isfinite(gap)) kv.emplace_back("gap", json_double(gap));
  kv.emplace_back("termination", json_string(termination));
  kv.emplace_back("iterations", std::to_string(iterations));
  kv.emplace_back("wall_ms", json_double(wall_ms));
  if (!certificate.empty()) {
    std::vector<std::string> c;
    for (int x : certificate) c.push_back(std::to_string(x));
    kv.emplace_back("certificate", json_array(c, 2));
    kv.emplace_back("certificate_value", json_double(certificate_value));
  }
  std::vector<std::string> recs;
  for (const auto& r : records)
    recs.push_back(json_object({{"m", std::to_string(r.iteration)},
                                {"bound", json_double(r.bound)},
                                {"gap", json_double(std::isfinite(r.gap) ? r.gap : -1.0)},
                                {"z_ms", json_double(r.z_ms)},
                                {"y_ms", json_double(r.y_ms)},
                                {"x_ms", json_double(r.x_ms)}},
                               4));
  kv.emplace_back("records", json_array(recs, 2));
  return json_object(kv, 0);
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

// BoundReport::to_json through the C-ABI (tests compare it byte for byte with
// the reference's nlohmann output).  recs: 6 doubles per record (iteration,
// bound, gap, z_ms, y_ms, x_ms).
extern "C" QAP_API int qapb_report_json(const char* instance, const char* variant, int sa_enabled,
                                        double best_bound, double upper_bound, double gap,
                                        const char* termination, int iterations, double wall_ms,
                                        const int* cert, int ncert, double cert_value,
                                        const double* recs, int nrec, char* out, size_t cap,
                                        size_t* len) {
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
  r.certificate.assign(cert, cert + (cert ? ncert : 0));
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
  if (!out || cap <= j.size()) return QAPB_EINVAL;
  std::memcpy(out, j.c_str(), j.size() + 1);
  return QAPB_OK;
}


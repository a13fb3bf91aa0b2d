// capi.cu — the C-ABI (include/qapb200.h) over the device engine.
//
// Exceptions never cross the boundary: each entry point maps the C++
// exception type the reference would throw (SURVEY.md §8b "Errors") onto a
// status code and a thread-local message.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qapb200.h"
#include "engine.h"
#include "nccl_dyn.h"
#include "kernels.h"
#include "store.h"

using qapb::CudaError;
using qapb::Engine;
using qapb::DeviceStore;
using qapb::collapse_store_device;
using qapb::store_nb;
using qapb::store_nc;
using qapb::store_nd;

namespace qapb {
std::vector<int> shard_plan(int n, int world);
void shard_counts(int n, const std::vector<int>& ab, int rank, std::vector<long long>& send,
                  std::vector<long long>& recv);
}  // namespace qapb

struct qapb_engine {
  std::unique_ptr<Engine> e;
};
struct qapb_store {
  std::unique_ptr<qapb::DeviceStore> s;
};

namespace {
thread_local std::string g_err;

// Debugging aid (QAPB_SERIALIZE=1): one C-ABI call at a time in the process,
// so concurrent callers (branch-and-bound banks) cannot interleave GPU work.
std::recursive_mutex& serial_mutex() {
  static std::recursive_mutex mu;
  return mu;
}
bool serialize_calls() {
  static const bool on = std::getenv("QAPB_SERIALIZE") != nullptr;
  return on;
}

template <class F>
qapb_status guard(F&& f) {
  std::unique_lock<std::recursive_mutex> lk(serial_mutex(), std::defer_lock);
  if (serialize_calls()) lk.lock();
  try {
    f();
    return QAPB_OK;
  } catch (const CudaError& e) {
    g_err = e.what();
    return QAPB_ECUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return QAPB_EINVAL;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return QAPB_ELOGIC;
  } catch (const std::bad_alloc& e) {
    g_err = "out of host memory";
    return QAPB_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QAPB_ERUNTIME;
  }
}

void cuda_check_set(int device) {
  if (cudaSetDevice(device) != cudaSuccess) throw CudaError("cudaSetDevice failed");
}

void need(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

size_t nb_of(int m) { return (size_t)m * m; }
size_t nc_of(int m) { return (size_t)m * m * (m - 1) * (m - 1); }
size_t nd_of(int m) { return store_nd(m); }
}  // namespace

namespace {
// stream-ordered device buffer, freed on every exit path
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DevBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) qapb::cuda_check(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync");
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};
constexpr int kNoSlot = 0x7f7f7f7f;  // memset(0x7f) sentinel: no undefined slot
}  // namespace

extern "C" {

QAPB_API const char* qapb_last_error(void) { return g_err.c_str(); }
QAPB_API int qapb_abi_version(void) { return 1; }

QAPB_API void qapb_config_init(qapb_config* c) {  // rlt2.hpp:98-121
  std::memset(c, 0, sizeof *c);
  c->variant = QAPB_F1;
  c->sa_enabled = 0;
  c->iter_limit = 100;
  c->min_gap = 0.0;
  c->kappa_z_upper = 2.0 / 3.0;
  c->phi_split = 0.5;
  c->kappa_y = 1.0;
  c->kappa_x = 1.0;
  c->varphi = 0.5;
  c->sa_t0_fraction = 0.04;
  c->sa_kappa_lb_cap = 0.25;
  c->sa_cool_factor = 0.99;
  c->sa_cool_period = 100;
  c->workers = 1;
  c->seed = 0;
  c->upper_bound = std::numeric_limits<double>::infinity();
  c->fathom_threshold = std::numeric_limits<double>::infinity();
  c->early_stop_window = 0;
  c->early_stop_delta = 0.0002;
  c->record_history = 1;
  c->device = 0;
}

QAPB_API qapb_status qapb_device_count(int* count) {
  return guard([&] { qapb::cuda_check(cudaGetDeviceCount(count), "cudaGetDeviceCount"); });
}

QAPB_API const char* qapb_variant_name(int v) {  // rlt2.cpp:24-32
  switch (v) {
    case QAPB_F1: return "F1";
    case QAPB_F2: return "F2";
    case QAPB_S1: return "S1";
    case QAPB_S2: return "S2";
  }
  return "?";
}

QAPB_API qapb_status qapb_parse_variant(const char* s, int* variant) {  // rlt2.cpp:34-42
  return guard([&] {
    std::string t;
    for (const char* p = s; *p; ++p) t += (char)std::toupper((unsigned char)*p);
    if (t == "F1") *variant = QAPB_F1;
    else if (t == "F2") *variant = QAPB_F2;
    else if (t == "S1") *variant = QAPB_S1;
    else if (t == "S2") *variant = QAPB_S2;
    else throw std::invalid_argument("unknown variant: " + std::string(s));
  });
}

// ---- LAP ---------------------------------------------------------------

// lap.cpp:104-138 over device pointers.  Any m: m <= lap_max_m() runs the
// warp-per-LAP solver, larger m one CTA per LAP.  Returns after the batch has
// completed on `stream` (the undefined-slot check reads a device flag).
QAPB_API qapb_status qapb_lap_solve_batch_device(const double* costs, int m, int count,
                                                 double* values, int* r2c, int* c2r, double* u,
                                                 double* v, void* stream) {
  return guard([&] {
    need(m > 0, "lap: m must be positive");  // lap.cpp:26
    need(count >= 0, "lap: count must be non-negative");
    if (count == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DevBuf flags(2 * sizeof(int), st);
    int* counter = flags.as<int>();
    qapb::cuda_check(cudaMemsetAsync(counter, 0, sizeof(int), st), "memset");
    qapb::cuda_check(cudaMemsetAsync(counter + 1, 0x7f, sizeof(int), st), "memset");
    qapb::BatchLapParams p{};
    p.costs = costs;
    p.m = m;
    p.count = count;
    p.counter = counter;
    p.undefined = counter + 1;
    p.values = values;
    p.r2c = r2c;
    p.c2r = c2r;
    p.u = u;
    p.v = v;
    qapb::cuda_check(qapb::launch_lap_batch(p, st), "lap batch");
    int und = kNoSlot;
    qapb::cuda_check(cudaMemcpyAsync(&und, counter + 1, sizeof(int), cudaMemcpyDeviceToHost, st),
                     "D2H");
    qapb::cuda_check(cudaStreamSynchronize(st), "lap batch");
    if (und != kNoSlot)
      throw std::invalid_argument("lap: slot " + std::to_string(und) +
                                  " has no finite-cost column to extend the assignment "
                                  "(undefined in LapSolver::solve, lap.cpp:53)");
  });
}

QAPB_API qapb_status qapb_lap_solve_batch(const double* costs, int m, int count, double* values,
                                          int* r2c, int* c2r, double* u, double* v) {
  return guard([&] {
    need(m > 0, "lap: m must be positive");
    need(count >= 0, "lap: count must be non-negative");
    if (count == 0) return;
    cudaStream_t st = cudaStreamPerThread;
    const size_t nc = (size_t)count * m * m, nv = (size_t)count * m;
    DevBuf dc(nc * 8, st), dval(values ? count * 8 : 0, st), du(u ? nv * 8 : 0, st),
        dv(v ? nv * 8 : 0, st), dr(r2c ? nv * 4 : 0, st), dcr(c2r ? nv * 4 : 0, st);
    qapb::cuda_check(cudaMemcpyAsync(dc.p, costs, nc * 8, cudaMemcpyHostToDevice, st), "H2D");
    const qapb_status rc = qapb_lap_solve_batch_device(
        dc.as<double>(), m, count, dval.as<double>(), dr.as<int>(), dcr.as<int>(),
        du.as<double>(), dv.as<double>(), st);
    if (rc == QAPB_EINVAL) throw std::invalid_argument(g_err);
    if (rc == QAPB_ECUDA) throw CudaError(g_err);
    if (rc) throw std::runtime_error(g_err);
    auto d2h = [&](void* dst, const DevBuf& src, size_t bytes) {
      if (dst) qapb::cuda_check(cudaMemcpyAsync(dst, src.p, bytes, cudaMemcpyDeviceToHost, st), "D2H");
    };
    d2h(values, dval, count * 8);
    d2h(u, du, nv * 8);
    d2h(v, dv, nv * 8);
    d2h(r2c, dr, nv * 4);
    d2h(c2r, dcr, nv * 4);
    qapb::cuda_check(cudaStreamSynchronize(st), "lap batch");
  });
}

QAPB_API qapb_status qapb_lap_solve(const double* cost, int m, int* r2c, int* c2r, double* u,
                                    double* v, double* value) {
  return qapb_lap_solve_batch(cost, m, 1, value, r2c, c2r, u, v);
}

// ---- store helpers -------------------------------------------------------
QAPB_API qapb_status qapb_init_coefficients(int n, const double* flow, const double* dist,
                                            const double* linear, double* b, double* c,
                                            double* d) {
  return guard([&] {
    need(n >= 3, "init_coefficients: n >= 3 required by RLT2");  // rlt2.cpp:67-68
    cudaStream_t st = cudaStreamPerThread;
    const size_t nn = (size_t)n * n;
    double *df, *dd, *dl = nullptr, *db, *dc;
    qapb::cuda_check(cudaMallocAsync((void**)&df, nn * 8, st), "alloc");
    qapb::cuda_check(cudaMallocAsync((void**)&dd, nn * 8, st), "alloc");
    if (linear) qapb::cuda_check(cudaMallocAsync((void**)&dl, nn * 8, st), "alloc");
    qapb::cuda_check(cudaMallocAsync((void**)&db, nb_of(n) * 8, st), "alloc");
    qapb::cuda_check(cudaMallocAsync((void**)&dc, nc_of(n) * 8, st), "alloc");
    cudaMemcpyAsync(df, flow, nn * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dd, dist, nn * 8, cudaMemcpyHostToDevice, st);
    if (linear) cudaMemcpyAsync(dl, linear, nn * 8, cudaMemcpyHostToDevice, st);
    qapb::cuda_check(qapb::launch_init_store(n, df, dd, dl, db, dc, st), "init_store");
    cudaMemcpyAsync(b, db, nb_of(n) * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(c, dc, nc_of(n) * 8, cudaMemcpyDeviceToHost, st);
    for (void* p : {(void*)df, (void*)dd, (void*)dl, (void*)db, (void*)dc})
      if (p) cudaFreeAsync(p, st);
    qapb::cuda_check(cudaStreamSynchronize(st), "init_coefficients");
    if (d) std::memset(d, 0, nd_of(n) * sizeof(double));
  });
}

// The reference's store helpers (store_evaluate, collapse_store,
// redistribute_family) run on the device (store.cu); host arrays are staged
// into a temporary device store on the calling thread's current device.
namespace {
int current_device() {
  int dev = 0;
  qapb::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  return dev;
}
std::unique_ptr<DeviceStore> stage_store(int m, const double* b, const double* c, const double* d,
                                         double offset) {
  auto s = std::make_unique<DeviceStore>(m, current_device());
  qapb::cuda_check(cudaMemcpyAsync(s->b, b, store_nb(m) * 8, cudaMemcpyDefault, s->stream), "H2D b");
  qapb::cuda_check(cudaMemcpyAsync(s->c, c, store_nc(m) * 8, cudaMemcpyDefault, s->stream), "H2D c");
  if (m >= 3 && d)
    qapb::cuda_check(cudaMemcpyAsync(s->d, d, store_nd(m) * 8, cudaMemcpyDefault, s->stream),
                     "H2D d");
  else if (m >= 3)
    qapb::cuda_check(cudaMemsetAsync(s->d, 0, store_nd(m) * 8, s->stream), "memset d");
  s->offset = offset;
  return s;
}
}  // namespace

// store_evaluate, rlt2.cpp:91-107 (device, qapb::store_evaluate_device)
QAPB_API qapb_status qapb_store_evaluate(int m, const double* b, const double* c,
                                         const double* d, double offset, const int* perm,
                                         double* value) {
  return guard([&] {
    need(m >= 3, "store_evaluate: m >= 3 required");
    auto s = stage_store(m, b, c, d, offset);
    *value = qapb::store_evaluate_device(*s, perm, s->offset);
  });
}

// collapse_store, rlt2.cpp:109-182 (device, qapb::collapse_store_device)
QAPB_API qapb_status qapb_collapse_store(int m, const double* b, const double* c,
                                         const double* d, double offset, int fac, int loc,
                                         double* ob, double* oc, double* od, double* ooffset) {
  return guard([&] {
    need(m - 1 >= 2, "collapse_store: store too small");  // rlt2.cpp:111
    auto s = stage_store(m, b, c, d, offset);
    auto o = collapse_store_device(*s, fac, loc);
    const int mc = m - 1;
    qapb::cuda_check(cudaMemcpyAsync(ob, o->b, store_nb(mc) * 8, cudaMemcpyDefault, o->stream), "D2H");
    qapb::cuda_check(cudaMemcpyAsync(oc, o->c, store_nc(mc) * 8, cudaMemcpyDefault, o->stream), "D2H");
    if (mc >= 3 && od)
      qapb::cuda_check(cudaMemcpyAsync(od, o->d, store_nd(mc) * 8, cudaMemcpyDefault, o->stream),
                       "D2H");
    o->synchronize();
    *ooffset = o->offset;
  });
}

// redistribute_family, rlt2.cpp:184-205 (device, the phase-2 kernel's rule)
QAPB_API qapb_status qapb_redistribute_family(const double pi[3], double add[3],
                                              int virtual_slots, double tol, int* ok) {
  return guard([&] {
    *ok = qapb::redistribute_family_device(pi, add, virtual_slots, tol, current_device()) ? 1 : 0;
  });
}

// ---- engine ------------------------------------------------------------
QAPB_API qapb_status qapb_engine_create(int m, const double* b, const double* c, const double* d,
                                        double offset, const qapb_config* cfg,
                                        qapb_engine** out) {
  return guard([&] {
    qapb_config c0;
    qapb_config_init(&c0);
    auto h = std::make_unique<qapb_engine>();
    h->e = std::make_unique<Engine>(m, b, c, d, offset, cfg ? *cfg : c0);
    *out = h.release();
  });
}

QAPB_API qapb_status qapb_engine_create_instance(int n, const double* flow, const double* dist,
                                                 const double* linear, const qapb_config* cfg,
                                                 qapb_engine** out) {
  return guard([&] {
    qapb_config c0;
    qapb_config_init(&c0);
    auto h = std::make_unique<qapb_engine>();
    h->e = std::make_unique<Engine>(n, flow, dist, linear, cfg ? *cfg : c0);
    *out = h.release();
  });
}

QAPB_API qapb_status qapb_engine_destroy(qapb_engine* e) {
  return guard([&] { delete e; });
}

QAPB_API qapb_status qapb_engine_iterate(qapb_engine* e, double* bound) {
  return guard([&] {
    const double b = e->e->iterate();
    if (bound) *bound = b;
  });
}

QAPB_API qapb_status qapb_engine_run(qapb_engine* e, qapb_report* rep, qapb_record* records,
                                     int max_records, int* certificate) {
  return guard([&] {
    std::vector<qapb_record> recs;
    std::vector<int> cert;
    qapb_report r{};
    e->e->run(&r, records ? &recs : nullptr, &cert);
    int k = 0;
    if (records) {
      k = std::min<int>(max_records, (int)recs.size());
      std::copy(recs.begin(), recs.begin() + k, records);
    }
    r.n_records = k;
    if (certificate && !cert.empty()) std::copy(cert.begin(), cert.end(), certificate);
    if (rep) *rep = r;
  });
}

QAPB_API qapb_status qapb_engine_best_bound(qapb_engine* e, double* v) {
  *v = e->e->best_bound();
  return QAPB_OK;
}
QAPB_API qapb_status qapb_engine_gap(qapb_engine* e, double* v) {
  *v = e->e->gap();
  return QAPB_OK;
}
QAPB_API qapb_status qapb_engine_iteration(qapb_engine* e, int* v) {
  *v = e->e->iteration();
  return QAPB_OK;
}
QAPB_API qapb_status qapb_engine_last_record(qapb_engine* e, qapb_record* r) {
  *r = e->e->last_record();
  return QAPB_OK;
}
QAPB_API qapb_status qapb_engine_certificate(qapb_engine* e, int* has, int* perm,
                                             double* value) {
  return guard([&] {
    *has = e->e->has_certificate();
    if (*has && perm) {
      auto c = e->e->certificate();
      std::copy(c.begin(), c.end(), perm);
    }
    if (value) *value = e->e->certificate_value();
  });
}
QAPB_API qapb_status qapb_engine_x_assignment(qapb_engine* e, int* xrow) {
  return guard([&] {
    auto x = e->e->x_assignment();
    std::copy(x.begin(), x.end(), xrow);
  });
}
QAPB_API qapb_status qapb_engine_array_size(qapb_engine* e, int which, size_t* count) {
  return guard([&] { *count = e->e->array_size(which); });
}
QAPB_API qapb_status qapb_engine_get_array(qapb_engine* e, int which, double* dst,
                                           size_t count) {
  return guard([&] { e->e->get_array(which, dst, count); });
}
QAPB_API qapb_status qapb_engine_store_offset(qapb_engine* e, double* offset) {
  *offset = e->e->offset();
  return QAPB_OK;
}
QAPB_API qapb_status qapb_engine_snapshot(qapb_engine* e, double* b, double* c, double* d,
                                          double* offset) {
  return guard([&] {
    if (e->e->is_fast())  // rlt2.cpp:537-541
      throw std::logic_error("warm-start snapshots are only offered from S variants");
    e->e->get_array(QAPB_ARR_STORE_B, b, e->e->array_size(QAPB_ARR_STORE_B));
    e->e->get_array(QAPB_ARR_STORE_C, c, e->e->array_size(QAPB_ARR_STORE_C));
    e->e->get_array(QAPB_ARR_STORE_D, d, e->e->array_size(QAPB_ARR_STORE_D));
    *offset = e->e->offset();
  });
}
QAPB_API qapb_status qapb_engine_launch_count(qapb_engine* e, long long* n) {
  *n = e->e->launches();
  return QAPB_OK;
}

QAPB_API qapb_status qapb_engine_enqueue(qapb_engine* e, int iters) {
  return guard([&] { e->e->enqueue(iters); });
}
QAPB_API qapb_status qapb_engine_synchronize(qapb_engine* e) {
  return guard([&] { e->e->synchronize(); });
}
QAPB_API qapb_status qapb_engine_stream(qapb_engine* e, void** stream) {
  *stream = (void*)e->e->stream();
  return QAPB_OK;
}
QAPB_API qapb_status qapb_engine_set_profiling(qapb_engine* e, int on) {
  return guard([&] { e->e->set_profiling(on != 0); });
}
QAPB_API qapb_status qapb_engine_time_kernel(qapb_engine* e, int kind, int reps, double* ms) {
  return guard([&] { *ms = e->e->time_kernel(kind, reps); });
}
QAPB_API qapb_status qapb_engine_history(qapb_engine* e, int from, int count, double* bounds,
                                         double* best) {
  return guard([&] { e->e->history(from, count, bounds, best); });
}
QAPB_API qapb_status qapb_engine_kernel_times(qapb_engine* e, double* ms, long long* launches,
                                              int reset) {
  return guard([&] { e->e->kernel_times(ms, launches, reset != 0); });
}

QAPB_API qapb_status qapb_shard_plan(int n, int world, int* p_bounds) {
  return guard([&] {
    need(n >= 3, "shard_plan: n >= 3 required");
    auto b = qapb::shard_plan(n, world);
    std::copy(b.begin(), b.end(), p_bounds);
  });
}

QAPB_API qapb_status qapb_shard_exchange_counts(int n, int world, int rank, long long* send,
                                                long long* recv) {
  return guard([&] {
    need(n >= 3, "shard_plan: n >= 3 required");
    need(rank >= 0 && rank < world, "bad rank");
    std::vector<long long> s, r;
    qapb::shard_counts(n, qapb::shard_plan(n, world), rank, s, r);
    std::copy(s.begin(), s.end(), send);
    std::copy(r.begin(), r.end(), recv);
  });
}

QAPB_API qapb_status qapb_nccl_unique_id(unsigned char id[128]) {
  return guard([&] {
    ncclUniqueId u;
    const ncclResult_t r = qapb::nccl().GetUniqueId(&u);
    if (r != ncclSuccess)
      throw CudaError(std::string("ncclGetUniqueId: ") + qapb::nccl().GetErrorString(r));
    static_assert(sizeof(u) == 128, "NCCL unique id size");
    std::memcpy(id, &u, 128);
  });
}

QAPB_API qapb_status qapb_engine_create_instance_sharded(int n, const double* flow,
                                                         const double* dist, const double* linear,
                                                         const qapb_config* cfg, int rank,
                                                         int world,
                                                         const unsigned char nccl_id[128],
                                                         qapb_engine** out) {
  return guard([&] {
    qapb_config c0;
    qapb_config_init(&c0);
    auto h = std::make_unique<qapb_engine>();
    h->e = std::make_unique<Engine>(n, flow, dist, linear, cfg ? *cfg : c0, rank, world,
                                    nccl_id);
    *out = h.release();
  });
}

QAPB_API qapb_status qapb_run_ascent(int n, const double* flow, const double* dist,
                                     const double* linear, const qapb_config* cfg,
                                     qapb_report* rep, qapb_record* records, int max_records,
                                     int* certificate) {
  return guard([&] {
    qapb_config c0;
    qapb_config_init(&c0);
    Engine eng(n, flow, dist, linear, cfg ? *cfg : c0);
    std::vector<qapb_record> recs;
    std::vector<int> cert;
    qapb_report r{};
    eng.run(&r, records ? &recs : nullptr, &cert);
    int k = 0;
    if (records) {
      k = std::min<int>(max_records, (int)recs.size());
      std::copy(recs.begin(), recs.begin() + k, records);
    }
    r.n_records = k;
    if (!cert.empty()) {  // run_ascent re-evaluates on the instance, rlt2.cpp:594-595
      double v = 0;
      for (int i = 0; i < n; ++i) {
        v += linear ? linear[(size_t)i * n + cert[i]] : 0.0;
        for (int j = 0; j < n; ++j) v += flow[(size_t)i * n + j] * dist[(size_t)cert[i] * n + cert[j]];
      }
      r.certificate_value = v;
      if (certificate) std::copy(cert.begin(), cert.end(), certificate);
    }
    if (rep) *rep = r;
  });
}

}  // extern "C"

// ---- device-resident stores (store.cu) -------------------
QAPB_API qapb_status qapb_store_upload(int m, const double* b, const double* c,
                                       const double* d, double offset, int device,
                                       qapb_store** out) {
  return guard([&] {
    need(m >= 2, "store: m >= 2 required");
    need(b && c && (m < 3 || d) && out, "store_upload: null pointer");
    auto h = std::make_unique<qapb_store>();
    h->s = std::make_unique<DeviceStore>(m, device);
    // on the store's stream, completed before return (a legacy-stream
    // cudaMemcpy from pageable memory may return before its DMA lands)
    auto up = [&](double* dst, const double* src, size_t n) {
      if (n && cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, h->s->stream) !=
                   cudaSuccess)
        throw CudaError("store_upload: copy failed");
    };
    up(h->s->b, b, store_nb(m));
    up(h->s->c, c, store_nc(m));
    if (m >= 3) up(h->s->d, d, store_nd(m));
    h->s->synchronize();
    h->s->offset = offset;
    *out = h.release();
  });
}

// AscentEngine::snapshot() (rlt2.cpp:537-542) kept in HBM
QAPB_API qapb_status qapb_store_from_engine(qapb_engine* e, qapb_store** out) {
  return guard([&] {
    need(e && out, "store_from_engine: null pointer");
    if (e->e->is_fast())  // rlt2.cpp:538-540
      throw std::logic_error("warm-start snapshots are only offered from S variants");
    const int m = e->e->m();
    auto h = std::make_unique<qapb_store>();
    h->s = std::make_unique<DeviceStore>(m, e->e->device());
    e->e->get_array(QAPB_ARR_STORE_B, h->s->b, e->e->array_size(QAPB_ARR_STORE_B));
    e->e->get_array(QAPB_ARR_STORE_C, h->s->c, e->e->array_size(QAPB_ARR_STORE_C));
    e->e->get_array(QAPB_ARR_STORE_D, h->s->d, e->e->array_size(QAPB_ARR_STORE_D));
    h->s->offset = e->e->offset();
    *out = h.release();
  });
}

QAPB_API qapb_status qapb_store_collapse(const qapb_store* s, int fac, int loc,
                                         qapb_store** out) {
  return guard([&] {
    need(s && out, "store_collapse: null pointer");
    cuda_check_set(s->s->device);
    auto h = std::make_unique<qapb_store>();
    h->s = collapse_store_device(*s->s, fac, loc);
    *out = h.release();
  });
}

QAPB_API qapb_status qapb_store_info(const qapb_store* s, int* m, double* offset) {
  return guard([&] {
    need(s, "store_info: null store");
    if (m) *m = s->s->m;
    if (offset) *offset = s->s->offset;
  });
}

QAPB_API qapb_status qapb_store_download(const qapb_store* s, double* b, double* c, double* d,
                                         double* offset) {
  return guard([&] {
    need(s, "store_download: null store");
    const int m = s->s->m;
    auto down = [&](double* dst, const double* src, size_t n) {
      if (dst && n &&
          cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, s->s->stream) !=
              cudaSuccess)
        throw CudaError("store_download: copy failed");
    };
    cuda_check_set(s->s->device);
    down(b, s->s->b, store_nb(m));
    down(c, s->s->c, store_nc(m));
    down(d, s->s->d, store_nd(m));
    s->s->synchronize();
    if (offset) *offset = s->s->offset;
  });
}

QAPB_API qapb_status qapb_store_destroy(qapb_store* s) {
  return guard([&] { delete s; });
}

// AscentEngine(CoefficientStore, cfg), rlt2.cpp:207-230, device-to-device
QAPB_API qapb_status qapb_engine_create_from_store_offset(const qapb_store* s, double offset,
                                                          const qapb_config* cfg,
                                                          qapb_engine** out) {
  return guard([&] {
    need(s && out, "engine_create_from_store: null pointer");
    qapb_config c0;
    qapb_config_init(&c0);
    qapb_config cc = cfg ? *cfg : c0;
    need(cc.device == s->s->device, "engine_create_from_store: cfg.device must be the store's");
    need(s->s->m >= 3, "AscentEngine: m >= 3 required");  // rlt2.cpp:209
    auto h = std::make_unique<qapb_engine>();
    h->e = std::make_unique<Engine>(s->s->m, s->s->b, s->s->c, s->s->d, offset, cc);
    *out = h.release();
  });
}

QAPB_API qapb_status qapb_engine_create_from_store(const qapb_store* s, const qapb_config* cfg,
                                                   qapb_engine** out) {
  if (!s) {
    g_err = "engine_create_from_store: null pointer";
    return QAPB_EINVAL;
  }
  return qapb_engine_create_from_store_offset(s, s->s->offset, cfg, out);
}

QAPB_API qapb_status qapb_store_collapse_offset(const qapb_store* s, double offset, int fac,
                                                int loc, qapb_store** out) {
  return guard([&] {
    need(s && out, "store_collapse: null pointer");
    auto h = std::make_unique<qapb_store>();
    h->s = collapse_store_device(*s->s, fac, loc, offset);
    *out = h.release();
  });
}

QAPB_API int qapb_exp_variant(void) { return qapb::exp_variant_host(); }

QAPB_API double qapb_exp_glibc(double x, int fma) { return qapb::exp_glibc_host(x, fma); }

QAPB_API qapb_status qapb_exp_batch_device(const double* x, double* y, size_t n, int fma,
                                           void* stream) {
  return guard([&] {
    qapb::cuda_check(qapb::launch_exp_batch(x, y, n, fma, static_cast<cudaStream_t>(stream)),
                     "exp batch");
  });
}

QAPB_API qapb_status qapb_device_memory(int device, size_t* free_bytes, size_t* total_bytes) {
  return guard([&] {
    qapb::DeviceGuard dg(device);
    size_t f = 0, t = 0;
    qapb::cuda_check(cudaMemGetInfo(&f, &t), "cudaMemGetInfo");
    // the stream-ordered pool keeps freed blocks cached (engine.cu
    // keep_pool_cached): count them as free
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      std::uint64_t reserved = 0, used = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      if (reserved > used) f += (size_t)(reserved - used);
    }
    if (free_bytes) *free_bytes = f;
    if (total_bytes) *total_bytes = t;
  });
}

QAPB_API qapb_status qapb_store_device(const qapb_store* s, int* device) {
  return guard([&] {
    need(s && device, "store_device: null pointer");
    *device = s->s->device;
  });
}

QAPB_API qapb_status qapb_store_init(int n, const double* flow, const double* dist,
                                     const double* linear, int device, qapb_store** out) {
  return guard([&] {
    need(out, "store_init: null pointer");
    need(n >= 3, "init_coefficients: n >= 3 required by RLT2");  // rlt2.cpp:67-68
    auto h = std::make_unique<qapb_store>();
    h->s = std::make_unique<DeviceStore>(n, device);
    qapb::DeviceGuard dg(device);
    cudaStream_t st = h->s->stream;
    const size_t nn = (size_t)n * n;
    DevBuf df(nn * 8, st), dd(nn * 8, st), dl(linear ? nn * 8 : 0, st);
    qapb::cuda_check(cudaMemcpyAsync(df.p, flow, nn * 8, cudaMemcpyDefault, st), "H2D flow");
    qapb::cuda_check(cudaMemcpyAsync(dd.p, dist, nn * 8, cudaMemcpyDefault, st), "H2D dist");
    if (linear)
      qapb::cuda_check(cudaMemcpyAsync(dl.p, linear, nn * 8, cudaMemcpyDefault, st), "H2D lin");
    qapb::cuda_check(qapb::launch_init_store(n, df.as<double>(), dd.as<double>(),
                                             dl.as<double>(), h->s->b, h->s->c, st),
                     "init_store");
    qapb::cuda_check(cudaMemsetAsync(h->s->d, 0, store_nd(n) * 8, st), "memset d");
    h->s->offset = 0.0;
    h->s->synchronize();
    *out = h.release();
  });
}

QAPB_API qapb_status qapb_store_evaluate_device(const qapb_store* s, double offset,
                                                const int* perm, double* value) {
  return guard([&] {
    need(s && perm && value, "store_evaluate: null pointer");
    *value = qapb::store_evaluate_device(*s->s, perm, offset);
  });
}

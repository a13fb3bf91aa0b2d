/*
 * qapb200.h — C-ABI of the B200-native RLT2 dual-ascent engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (`qap::AscentEngine` + the Hungarian LAP solver it calls).  Every entry
 * point takes plain pointers and sizes; no C++ or torch types cross it.
 * The C++ facade in include/qap/ (instance, lap, rlt2 .hpp) rebuilds the reference API
 * (same class names, signatures and exception types) on top of these
 * calls; Python reaches them through ctypes.
 *
 * Reference citations are `path:line` inside /root/reference/proj.
 *
 * Error convention: every function returns a qapb_status.  A non-zero status
 * maps 1:1 onto the exception the reference throws at the same point
 * (std::invalid_argument / std::logic_error / std::runtime_error); the
 * message is available from qapb_last_error() (thread-local).
 *
 * Layouts are the reference layouts (StoreIndex, rlt2.hpp:25-69):
 *   b : m*m                      row-major (i, p)
 *   c : m*m*(m-1)*(m-1)          cidx(i,p,j,q), rlt2.hpp:65-68
 *   d : tiles*(m-2)^2            half-Z tiles, tile(i<j,p!=q), rlt2.hpp:43-52
 * and the device keeps them unchanged: each Z tile ((m-2)^2 doubles) and
 * each Y block ((m-1)^2 doubles) is contiguous and is bulk-copied into
 * shared memory by the LAP kernels.
 */
#ifndef QAPB200_H
#define QAPB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define QAPB_API __attribute__((visibility("default")))
#else
#define QAPB_API
#endif

typedef int qapb_status;
enum {
  QAPB_OK = 0,
  QAPB_EINVAL = 1,   /* std::invalid_argument (rlt2.cpp:67-68,209; lap.cpp:26,99-100) */
  QAPB_ELOGIC = 2,   /* std::logic_error (rlt2.cpp:332-335, 538-540) */
  QAPB_ERUNTIME = 3, /* std::runtime_error (instance.cpp parse / IO) */
  QAPB_ECUDA = 4     /* device failure (no reference equivalent; never silent) */
};

/* qap::Variant, rlt2.hpp:18 */
enum { QAPB_F1 = 0, QAPB_F2 = 1, QAPB_S1 = 2, QAPB_S2 = 3 };

/* BoundReport::termination strings, rlt2.cpp:550,557,561,565,574 */
enum {
  QAPB_TERM_ITERATION_LIMIT = 0,
  QAPB_TERM_GAP_CLOSED = 1,
  QAPB_TERM_FEASIBLE_FOUND = 2,
  QAPB_TERM_EARLY_STOP = 3
};

/* Arrays readable through qapb_engine_get_array (the const& accessors of
 * AscentEngine, rlt2.hpp:164-175, plus two private arrays exposed for
 * parity testing). */
enum {
  QAPB_ARR_PI_Z = 0,    /* pi_z()   tiles*(m-2)^2 */
  QAPB_ARR_PI_Y = 1,    /* pi_y()   m*m*(m-1)^2   */
  QAPB_ARR_PI_X = 2,    /* pi_x()   m*m           */
  QAPB_ARR_STORE_B = 3, /* store().b */
  QAPB_ARR_STORE_C = 4, /* store().c */
  QAPB_ARR_STORE_D = 5, /* store().d */
  QAPB_ARR_THETA = 6,   /* theta_ (per-tile Z-LAP optima, rlt2.hpp:196) */
  QAPB_ARR_DELTA = 7,   /* delta_ (per-(i,p) Y-LAP optima, rlt2.hpp:197) */
  QAPB_ARR_INCZ = 8     /* incz_  (F variants only, rlt2.hpp:202) */
};

/* qap::AscentConfig, rlt2.hpp:98-121 (same fields, same defaults through
 * qapb_config_init). */
typedef struct qapb_config {
  int variant;
  int sa_enabled;
  int iter_limit;
  double min_gap;
  double kappa_z_upper;
  double phi_split;
  double kappa_y;
  double kappa_x;
  double varphi;
  double sa_t0_fraction;
  double sa_kappa_lb_cap;
  double sa_cool_factor;
  int sa_cool_period;
  int workers;           /* kept for API parity; never changes results */
  uint64_t seed;
  double upper_bound;
  double fathom_threshold;
  int early_stop_window;
  double early_stop_delta;
  int record_history;
  int device;            /* CUDA device ordinal (B200 extension) */
} qapb_config;

/* qap::IterationRecord, rlt2.hpp:123-128 */
typedef struct qapb_record {
  int iteration;
  double bound;
  double gap;
  double z_ms, y_ms, x_ms;
} qapb_record;

/* Scalar part of qap::BoundReport, rlt2.hpp:130-146 */
typedef struct qapb_report {
  double best_bound;
  double upper_bound;
  double gap;
  int termination;       /* QAPB_TERM_* */
  int iterations;
  int has_certificate;
  double certificate_value;
  double wall_ms;
  int n_records;         /* records written to the caller's buffer */
} qapb_report;

typedef struct qapb_engine qapb_engine;

/* ---- library --------------------------------------------------------- */
QAPB_API const char* qapb_last_error(void);
QAPB_API int qapb_abi_version(void);
QAPB_API void qapb_config_init(qapb_config* cfg);       /* rlt2.hpp:98-121 */
QAPB_API qapb_status qapb_device_count(int* count);
QAPB_API const char* qapb_variant_name(int variant);     /* rlt2.cpp:24-32 */
QAPB_API qapb_status qapb_parse_variant(const char* s, int* variant); /* rlt2.cpp:34-42 */

/* ---- LAP (lap.hpp) ---------------------------------------------------- */
/* LapSolver::solve / solve_lap, lap.cpp:24-102.  Host buffers. */
QAPB_API qapb_status qapb_lap_solve(const double* cost, int m, int* row_to_col,
                                    int* col_to_row, double* u, double* v,
                                    double* value);
/* solve_batch / solve_batch_serial, lap.cpp:122-138.  Host buffers; every
 * output pointer may be NULL.  Bitwise identical to the reference for any
 * batch size. */
QAPB_API qapb_status qapb_lap_solve_batch(const double* costs, int m, int count,
                                          double* values, int* row_to_col,
                                          int* col_to_row, double* u, double* v);
/* Same on device-resident buffers, enqueued on `stream` (cudaStream_t). */
QAPB_API qapb_status qapb_lap_solve_batch_device(const double* costs, int m,
                                                 int count, double* values,
                                                 int* row_to_col, int* col_to_row,
                                                 double* u, double* v,
                                                 void* stream);

/* ---- coefficient store helpers (rlt2.hpp:84-96) ----------------------- */
/* init_coefficients, rlt2.cpp:66-89 (computed on the device). */
QAPB_API qapb_status qapb_init_coefficients(int n, const double* flow,
                                            const double* dist,
                                            const double* linear, double* b,
                                            double* c, double* d);
/* store_evaluate, rlt2.cpp:91-107 */
QAPB_API qapb_status qapb_store_evaluate(int m, const double* b, const double* c,
                                         const double* d, double offset,
                                         const int* perm, double* value);
/* collapse_store, rlt2.cpp:109-182: out arrays sized for m-1. */
QAPB_API qapb_status qapb_collapse_store(int m, const double* b, const double* c,
                                         const double* d, double offset, int fac,
                                         int loc, double* ob, double* oc,
                                         double* od, double* ooffset);
/* redistribute_family, rlt2.cpp:184-205 */
QAPB_API qapb_status qapb_redistribute_family(const double pi[3], double add[3],
                                              int virtual_slots, double tol,
                                              int* ok);

/* ---- engine (AscentEngine, rlt2.hpp:151-213) -------------------------- */
/* AscentEngine(CoefficientStore, cfg), rlt2.cpp:207-230.  Copies the host
 * store to the device; d may be NULL for an all-zero D' (init state). */
QAPB_API qapb_status qapb_engine_create(int m, const double* b, const double* c,
                                        const double* d, double offset,
                                        const qapb_config* cfg,
                                        qapb_engine** out);
/* AscentEngine(init_coefficients(inst), cfg): the store is built on the
 * device from the instance (run_ascent, rlt2.cpp:590-592). */
QAPB_API qapb_status qapb_engine_create_instance(int n, const double* flow,
                                                 const double* dist,
                                                 const double* linear,
                                                 const qapb_config* cfg,
                                                 qapb_engine** out);
QAPB_API qapb_status qapb_engine_destroy(qapb_engine* e);
/* iterate(), rlt2.cpp:515-530 */
QAPB_API qapb_status qapb_engine_iterate(qapb_engine* e, double* bound);
/* run(), rlt2.cpp:544-588.  `records` may be NULL (max_records ignored). */
QAPB_API qapb_status qapb_engine_run(qapb_engine* e, qapb_report* rep,
                                     qapb_record* records, int max_records,
                                     int* certificate);
QAPB_API qapb_status qapb_engine_best_bound(qapb_engine* e, double* v);  /* rlt2.hpp:161 */
QAPB_API qapb_status qapb_engine_gap(qapb_engine* e, double* v);         /* rlt2.cpp:532-535 */
QAPB_API qapb_status qapb_engine_iteration(qapb_engine* e, int* v);      /* rlt2.hpp:163 */
QAPB_API qapb_status qapb_engine_last_record(qapb_engine* e, qapb_record* r);
/* has_certificate/certificate/certificate_value, rlt2.hpp:168-170 */
QAPB_API qapb_status qapb_engine_certificate(qapb_engine* e, int* has,
                                             int* perm, double* value);
QAPB_API qapb_status qapb_engine_x_assignment(qapb_engine* e, int* xrow); /* rlt2.hpp:171 */
QAPB_API qapb_status qapb_engine_array_size(qapb_engine* e, int which,
                                            size_t* count);
QAPB_API qapb_status qapb_engine_get_array(qapb_engine* e, int which,
                                           double* dst, size_t count);
QAPB_API qapb_status qapb_engine_store_offset(qapb_engine* e, double* offset);
/* snapshot(), rlt2.cpp:537-542: QAPB_ELOGIC on F variants. */
QAPB_API qapb_status qapb_engine_snapshot(qapb_engine* e, double* b, double* c,
                                          double* d, double* offset);
/* Kernels launched by this engine since creation (launch accounting for
 * the bench's gpu_launches claim). */
QAPB_API qapb_status qapb_engine_launch_count(qapb_engine* e, long long* n);

/* ---- device-loop / measurement hooks (B200 extension) ----------------
 * enqueue: put `iters` iterate() steps on the engine's stream without any
 * host synchronisation (SA must be off); synchronize: wait, then surface any
 * deferred error (phase-2 regression -> QAPB_ELOGIC).  stream returns the
 * engine's cudaStream_t.  With profiling on, every kernel is bracketed by
 * CUDA events on that stream; kernel_times returns the accumulated device
 * milliseconds and launch counts per kernel kind (QAPB_K_*) since the last
 * reset, and run() fills IterationRecord::{z,y,x}_ms. */
enum {
  QAPB_K_XYFOLD = 0,  /* ascent_update x/y levels, rlt2.cpp:244-262 */
  QAPB_K_ZFOLD = 1,   /* ascent_update z level,    rlt2.cpp:269-298 */
  QAPB_K_ZLAP = 2,    /* Z-LAP batch,              rlt2.cpp:308-325 */
  QAPB_K_PHASE2 = 3,  /* stage_z_second_phase,     rlt2.cpp:344-381 */
  QAPB_K_YSTAGE = 4,  /* stage_y,                  rlt2.cpp:383-426 */
  QAPB_K_XSTAGE = 5,  /* stage_x + feasibility,    rlt2.cpp:428-473 */
  QAPB_K_XCHG = 6,    /* multi-GPU: cross-rank barrier + theta segment exchange */
  QAPB_K_COUNT = 7
};
QAPB_API qapb_status qapb_engine_enqueue(qapb_engine* e, int iters);
QAPB_API qapb_status qapb_engine_synchronize(qapb_engine* e);
QAPB_API qapb_status qapb_engine_stream(qapb_engine* e, void** stream);
QAPB_API qapb_status qapb_engine_set_profiling(qapb_engine* e, int on);
/* Kernel-isolation timing (tuning only): launch kernel `kind` (QAPB_K_*)
 * `reps` times on the engine's current state and return the mean device
 * milliseconds.  DESTROYS the engine's numerical state (the fold is applied
 * repeatedly); the engine must not be used for results afterwards. */
QAPB_API qapb_status qapb_engine_time_kernel(qapb_engine* e, int kind, int reps,
                                             double* ms);
/* Per-iteration bound history (IterationRecord::bound of iterations
 * [from, from+count), 0-based), kept on the device for every iteration. */
QAPB_API qapb_status qapb_engine_history(qapb_engine* e, int from, int count,
                                         double* bounds, double* best);
QAPB_API qapb_status qapb_engine_kernel_times(qapb_engine* e, double* ms,
                                              long long* launches, int reset);

/* ---- multi-GPU: one process per GPU, z state sharded -----
 * Rank r owns the half-Z tiles whose first location lies in
 * [p_bounds[r], p_bounds[r+1]) -- equal shares of tiles, fold work and
 * exchange volume -- and folds every facility triple for its own locations.
 * In a family the X3 member T(b,c,pb,pc)[a,pa] lies in a tile of owner(pb):
 * owner(pb)'s Z-LAP stores its slack into owner(pa)'s buffer and owner(pa)'s
 * fold (which keeps its D') stores its new cost into owner(pb)'s buffer,
 * both directly over NVLink through CUDA IPC mappings (no copy kernels); one
 * all-reduce barrier and the theta broadcasts order them, the O(n^4) Y/X
 * stages run replicated, so every rank holds the same bound.  Results are
 * bitwise those of the single-GPU engine. */
/* Location ranges per rank (p_bounds has world+1 entries). */
QAPB_API qapb_status qapb_shard_plan(int n, int world, int* p_bounds);
/* Doubles rank `rank` stores into (send[p]) / receives from (recv[p]) every
 * peer p per iteration in ONE direction of the X3 exchange (pi one way, the
 * new costs the other; kernels.h ShardInfo). */
QAPB_API qapb_status qapb_shard_exchange_counts(int n, int world, int rank,
                                                long long* send, long long* recv);
QAPB_API qapb_status qapb_nccl_unique_id(unsigned char id[128]);
/* AscentEngine(init_coefficients(inst), cfg) on rank `rank` of `world`;
 * every rank passes the same instance, cfg and NCCL unique id, and the
 * device cfg->device.  F1 and S1 variants. */
QAPB_API qapb_status qapb_engine_create_instance_sharded(
    int n, const double* flow, const double* dist, const double* linear,
    const qapb_config* cfg, int rank, int world, const unsigned char nccl_id[128],
    qapb_engine** out);

/* run_ascent(inst, cfg), rlt2.cpp:590-597: instance in, report out.  The
 * certificate value is re-evaluated on the instance as the reference does. */
QAPB_API qapb_status qapb_run_ascent(int n, const double* flow,
                                     const double* dist, const double* linear,
                                     const qapb_config* cfg, qapb_report* rep,
                                     qapb_record* records, int max_records,
                                     int* certificate);

/* BoundReport::to_json, rlt2.cpp:604-630, byte-identical to the reference's
 * nlohmann output.  recs: 6 doubles per record (iteration, bound, gap, z_ms,
 * y_ms, x_ms).  QAPB_EINVAL when cap <= *len (the length is still set). */
QAPB_API qapb_status qapb_report_json(const char* instance, const char* variant,
                                      int sa_enabled, double best_bound, double upper_bound,
                                      double gap, const char* termination, int iterations,
                                      double wall_ms, const int* cert, int ncert,
                                      double cert_value, const double* recs, int nrec,
                                      char* out, size_t cap, size_t* len);

/* ---- Device-resident stores: branch-and-bound node evaluation ----
 * A qapb_store is a CoefficientStore (rlt2.hpp:72-82) held in HBM.  The B&B
 * flow of bnb.cpp:317-387 (parent snapshot -> collapse_store per child ->
 * AscentEngine(child) -> run) runs without host round trips:
 *   qapb_store_from_engine   AscentEngine::snapshot(), rlt2.cpp:537-542
 *                            (S variants only: std::logic_error otherwise)
 *   qapb_store_collapse      collapse_store(st, fac, loc), rlt2.cpp:109-182,
 *                            bitwise identical to the host function
 *   qapb_engine_create_from_store
 *                            AscentEngine(CoefficientStore, cfg), rlt2.cpp:207,
 *                            device-to-device
 * Stores live on one device (cfg->device for engines built from them must
 * match). */
typedef struct qapb_store qapb_store;
QAPB_API qapb_status qapb_store_upload(int m, const double* b, const double* c,
                                       const double* d, double offset, int device,
                                       qapb_store** out);
QAPB_API qapb_status qapb_store_from_engine(qapb_engine* e, qapb_store** out);
QAPB_API qapb_status qapb_store_collapse(const qapb_store* s, int fac, int loc,
                                         qapb_store** out);
QAPB_API qapb_status qapb_store_info(const qapb_store* s, int* m, double* offset);
QAPB_API qapb_status qapb_store_download(const qapb_store* s, double* b, double* c,
                                         double* d, double* offset);
QAPB_API qapb_status qapb_store_destroy(qapb_store* s);
QAPB_API qapb_status qapb_engine_create_from_store(const qapb_store* s,
                                                   const qapb_config* cfg,
                                                   qapb_engine** out);
/* As above with the store's constant term given explicitly (the facade's
 * CoefficientStore::offset is host-side and may be changed after the device
 * data was made, e.g. bnb.cpp:203 cold_store). */
QAPB_API qapb_status qapb_engine_create_from_store_offset(const qapb_store* s, double offset,
                                                          const qapb_config* cfg,
                                                          qapb_engine** out);
/* collapse_store with the parent's constant term given explicitly
 * (child offset = offset + b[fac, loc], rlt2.cpp:116). */
QAPB_API qapb_status qapb_store_collapse_offset(const qapb_store* s, double offset, int fac,
                                                int loc, qapb_store** out);
/* free / total bytes of a device (cudaMemGetInfo) */
QAPB_API qapb_status qapb_device_memory(int device, size_t* free_bytes, size_t* total_bytes);

/* ---- the SA acceptance exp (rlt2.cpp:494 std::exp) -------------------- */
/* The device SA step evaluates glibc's double exp op for op (csrc/glibc_exp.cuh).
 * qapb_exp_variant: which glibc build the host libm resolves exp to
 * (1 = FMA, 0 = SSE2/AVX, -1 = neither; QAPB_EXP_VARIANT overrides).
 * qapb_exp_glibc: the host restatement of that build (no GPU needed).
 * qapb_exp_batch_device: y[i] = exp(x[i]) on the device, device pointers,
 * enqueued on `stream` -- the function the SA kernel inlines. */
QAPB_API int qapb_exp_variant(void);
QAPB_API double qapb_exp_glibc(double x, int fma);
QAPB_API qapb_status qapb_exp_batch_device(const double* x, double* y, size_t n, int fma,
                                           void* stream);
/* the CUDA device a store lives on */
QAPB_API qapb_status qapb_store_device(const qapb_store* s, int* device);
/* init_coefficients(inst), rlt2.cpp:66-89, built in HBM (D' = 0). */
QAPB_API qapb_status qapb_store_init(int n, const double* flow, const double* dist,
                                     const double* linear, int device, qapb_store** out);
/* store_evaluate(st, perm), rlt2.cpp:91-107, on a device store; `offset`
 * replaces the store's constant term. */
QAPB_API qapb_status qapb_store_evaluate_device(const qapb_store* s, double offset,
                                                const int* perm, double* value);

#ifdef __cplusplus
}
#endif
#endif /* QAPB200_H */

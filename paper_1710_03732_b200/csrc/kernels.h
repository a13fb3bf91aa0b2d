// kernels.h — host-side launch interface of the RLT2 sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace qapb {

// Device-resident scalar state of one engine (AscentEngine's scalar members,
// rlt2.hpp:191-212, plus the device-loop control words).
struct DevScalars {
  double running;     // F variants: accumulated captured mass (rlt2.hpp:194)
  double last_bound;  // rlt2.hpp:195
  double best;        // rlt2.hpp:193
  double offset;      // CoefficientStore::offset (rlt2.hpp:78)
  double cert_val;    // rlt2.hpp:208
  int iter;           // iterations completed (rlt2.hpp:192)
  int has_cert;
  int stop;           // device loop: set when run() terminates
  int term;           // QAPB_TERM_*
  int run_mode;       // 1 inside run(): evaluate termination on device
  int run_start;      // iter at run() entry (best_hist origin)
  int err_tile;       // phase-2 theta regression: smallest tile, INT_MAX = none
  int pad;
};

struct BatchLapParams {
  const double* costs;  // count tiles of m*m, contiguous
  int m, count;
  int* counter;         // dynamic scheduler, zeroed before launch
  const int* stop;      // optional device-loop stop flag
  int* stop_w;          // optional: raised on a phase-2 regression
  double* values;       // optional per-tile optimum
  double* pi;           // optional slack (cost - u - v), same layout as costs
  int *r2c, *c2r;       // optional
  double *u, *v;        // optional
  const double* theta_ref;  // optional: phase-2 regression check (rlt2.cpp:332-335)
  int* err_tile;
  int tile_base;            // global index of tile 0 of this launch (error reports)
};

constexpr int kMaxRanks = 8;

// Shard description (multi-GPU).  Rank r owns first facilities
// [abound[r], abound[r+1]) and tiles [tbase[r], tbase[r+1]).
struct ShardInfo {
  int world, rank;
  int abound[kMaxRanks + 1];
  int tbase[kMaxRanks + 1];
  // exchange buffers indexed by peer rank (null where unused)
  const double* sig_recv[kMaxRanks];   // from higher ranks: sigma of my X3 partners
  double* gain_send[kMaxRanks];        // to higher ranks: gain of their X3 cells
  double* sig_send[kMaxRanks];         // to lower ranks
  const double* gain_recv[kMaxRanks];  // from lower ranks
};

struct FoldParams {
  int m;
  const int* triples;  // (a,b,c) a<b<c, 3 ints each, lexicographic
  int ntriples, chunk, nchunks;  // triples of this launch start at `triples`
  double kz, phi;
  int fast;
  double* d;           // D' (store)
  double* piz;         // pi(z) of the previous iteration (read-only in fold)
  double* incz;        // F variants: incremental Z costs (written)
  const double* push;  // per tile
  double* sa_fac;      // zeroed by block 0 (rlt2.cpp:297-298)
  double* sa_loc;
  const int* stop;
  // phase 2 (rlt2.cpp:344-381): costs mutated in place from pi(z)
  double* costs;
  const ShardInfo* shard;  // null on one GPU
  // multi-GPU passes over triples whose X3 member is remote (owner(b) != me):
  // 0 whole fold, 1 gains of the X3 members only (before the exchange),
  // 2 X1/X2 updates with the received sigma (after it)
  int mode;
};

struct XYFoldParams {
  int m;
  double kx, ky, vph;
  const double* pix;
  const double* sa_fac;
  const double* sa_loc;
  double* dx;
  double* b;
  double* c;
  const double* piy;
  double* ybar;
  double* push;
  const int* fpair_ij;  // fpair -> i | j<<16
  const int* stop;
};

struct YStageParams {
  int m;
  const double* c;
  const double* theta;
  const double* ybar;
  const double* dx;
  int inc;
  double* delta;
  double* piy;
  const int* stop;
};

struct XStageParams {
  int m;
  const double* delta;
  const double* b;
  int inc, fast;
  double* pix;
  int* xrow;
  int* xcol;
  const double* piy;
  const double* piz;
  DevScalars* S;
  double* hist_bound;
  double* hist_best;
  int* cert;
  double upper_bound, min_gap, fathom, es_delta;
  int es_window, iter_limit;
  int* feas_bad;           // device flag: 1 if any induced slack > 1e-7
  int zt_lo, zt_hi;        // tiles whose pi(z) this rank checks (feasibility)
};

// ---- launches (all asynchronous on `st`) ----
cudaError_t launch_init_store(int n, const double* flow, const double* dist,
                              const double* linear, double* b, double* c, cudaStream_t st);
cudaError_t launch_xyfold(const XYFoldParams& p, int tiles, cudaStream_t st);
cudaError_t launch_zfold(const FoldParams& p, cudaStream_t st);
cudaError_t launch_phase2(const FoldParams& p, cudaStream_t st);
// Z-stage and the public batch API: one warp per LAP, TMA bulk tile loads.
cudaError_t launch_lap_batch(const BatchLapParams& p, cudaStream_t st);
cudaError_t launch_ystage(const YStageParams& p, cudaStream_t st);
cudaError_t launch_xstage(const XStageParams& p, cudaStream_t st);
cudaError_t launch_xfinish(const XStageParams& p, cudaStream_t st);
// multi-GPU exchange kernels
cudaError_t launch_sigma_pack(int m, const double* piz, const double* push, double kz,
                              const ShardInfo& sh, const int* stop, cudaStream_t st);
cudaError_t launch_x3_update(int m, double* d, double* incz, const double* piz, double kz,
                             int fast, const ShardInfo& sh, const int* stop, cudaStream_t st);
cudaError_t launch_sa_apply(int m, double* b, const double* sa_fac, const double* sa_loc,
                            DevScalars* S, double drained, int fast, cudaStream_t st);

// chunk size (locations per fold CTA) used for a given m
int fold_chunk(int m);
size_t fold_smem_bytes(int m, int chunk);
int lap_max_m();

}  // namespace qapb

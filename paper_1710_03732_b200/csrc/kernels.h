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
  int sa_pending;     // set by the X stage's finish kernel, consumed by the device SA step
};

// Device SA (rlt2.cpp:477-513): std::mt19937_64 state and the temperature
struct SaState {
  double temp;
  int idx, pad;
  unsigned long long mt[312];
};
struct SaParams {
  int m, cool_period, fast;
  int exp_fma;  // which glibc exp build to restate (exp_variant_host())
  double t0_fraction, kappa_cap, cool_factor, upper_bound;
};
// glibc's double exp, restated bitwise (glibc_exp.cuh).  fma: 1 = the FMA
// build, 0 = SSE2/AVX.  exp_variant_host(): the build the host libm uses
// (-1: neither, i.e. not glibc >= 2.28).
int exp_variant_host();
double exp_glibc_host(double x, int fma);
cudaError_t launch_exp_batch(const double* x, double* y, size_t n, int fma, cudaStream_t stream);
// mt19937_64 seeding (std::mersenne_twister_engine::seed)
void sa_seed(SaState* host_state, unsigned long long seed);

struct ShardInfo;

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
  int* undefined;           // optional: smallest slot whose LAP is undefined in the
                            // reference (no column found by lap.cpp:53), INT_MAX = none
  int tile_base;            // global index of tile 0 of this launch (error reports)
  // optional run mapping (multi-GPU): launch tile t is global tile
  // (t / run_len) * run_stride + run_off + t % run_len
  int run_len, run_stride, run_off;
  // multi-GPU Z stage (location sharding), null on one GPU: the LAP kernel
  // takes the cost of its remote-folded X3 cells from the fold owners'
  // stores (patch) and stores those cells' slack straight into the fold
  // owners' pi buffers after solving (NVLink peer stores)
  const ShardInfo* sh;
  const int* fpair_ij;
  int patch;
  // X3 split (1-phase variants): the X3 member T(b,c,pb,pc)[a,pa] of every
  // family folded here keeps its D' in fold order (FoldParams::d3) and passes
  // pi (mode 2: written by the LAP, read by the fold; mode 1 also the fold's
  // new cost the other way) through x3buf, slot
  //   ((T*ng + po/G)*lpairs + lpair(pb,pc))*G + po%G,  po = pa - first location,
  // groups of G locations (a multiple of the fold chunk): the fold reads whole
  // chunks, a Z-LAP row store touches only n/G segments
  double* x3buf;
  double* costs_w;
  int x3_group, x3_ngroups;
  // RI layout (z_ri_offset): tiles move by 3-D TMA tensor copies through
  // these tensor maps (device memory, 64-byte aligned CUtensorMap; costs and
  // pi are then base pointers and tile_base + t the global tile index)
  const void* tmap_cost;
  const void* tmap_pi;
  size_t nx3;  // element count of x3buf (bounds checks of a -DQAPB_BOUNDS build)
  // per-stage device timestamps (IterationRecord::z_ms, rlt2.cpp:302,337):
  // block 0 of the iteration's first Z-LAP launch stores %globaltimer in
  // tstamp[4 * *iter + 0]
  unsigned long long* tstamp;
  const int* iter;
};

constexpr int kMaxRanks = 8;

// Shard description (multi-GPU).  Rank r owns the half-Z
// tiles whose FIRST location lies in [pbound[r], pbound[r+1]): one run of
// rl(r) = (pbound[r+1]-pbound[r])*(n-1) tiles inside every facility-pair
// block, and solves their Z-LAPs.  It folds every facility triple for its
// own locations pa; in a family the X3 member T(b,c,pb,pc)[a,pa] lies in a
// tile of owner(pb).  When owner(pb) = B != A = owner(pa), A owns that
// cell's D' (in d3[B], in the cost layout below; B's copy is stale) and B
// owns its pi and its LAP.
// Per iteration two values cross per such cell, both stored by the producing
// kernel straight into a buffer on the consuming rank through CUDA IPC
// mappings over NVLink (no copy step):
//   pi   (B's Z-LAP -> A's next fold), layout per (pair f=(b,c), B's local
//        location pair, row a<b, pa of A), so B stores whole row segments:
//        index = ((rl(B)*rows_before[f] + lp_local*b + a) * n(A)) + (pa - pbound[A])
//   cost (A's fold -> B's Z-LAP: the cell's new incremental cost, F variants,
//        or new D', S variants), fold order, so each fold CTA stores one
//        contiguous block:
//        slot = (T*nch(A) + chunk) * n(B)*(n-1)*chunk_cap
//               + ((pb - pbound[B])*(n-1) + pci)*chunk_cap + pa_l,
//        T = lexicographic triple index.
// A kernel's peer stores are complete when it completes; the NCCL collective
// that follows it on the engine stream (the barrier after the fold, the theta
// broadcast after the Z-LAPs) orders them before the peer's next kernel, so
// no system fences are needed inside the kernels.
struct ShardInfo {
  int world, rank;
  int pbound[kMaxRanks + 1];
  int chunk;                           // fold chunk capacity (pa values per CTA)
  const int* rows_before;              // [fpairs+1], prefix sums of b over pairs (b<c)
  const double* pi_recv[kMaxRanks];    // local: pi of my families' remote X3 cells
  double* cost_send[kMaxRanks];        // PEER: X3 owner's cost buffer for my families
  double* pi_send[kMaxRanks];          // PEER: fold owner's pi buffer for my X3 cells
  const double* cost_recv[kMaxRanks];  // local: costs of my remote-folded X3 cells
  double* d3[kMaxRanks];               // local: D' of my families' X3 cells in rank r (fold order)
  double* keep[kMaxRanks];             // local (F2 sharded): the fold's new cost of those cells,
                                       // which phase 2 updates (same layout as d3)
};

__host__ __device__ inline int shard_chunks(const ShardInfo& sh, int r) {
  return (sh.pbound[r + 1] - sh.pbound[r] + sh.chunk - 1) / sh.chunk;
}
__host__ __device__ inline long long shard_cost_count(const ShardInfo& sh, int n, int A, int B) {
  const long long tri = (long long)n * (n - 1) * (n - 2) / 6;
  return tri * shard_chunks(sh, A) * (long long)(sh.pbound[B + 1] - sh.pbound[B]) * (n - 1) *
         sh.chunk;
}

__host__ __device__ inline int shard_owner(const ShardInfo& sh, int p) {
  int r = sh.world - 1;
  while (r > 0 && p < sh.pbound[r]) --r;
  return r;
}

struct FoldParams {
  int m;
  const int* triples;  // (a,b,c) a<b<c, 3 ints each, lexicographic
  int ntriples, chunk, nchunks;  // triples of this launch start at `triples`
  int tri0;                      // global index of the launch's first triple
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
  const ShardInfo* shard;  // null on one GPU: the CTA's pa chunk comes from the rank's range
  // single-GPU X3 split (BatchLapParams::x3buf): X3 pi and new cost in
  // x3buf, X3 D' in d3, both in fold order (unit * lpairs * chunk + pair * chunk + pa_l)
  double* x3buf;
  double* d3;
  int x3mode;  // 1: split (LAP patches), 2: hybrid (fold stores the cost to the tile)
  int x3_group, x3_ngroups;  // x3buf layout (BatchLapParams::x3buf)
  // pipelined fold: the order in which triples are processed (a permutation
  // of 0..ntriples-1 in blocks of a, b and c for DRAM row locality); null =
  // lexicographic.  Only the processing order changes, never a buffer index.
  const int* order;
  // z arrays (d, piz, incz) in the row-interleaved device layout (see
  // z_ri_offset below) instead of the reference tile layout
  int ri;
  // element counts of d / x3buf / d3 (bounds checks of a -DQAPB_BOUNDS build)
  size_t nz, nx3, nd3;
  int costs_are_d;  // phase 2: the solve costs are D' (X3 members also in d3)
  // RI: CUtensorMap (global, 64-byte aligned) of pi(z) as rows of n-2 with a
  // box of {n, chunk*(n-1)} -- a unit's X1 / X2 rows, padded to n in smem
  const void* tmap_rows;
  int l2_hints;  // zfold_lean_kernel: X3 tile stores evict_last (QAPB_LEAN_HINTS)
  int keep_cost; // sharded fold: also keep remote X3 costs in ShardInfo::keep (2-phase F2)
  int rows_cp;   // stage the X1 / X2 pi rows with cp.async pieces, not TMA boxes
};

// Row-interleaved ("RI") device layout of the z arrays (pi(z), D', incz) of a
// single-GPU 1-phase engine: element (tile t = f*lpairs + lp, row k, col r)
// of the reference layout (StoreIndex, rlt2.hpp:43-52) lives at
//   ((f*(n-2) + k)*lpairs + lp)*(n-2) + r,
// i.e. row k of all lpairs tiles of facility pair f is one contiguous block.
// The fold's X1 / X2 rows of a unit (row c or b of 2(n-1) consecutive tiles)
// are then one contiguous 13 KB run instead of 224-byte pieces 6 KB apart
// (tools/layout_probe.cu: 3.4 vs 4.9+ TB/s for the same bytes), and a Z-LAP
// tile is one 3-D TMA tensor copy whose rows, across the warps working on
// consecutive tiles, are again contiguous in DRAM.
__host__ __device__ inline size_t z_ri_offset(int n, size_t t, int k, int r) {
  const size_t lpairs = (size_t)n * (n - 1), nm2 = (size_t)(n - 2);
  const size_t f = t / lpairs, lp = t - f * lpairs;
  return ((f * nm2 + k) * lpairs + lp) * nm2 + r;
}

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
  unsigned long long* tstamp;  // [4 * *iter + 1]: Y stage start (rlt2.cpp:384)
  const int* iter;
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
  int zp_lo, zp_hi;        // first locations of the pi(z) tiles this rank checks
  int ri;                  // pi(z) in the RI layout (z_ri_offset)
  unsigned long long* tstamp;  // [4 * iter + 2]: X stage start, [+3]: its end (rlt2.cpp:429,448)
};

// ---- launches (all asynchronous on `st`) ----
cudaError_t launch_init_store(int n, const double* flow, const double* dist,
                              const double* linear, double* b, double* c, cudaStream_t st);
cudaError_t launch_xyfold(const XYFoldParams& p, int tiles, cudaStream_t st);
cudaError_t launch_zfold(const FoldParams& p, cudaStream_t st);
cudaError_t launch_phase2(const FoldParams& p, cudaStream_t st);
// phase 2 on the RI + X3-split layout (single GPU); costs_are_d: the solve
// costs are the store's D' (S variants, and iteration 0), whose X3 members
// also live in d3
cudaError_t launch_phase2_ri(const FoldParams& p, bool costs_are_d, cudaStream_t st);
// Z-stage and the public batch API: one warp per LAP, TMA bulk tile loads.
cudaError_t launch_lap_batch(const BatchLapParams& p, cudaStream_t st);
cudaError_t launch_ystage(const YStageParams& p, cudaStream_t st);
cudaError_t launch_xstage(const XStageParams& p, cudaStream_t st);
cudaError_t launch_xfinish(const XStageParams& p, cudaStream_t st);
// z array layout conversion: reference tile layout <-> RI (to_ri = 1: src is
// in the reference layout).  Out of place.
cudaError_t launch_z_relayout(int n, const double* src, double* dst, int to_ri, cudaStream_t st);
// The RI path's kernels exist for this (n, fold chunk, x3 group): even n, the
// warp-specialised fold, TMA tensor maps available.
bool ri_supported(int n, int chunk, int x3_group);
// CUtensorMap (128 bytes) of an RI z array for the Z-LAP tile copies
void encode_z_tmap(void* out128, const double* base, int n);
// pi(z) (RI) as a 2-D tensor of rows of n-2 doubles, box {n, chunk*(n-1)}:
// a fold unit's X1 / X2 rows with two zero-filled pad columns (FoldParams::tmap_rows)
void encode_rows_tmap(void* out128, const double* base, int n, int chunk);
// theta of every rank's tile runs <-> one contiguous buffer (rank segments)
// single-GPU X3 split: D' of the X3 members, tile layout <-> fold order
cudaError_t launch_x3_sync(int n, int chunk, int nchunks, const int* triples, int ntriples,
                           int p_lo, int p_hi, double* d, double* d3, int to_d3, cudaStream_t st,
                           int ri = 0);
// one SA step on the device after an iteration (no-op unless that iteration's
// X stage ran, when a certificate exists, or when best <= 0)
// sharded 2-phase: raise stop when the reduced phase-2 regression flag is set
cudaError_t launch_err_to_stop(DevScalars* S, cudaStream_t st);
cudaError_t launch_sa_device(const SaParams& p, double* b, DevScalars* S, SaState* st,
                             double* sa_fac, double* sa_loc, cudaStream_t st_);
// sharded: remote-folded X3 costs (cost_recv) -> the tile-layout cost array
cudaError_t launch_x3_cost_scatter(int n, const ShardInfo& sh, const int* triples, double* costs,
                                   cudaStream_t st);
// sharded z-state assembly (Engine::get_array on a sharded engine)
cudaError_t launch_shard_state_scatter(int n, const ShardInfo& sh, const int* triples,
                                       double* dst, int costs, cudaStream_t st);
cudaError_t launch_shard_state_mask(int n, const ShardInfo& sh, const double* src,
                                    unsigned long long* out, int fold_owned, cudaStream_t st);
cudaError_t launch_theta_xfer(int m, double* theta, double* buf, const ShardInfo& sh, int pack,
                              cudaStream_t st);
cudaError_t launch_sa_apply(int m, double* b, const double* sa_fac, const double* sa_loc,
                            DevScalars* S, double drained, int fast, cudaStream_t st);

// chunk size (locations per fold CTA) used for a given m
int fold_chunk(int m);
size_t fold_smem_bytes(int m, int chunk);
int lap_max_m();

}  // namespace qapb

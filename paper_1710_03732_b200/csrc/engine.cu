// engine.cu — host side of the device-resident RLT2 dual-ascent engine.
#include "engine.h"
#include "nccl_dyn.h"

#include <chrono>
#include <climits>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <cstdio>
#include <mutex>
#include <set>
#include <string>
#include <limits>

namespace qapb {

// Location ranges per rank: every first location owns the same
// n(n-1)^2/2 tiles and the same share of fold work, so contiguous, near-equal
// ranges balance the Z-LAPs, the fold and the exchange volume at once.
std::vector<int> shard_plan(int n, int world) {
  if (world < 1 || world > n) throw std::invalid_argument("shard_plan: bad world size");
  std::vector<int> b(world + 1);
  for (int r = 0; r <= world; ++r) b[r] = (int)(((long long)r * n) / world);
  return b;
}

// pi values rank `rank` stores into (send[p]) / receives from (recv[p]) each
// peer per iteration; the cost stores move the same amounts back.
void shard_counts(int n, const std::vector<int>& pb, int rank, std::vector<long long>& send,
                  std::vector<long long>& recv) {
  const int world = (int)pb.size() - 1;
  long long rows = 0;  // sum over pairs b<c of b
  for (int b = 0; b < n; ++b) rows += (long long)b * (n - 1 - b);
  auto rl = [&](int r) { return (long long)(pb[r + 1] - pb[r]) * (n - 1); };
  auto nl = [&](int r) { return (long long)(pb[r + 1] - pb[r]); };
  send.assign(world, 0);
  recv.assign(world, 0);
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    send[p] = rl(rank) * rows * nl(p);  // pi of my X3 cells folded by p
    recv[p] = rl(p) * rows * nl(rank);  // pi of p's X3 cells folded here
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

namespace {
// Debugging aid (QAPB_SYNC_CHECK=1, eager mode): every engine kernel launch
// is followed by a synchronisation of the current device, so a faulting
// kernel is named by the error it raises.
bool sync_check_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("QAPB_SYNC_CHECK");
    return v && *v && std::strcmp(v, "0") != 0;
  }();
  return on;
}
// QAPB_SYNC_CHECK=<substring>: only launches whose label contains it
bool sync_check_matches(const char* what) {
  static const std::string sel = [] {
    const char* v = std::getenv("QAPB_SYNC_CHECK");
    return std::string(v ? v : "");
  }();
  return sel == "1" || std::string(what).find(sel) != std::string::npos;
}
}  // namespace

// a kernel launch of this engine; under QAPB_SYNC_CHECK its streams are
// synchronised right away (other engines' kernels keep running concurrently)
void Engine::kcheck(cudaError_t e, const char* what) const {
  cuda_check(e, what);
  if (sync_check_enabled() && sync_check_matches(what)) {
    cuda_check(cudaStreamSynchronize(st_), what);
    if (st2_) cuda_check(cudaStreamSynchronize(st2_), what);
  }
}

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

template <class T>
void dalloc(T** p, size_t n) {
  cuda_check(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T)),
             "cudaMalloc");
}
template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// Engine state comes from the device's stream-ordered pool: creating and
// destroying engines (one per branch-and-bound node, several banks at once,
// bnb.cpp:549-556) must not serialise the device the way cudaMalloc/cudaFree
// do, and freed blocks stay cached for the next engine.
bool env_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && *v && std::strcmp(v, "0") != 0;
}

void keep_pool_cached(int dev) {
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert(dev).second) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    std::uint64_t keep = ~std::uint64_t{0};
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (env_flag("QAPB_POOL_NO_XSTREAM")) {  // debugging aid: no cross-stream reuse
      int off = 0;
      cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &off);
      cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &off);
    }
  }
}
template <class T>
void salloc(cudaStream_t st, T** p, size_t n) {
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T), st),
             "cudaMallocAsync");
}
template <class T>
void sfree(cudaStream_t st, T*& p) {
  if (p) cudaFreeAsync(p, st);
  p = nullptr;
}

// Pinned host blocks for the engines' scalar mirrors, recycled for the life of
// the process: cudaFreeHost synchronises the device, which would make every
// branch-and-bound node's engine teardown wait for all other banks' work.
constexpr size_t kPinnedBlock = 512;
struct PinnedPool {
  std::mutex mu;
  std::vector<void*> free_list;
};
PinnedPool& pinned_pool() {
  static PinnedPool* pool = new PinnedPool;  // never destroyed: engines may outlive statics
  return *pool;
}
void* pinned_get() {
  static_assert(sizeof(DevScalars) <= kPinnedBlock, "DevScalars");
  PinnedPool& pp = pinned_pool();
  std::lock_guard<std::mutex> lk(pp.mu);
  std::vector<void*>& free_list = pp.free_list;
  if (free_list.empty()) {
    constexpr int kPer = 64;
    char* slab = nullptr;
    cuda_check(cudaMallocHost(reinterpret_cast<void**>(&slab), kPer * kPinnedBlock),
               "cudaMallocHost");
    for (int k = 0; k < kPer; ++k) free_list.push_back(slab + k * kPinnedBlock);
  }
  void* p = free_list.back();
  free_list.pop_back();
  return p;
}
void pinned_put(void* p) {
  PinnedPool& pp = pinned_pool();
  std::lock_guard<std::mutex> lk(pp.mu);
  pp.free_list.push_back(p);
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}


// One NCCL communicator per (unique id, rank, device) for the process
// lifetime: engines created again with the same id (a B&B bank, repeated
// run_ascent calls) reuse it instead of paying ncclCommInitRank each time.
ncclComm_t cached_comm(const ncclUniqueId& id, int world, int rank, int dev) {
  static std::mutex mu;
  static std::map<std::string, ncclComm_t> cache;
  std::string key(reinterpret_cast<const char*>(&id), sizeof id);
  key += ":" + std::to_string(world) + ":" + std::to_string(rank) + ":" + std::to_string(dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().CommInitRank(&c, world, id, rank);
  if (r != ncclSuccess)
    throw CudaError(std::string("NCCL error in ncclCommInitRank: ") + nccl().GetErrorString(r));
  cache.emplace(key, c);
  return c;
}
}  // namespace

Engine::Engine(int m, const double* b, const double* c, const double* d, double offset,
               const qapb_config& cfg)
    : m_(m), dev_(cfg.device), cfg_(cfg), rng_(cfg.seed) {
  // arguments first: a bad call fails the reference's way without touching the device
  if (m_ < 3) throw std::invalid_argument("AscentEngine: m >= 3 required");  // rlt2.cpp:209
  if (m_ > lap_max_m()) throw std::invalid_argument("AscentEngine: m too large for device LAP");
  const DeviceGuard dg(dev_);
  alloc();
  setup_shards(nullptr);
  init_state();
  cuda_check(cudaMemcpyAsync(b_, b, nb_ * sizeof(double), cudaMemcpyDefault, st_), "H2D b");
  cuda_check(cudaMemcpyAsync(c_, c, nc_ * sizeof(double), cudaMemcpyDefault, st_), "H2D c");
  if (d && ri_) {  // reference layout in, RI layout on the device (pi(z) as scratch)
    cuda_check(cudaMemcpyAsync(piz_, d, nd_ * sizeof(double), cudaMemcpyDefault, st_), "H2D d");
    kcheck(launch_z_relayout(m_, piz_, d_, 1, st_), "relayout d");
    ++launches_;
    cuda_check(cudaMemsetAsync(piz_, 0, nd_ * sizeof(double), st_), "memset");
  } else if (d) {
    cuda_check(cudaMemcpyAsync(d_, d, nd_ * sizeof(double), cudaMemcpyDefault, st_), "H2D d");
  } else {
    cuda_check(cudaMemsetAsync(d_, 0, nd_ * sizeof(double), st_), "memset d");
  }
  split_gather();
  hS_.offset = offset;
  push_scalars();
  cuda_check(cudaStreamSynchronize(st_), "engine create");
}

Engine::Engine(int n, const double* flow, const double* dist, const double* linear,
               const qapb_config& cfg, int rank, int world, const unsigned char* nccl_id)
    : rank_(rank), world_(world), m_(n), dev_(cfg.device), cfg_(cfg), rng_(cfg.seed) {
  // arguments first: a bad call fails the reference's way without touching the device
  if (n < 3) throw std::invalid_argument("init_coefficients: n >= 3 required by RLT2");
  if (m_ > lap_max_m()) throw std::invalid_argument("AscentEngine: m too large for device LAP");
  if (world_ < 1 || world_ > kMaxRanks || rank_ < 0 || rank_ >= world_)
    throw std::invalid_argument("AscentEngine: bad rank/world");
  if (world_ > 1 && cfg.sa_enabled && env_int("QAPB_HOST_SA", 0))
    throw std::invalid_argument("sharded engine: SA runs on the device (QAPB_HOST_SA unsupported)");
  if (world_ > 1 && is_two_phase() && n % 2)
    throw std::invalid_argument("sharded engine: the 2-phase variants need even n "
                                "(row-interleaved layout)");
  if (world_ > n) throw std::invalid_argument("sharded engine: more ranks than locations");
  const DeviceGuard dg(dev_);
  alloc();
  setup_shards(nccl_id);
  init_state();
  double *df = nullptr, *dd = nullptr, *dl = nullptr;
  const size_t nn = (size_t)n * n;
  salloc(st_, &df, nn);
  salloc(st_, &dd, nn);
  if (linear) salloc(st_, &dl, nn);
  cuda_check(cudaMemcpyAsync(df, flow, nn * 8, cudaMemcpyHostToDevice, st_), "H2D flow");
  cuda_check(cudaMemcpyAsync(dd, dist, nn * 8, cudaMemcpyHostToDevice, st_), "H2D dist");
  if (linear)
    cuda_check(cudaMemcpyAsync(dl, linear, nn * 8, cudaMemcpyHostToDevice, st_), "H2D lin");
  kcheck(launch_init_store(n, df, dd, dl, b_, c_, st_), "init_store");
  ++launches_;
  cuda_check(cudaMemsetAsync(d_, 0, nd_ * sizeof(double), st_), "memset d");
  split_gather();
  hS_.offset = 0.0;
  push_scalars();
  sfree(st_, df);
  sfree(st_, dd);
  sfree(st_, dl);
  cuda_check(cudaStreamSynchronize(st_), "engine create");
}

void Engine::alloc() {
  cuda_check(cudaSetDevice(dev_), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking), "stream");
  keep_pool_cached(dev_);
  const int m = m_;
  fpairs_ = m * (m - 1) / 2;
  lpairs_ = m * (m - 1);
  tiles_ = fpairs_ * lpairs_;
  esz_ = (m - 2) * (m - 2);
  nb_ = (size_t)m * m;
  nc_ = (size_t)m * m * (m - 1) * (m - 1);
  nd_ = (size_t)tiles_ * esz_;
  ntriples_ = m * (m - 1) * (m - 2) / 6;
  chunk_ = fold_chunk(m);
  // even n >= 20: two locations per fold unit, so that the row-interleaved
  // layout and the warp-specialised fold apply (measured: n=20 fold 0.246 ->
  // 0.210 ms, n=22 0.433 -> 0.317; below 20 the family-cube folds are faster)
  if (world_ == 1 && m % 2 == 0 && m >= 20 && chunk_ > 2 && !std::getenv("QAPB_FOLD_CHUNK"))
    chunk_ = 2;
  // sharded 2-phase runs phase 2 in the warp-specialised pipeline (chunk 2)
  if (world_ > 1 && is_two_phase() && m % 2 == 0) chunk_ = 2;
  nchunks_ = (m + chunk_ - 1) / chunk_;
  salloc(st_, &b_, nb_);
  salloc(st_, &c_, nc_);
  salloc(st_, &d_, nd_);
  salloc(st_, &piz_, nd_);
  if (is_fast()) salloc(st_, &incz_, nd_);
  salloc(st_, &piy_, nc_);
  salloc(st_, &pix_, nb_);
  salloc(st_, &theta_, tiles_);
  if (is_two_phase()) salloc(st_, &theta1_, tiles_);
  salloc(st_, &delta_, nb_);
  salloc(st_, &ybar_, tiles_);
  salloc(st_, &dx_, nb_);
  salloc(st_, &push_, tiles_);
  salloc(st_, &sa_fac_, m);
  salloc(st_, &sa_loc_, m);
  salloc(st_, &xrow_, m);
  salloc(st_, &xcol_, m);
  salloc(st_, &cert_, m);
  salloc(st_, &triples_, 3 * (size_t)ntriples_);
  salloc(st_, &fpair_ij_, fpairs_);
  plan_pipeline();
  split_mode_ = env_int("QAPB_X3SPLIT", 2);
  // sharded engines split only their local X3 members, in hybrid mode; the
  // 2-phase variants take the split only together with the RI layout (their
  // phase-2 kernel, phase2_ri_kernel, exists for that layout alone)
  const int x3g = std::max(1, env_int("QAPB_X3_GROUP", 4) / chunk_) * chunk_;
  if (!is_two_phase())
    split_ = world_ == 1 ? split_mode_ != 0 : split_mode_ == 2;
  else
    split_ = split_mode_ == 2 && stage_ev_.size() == 1 && env_int("QAPB_ZLAYOUT", 1) != 0 &&
             ri_supported(m, chunk_, x3g);
  if (split_) {  // X3 members in fold order (kernels.h, FoldParams::x3buf)
    int range = m;
    if (world_ > 1) {
      const std::vector<int> pb = shard_plan(m, world_);
      range = pb[rank_ + 1] - pb[rank_];
    }
    const int nch = (range + chunk_ - 1) / chunk_;
    x3_group_ = x3g;
    x3_ngroups_ = (range + x3_group_ - 1) / x3_group_;
    salloc(st_, &x3buf_, (size_t)ntriples_ * x3_ngroups_ * lpairs_ * x3_group_);
    salloc(st_, &d3_, (size_t)ntriples_ * nch * lpairs_ * chunk_);
  }
  // RI layout for the single-GPU 1-phase split engine (the warp-specialised
  // fold + tensor-map Z-LAPs); QAPB_ZLAYOUT=0 keeps the reference tile layout
  ri_ = split_ && split_mode_ == 2 && stage_ev_.size() == 1 &&
        env_int("QAPB_ZLAYOUT", 1) != 0 && ri_supported(m, chunk_, x3_group_) &&
        (world_ == 1 || env_int("QAPB_ZLAYOUT_SHARDED", 1) != 0);
  if (world_ > 1 && is_two_phase() && !ri_)
    throw std::invalid_argument("sharded engine: the 2-phase variants need the row-interleaved "
                                "layout (QAPB_ZLAYOUT, QAPB_X3SPLIT=2, n < 64)");
  if (ri_) {
    unsigned char h[4 * 128];
    encode_z_tmap(h, d_, m);
    if (incz_) encode_z_tmap(h + 128, incz_, m);
    encode_z_tmap(h + 256, piz_, m);
    encode_rows_tmap(h + 384, piz_, m, chunk_);
    salloc(st_, &tmaps_, sizeof h);  // pool blocks are 256-byte aligned (CUtensorMap: 64)
    cuda_check(cudaMemcpyAsync(tmaps_, h, sizeof h, cudaMemcpyHostToDevice, st_),
               "H2D tensor maps");
    cuda_check(cudaStreamSynchronize(st_), "H2D tensor maps");
  }
  // every rank of a sharded engine holds the same b, best and RNG stream, so
  // each runs the same SA step and the replicated state stays identical
  sa_dev_ = cfg_.sa_enabled && m_ <= 128 && env_int("QAPB_HOST_SA", 0) == 0;
  if (sa_dev_) {
    salloc(st_, &sa_state_, 1);
    SaState h;
    sa_seed(&h, cfg_.seed);
    cuda_check(cudaMemcpyAsync(sa_state_, &h, sizeof h, cudaMemcpyHostToDevice, st_), "H2D sa");
    cuda_check(cudaStreamSynchronize(st_), "sa seed");
    exp_fma_ = exp_variant_host();
    if (exp_fma_ < 0) {  // not glibc >= 2.28: the accept test may differ from std::exp
      static std::once_flag warned;
      std::call_once(warned, [] {
        std::fprintf(stderr, "qapb: host libm exp matches neither glibc build; device SA "
                             "uses the FMA build (set QAPB_EXP_VARIANT=fma|nofma)\n");
      });
      exp_fma_ = 1;
    }
  }
  salloc(st_, &counter_, stage_ev_.size() + 2);
  salloc(st_, &S_, 1);
  hSpin_ = static_cast<DevScalars*>(pinned_get());
  std::vector<int> tr;
  tr.reserve(3 * (size_t)ntriples_);
  for (int a = 0; a < m; ++a)
    for (int b = a + 1; b < m; ++b)
      for (int c = b + 1; c < m; ++c) {
        tr.push_back(a);
        tr.push_back(b);
        tr.push_back(c);
      }
  std::vector<int> fp(fpairs_);
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) fp[i * m - i * (i + 1) / 2 + (j - i - 1)] = i | (j << 16);
  cuda_check(cudaStreamSynchronize(st_), "stream-ordered allocations");
  // H2D copies of engine tables go through the engine's stream: a legacy-stream
  // cudaMemcpy from pageable memory may return before its DMA lands, and the
  // engine's kernels run on non-blocking streams that do not wait for it (a
  // branch-and-bound run with 8-16 banks read half-written fpair tables)
  cuda_check(cudaMemcpyAsync(triples_, tr.data(), tr.size() * sizeof(int), cudaMemcpyHostToDevice,
                             st_),
             "H2D triples");
  // fold processing order: triples in blocks of B values of a, b and c, so the
  // units in flight together read several adjacent rows of each tile they touch
  // (X1 rows c, X2 rows b, X3 rows a) instead of single 8(n-2)-byte rows
  const int ob = env_int("QAPB_FOLD_ORDER_BLOCK", 0);
  if (split_ && world_ == 1 && ob > 0) {
    std::vector<int> lex((size_t)m * m * m, -1), ord;
    ord.reserve(ntriples_);
    for (int t = 0; t < ntriples_; ++t)
      lex[((size_t)tr[3 * t] * m + tr[3 * t + 1]) * m + tr[3 * t + 2]] = t;
    for (int a0 = 0; a0 < m; a0 += ob)
      for (int b0 = a0; b0 < m; b0 += ob)
        for (int c0 = b0; c0 < m; c0 += ob)
          for (int a = a0; a < std::min(m, a0 + ob); ++a)
            for (int b = std::max(b0, a + 1); b < std::min(m, b0 + ob); ++b)
              for (int c = std::max(c0, b + 1); c < std::min(m, c0 + ob); ++c)
                ord.push_back(lex[((size_t)a * m + b) * m + c]);
    if ((int)ord.size() != ntriples_) throw std::logic_error("fold order: not a permutation");
    salloc(st_, &order_, ord.size());
    cuda_check(cudaMemcpyAsync(order_, ord.data(), ord.size() * sizeof(int),
                               cudaMemcpyHostToDevice, st_),
               "H2D fold order");
  }
  cuda_check(cudaMemcpyAsync(fpair_ij_, fp.data(), fp.size() * sizeof(int),
                             cudaMemcpyHostToDevice, st_),
             "H2D fpairs");
  cuda_check(cudaStreamSynchronize(st_), "H2D tables");
  ensure_hist(std::max(cfg_.iter_limit, 64) + 1);
}

void Engine::init_state() {
  auto z = [&](void* p, size_t bytes) {
    if (p) cuda_check(cudaMemsetAsync(p, 0, bytes, st_), "memset");
  };
  z(piz_, nd_ * 8);
  z(incz_, nd_ * 8);
  z(piy_, nc_ * 8);
  z(pix_, nb_ * 8);
  z(theta_, tiles_ * 8);
  z(theta1_, tiles_ * 8);
  z(delta_, nb_ * 8);
  z(ybar_, tiles_ * 8);
  z(dx_, nb_ * 8);
  z(push_, tiles_ * 8);
  z(sa_fac_, m_ * 8);
  z(sa_loc_, m_ * 8);
  cuda_check(cudaMemsetAsync(xrow_, 0xff, m_ * sizeof(int), st_), "memset");
  cuda_check(cudaMemsetAsync(xcol_, 0xff, m_ * sizeof(int), st_), "memset");
  std::memset(&hS_, 0, sizeof hS_);
  hS_.best = -kInf;
  hS_.err_tile = INT_MAX;
  hS_.term = QAPB_TERM_ITERATION_LIMIT;
}

Engine::~Engine() {
  int prev = -1;  // DeviceGuard without throwing from a destructor
  cudaGetDevice(&prev);
  if (prev != dev_) cudaSetDevice(dev_);
  if (st_) cudaStreamSynchronize(st_);
  if (graph_) cudaGraphExecDestroy(graph_);
  for (auto& pe : pending_) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (double** p : {&b_, &c_, &d_, &piz_, &incz_, &piy_, &pix_, &theta_, &theta1_, &delta_, &ybar_,
                     &dx_, &push_, &sa_fac_, &sa_loc_, &x3buf_, &d3_})
    sfree(st_, *p);
  for (int** p : {&xrow_, &xcol_, &cert_, &triples_, &order_, &fpair_ij_, &counter_})
    sfree(st_, *p);
  sfree(st_, S_);
  sfree(st_, sa_state_);
  sfree(st_, hist_bound_);
  sfree(st_, hist_best_);
  sfree(st_, hist_t_);
  if (hSpin_) {
    cudaStreamSynchronize(st_);  // no copy may still target the block
    pinned_put(hSpin_);
  }
  for (void* p : peer_maps_) cudaIpcCloseMemHandle(p);
  if (comm_ && barrier_) {  // no peer may still map my receive buffers
    barrier();
    cudaStreamSynchronize(st_);
  }
  for (auto* p : xbufs_) cudaFree(p);
  sfree(st_, tmaps_);
  if (shard_dev_) cudaFree(shard_dev_);
  sfree(st_, feas_bad_);
  if (rows_before_) cudaFree(rows_before_);
  if (barrier_) cudaFree(barrier_);
  if (theta_buf_) cudaFree(theta_buf_);
  for (auto e : stage_ev_) cudaEventDestroy(e);
  if (join_ev_) cudaEventDestroy(join_ev_);
  if (st2_) cudaStreamDestroy(st2_);
  if (st_) cudaStreamDestroy(st_);
  if (prev >= 0 && prev != dev_) cudaSetDevice(prev);
}

void Engine::ensure_hist(int need) {
  if (need <= hist_cap_) return;
  int cap = std::max(need, 2 * hist_cap_);
  double *nb = nullptr, *nbest = nullptr;
  unsigned long long* nt = nullptr;
  salloc(st_, &nb, cap);
  salloc(st_, &nbest, cap);
  salloc(st_, &nt, 4 * (size_t)cap);
  cuda_check(cudaMemsetAsync(nt, 0, 4 * (size_t)cap * sizeof(unsigned long long), st_),
             "memset");
  if (hist_cap_) {
    cuda_check(cudaMemcpyAsync(nb, hist_bound_, hist_cap_ * 8, cudaMemcpyDeviceToDevice, st_),
               "hist");
    cuda_check(cudaMemcpyAsync(nbest, hist_best_, hist_cap_ * 8, cudaMemcpyDeviceToDevice, st_),
               "hist");
    cuda_check(cudaMemcpyAsync(nt, hist_t_, 4 * (size_t)hist_cap_ * 8, cudaMemcpyDeviceToDevice,
                               st_),
               "hist");
    cuda_check(cudaStreamSynchronize(st_), "hist");
  }
  sfree(st_, hist_bound_);
  sfree(st_, hist_best_);
  sfree(st_, hist_t_);
  hist_bound_ = nb;
  hist_best_ = nbest;
  hist_t_ = nt;
  hist_cap_ = cap;
  if (graph_) {  // the captured X stage writes the history arrays
    cudaGraphExecDestroy(graph_);
    graph_ = nullptr;
  }
}

void Engine::push_scalars() {
  *hSpin_ = hS_;
  cuda_check(cudaMemcpyAsync(S_, hSpin_, sizeof(DevScalars), cudaMemcpyHostToDevice, st_),
             "H2D scalars");
}

void Engine::pull_scalars() {
  cuda_check(cudaMemcpyAsync(hSpin_, S_, sizeof(DevScalars), cudaMemcpyDeviceToHost, st_),
             "D2H scalars");
  cuda_check(cudaStreamSynchronize(st_), "iteration");
  hS_ = *hSpin_;
}

void Engine::nccl_check(ncclResult_t r, const char* what) const {
  if (r != ncclSuccess)
    throw CudaError(std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
}

void Engine::setup_shards(const unsigned char* nccl_id) {
  const int m = m_;
  std::vector<int> pb = world_ > 1 ? shard_plan(m, world_) : std::vector<int>{0, m};
  shard_ = ShardInfo{};
  shard_.world = world_;
  shard_.rank = rank_;
  for (int r = 0; r <= world_; ++r) shard_.pbound[r] = pb[r];
  p_lo_ = pb[rank_];
  p_hi_ = pb[rank_ + 1];
  salloc(st_, &feas_bad_, 1);
  if (world_ == 1) return;
  // fold chunks of my locations
  chunks_me_ = (p_hi_ - p_lo_ + chunk_ - 1) / chunk_;
  // rows_before[f] = sum over pairs f' < f of b(f')
  std::vector<int> rb(fpairs_ + 1, 0);
  for (int i = 0, f = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j, ++f) rb[f + 1] = rb[f] + i;
  dalloc(&rows_before_, rb.size());
  cuda_check(cudaMemcpyAsync(rows_before_, rb.data(), rb.size() * 4, cudaMemcpyHostToDevice, st_),
             "H2D");
  shard_.rows_before = rows_before_;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof id);
  comm_ = cached_comm(id, world_, rank_, dev_);
  shard_.chunk = chunk_;
  cost_scatter_ = env_int("QAPB_COST_SCATTER", 0) != 0 && !ri_;  // the scatter writes the tile layout
  // Receive buffers live here; peers write them directly over NVLink through
  // CUDA IPC mappings (pi from X3 owners, costs from fold owners).
  std::vector<long long> send, recv;
  shard_counts(m, pb, rank_, send, recv);
  xcount_.assign(2 * world_, 0);
  std::vector<cudaIpcMemHandle_t> mine(2 * world_);
  for (int p = 0; p < world_; ++p) {
    if (p == rank_) continue;
    double *sr = nullptr, *gr = nullptr, *d3 = nullptr;
    dalloc(&sr, recv[p]);                                // pi from p
    dalloc(&gr, shard_cost_count(shard_, m, p, rank_));  // costs from p
    dalloc(&d3, shard_cost_count(shard_, m, rank_, p));  // D' of my families' X3 cells in p
    xbufs_.push_back(sr);
    xbufs_.push_back(gr);
    xbufs_.push_back(d3);
    shard_.pi_recv[p] = sr;
    shard_.cost_recv[p] = gr;
    shard_.d3[p] = d3;
    if (is_two_phase() && is_fast()) {  // F2: the fold's remote X3 costs, updated by phase 2
      double* kp = nullptr;
      dalloc(&kp, shard_cost_count(shard_, m, rank_, p));
      xbufs_.push_back(kp);
      shard_.keep[p] = kp;
    }
    // sharded engines start from init_coefficients (D' = 0, rlt2.cpp:87)
    cuda_check(cudaMemsetAsync(d3, 0, shard_cost_count(shard_, m, rank_, p) * sizeof(double),
                               st_),
               "memset d3");
    cuda_check(cudaIpcGetMemHandle(&mine[2 * p], sr), "cudaIpcGetMemHandle");
    cuda_check(cudaIpcGetMemHandle(&mine[2 * p + 1], gr), "cudaIpcGetMemHandle");
    xcount_[p] = send[p];
    xcount_[world_ + p] = recv[p];
  }
  // all-gather every rank's handle table through NCCL
  const size_t hb = sizeof(cudaIpcMemHandle_t) * 2 * world_;
  unsigned char *dh = nullptr, *dall = nullptr;
  dalloc(&dh, hb);
  dalloc(&dall, hb * world_);
  cuda_check(cudaMemcpyAsync(dh, mine.data(), hb, cudaMemcpyHostToDevice, st_), "H2D handles");
  nccl_check(nccl().AllGather(dh, dall, hb, ncclUint8, comm_, st_), "allgather handles");
  std::vector<cudaIpcMemHandle_t> all(2 * world_ * world_);
  cuda_check(cudaMemcpyAsync(all.data(), dall, hb * world_, cudaMemcpyDeviceToHost, st_), "D2H");
  cuda_check(cudaStreamSynchronize(st_), "handles");
  cudaFree(dh);
  cudaFree(dall);
  for (int p = 0; p < world_; ++p) {
    if (p == rank_) continue;
    void *sp = nullptr, *gp = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&sp, all[(size_t)p * 2 * world_ + 2 * rank_],
                                    cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle");
    cuda_check(cudaIpcOpenMemHandle(&gp, all[(size_t)p * 2 * world_ + 2 * rank_ + 1],
                                    cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle");
    shard_.pi_send[p] = static_cast<double*>(sp);   // p's pi buffer for my X3 cells
    shard_.cost_send[p] = static_cast<double*>(gp);  // p's cost buffer for my families
    peer_maps_.push_back(sp);
    peer_maps_.push_back(gp);
  }
  dalloc(&barrier_, 1);
  dalloc(&theta_buf_, tiles_);
  dalloc(&shard_dev_, 1);
  cuda_check(cudaMemcpyAsync(shard_dev_, &shard_, sizeof shard_, cudaMemcpyHostToDevice, st_),
             "H2D shard");
  cuda_check(cudaStreamSynchronize(st_), "H2D shard");
}

// Cross-rank barrier on the engine stream: after it, every rank's earlier
// kernels, and with them their peer stores, are complete.
void Engine::barrier() {
  nccl_check(nccl().AllReduce(barrier_, barrier_, 1, ncclInt, ncclMax, comm_, st_), "barrier");
}

// Steady sharded Z stage (location ownership, transfers fused into kernels
// over NVLink peer memory, ShardInfo in kernels.h):
//   fold of every triple for my pa chunks; the new cost of each remote X3
//   cell is stored into its owner's buffer; barrier;
//   Z-LAPs of my tile runs: remote-folded X3 cells take their cost from that
//   buffer before solving; their slack is stored into the fold owners' pi
//   buffers after solving;
//   theta segments re-assembled on every rank (this collective is also the
//   barrier that orders those pi stores before the next fold).
void Engine::enqueue_sharded_z(int it) {
  const bool fast = is_fast();
  double* costs = (fast && it > 0) ? incz_ : d_;
  const int S = (int)stage_ev_.size();
  cuda_check(cudaMemsetAsync(counter_, 0, (S + 2) * sizeof(int), st_), "memset counters");
  if (it > 0) {
    FoldParams f = fold_params(-1);
    f.nchunks = chunks_me_;
    f.shard = shard_dev_;
    f.keep_cost = is_two_phase() && fast ? 1 : 0;
    kbegin(QAPB_K_ZFOLD, st_);
    kcheck(launch_zfold(f, st_), "z-fold");
    kend(st_);
    kbegin(QAPB_K_XCHG, st_);
    barrier();  // costs have landed in every X3 owner's buffer
    kend(st_);
    ++launches_;
    if (cost_scatter_) {  // into the tile layout the Z-LAPs load (else they patch per row)
      kbegin(QAPB_K_XCHG, st_);
      kcheck(launch_x3_cost_scatter(m_, shard_, triples_, costs, st_), "x3 cost scatter");
      kend(st_);
      ++launches_;
    }
  }
  // Z-LAPs of my runs: one run of rl tiles per facility-pair block
  auto zlaps = [&](double* values, const double* theta_ref, int counter, bool patch) {
    const int rl = (p_hi_ - p_lo_) * (m_ - 1);
    BatchLapParams p{};
    p.costs = costs;
    p.m = m_ - 2;
    p.count = fpairs_ * rl;
    p.counter = counter_ + counter;
    p.stop = &S_->stop;
    p.stop_w = &S_->stop;
    p.values = values;
    p.theta_ref = theta_ref;
    p.pi = piz_;
    p.err_tile = &S_->err_tile;
    p.run_len = rl;
    p.run_stride = lpairs_;
    p.run_off = p_lo_ * (m_ - 1);
    p.sh = shard_dev_;
    p.fpair_ij = fpair_ij_;
    p.patch = (patch && !cost_scatter_) ? 1 : 0;
    if (split_) {  // local X3 members: slack into the fold-order split buffer
      p.x3buf = x3buf_;
      p.x3_group = x3_group_;
      p.x3_ngroups = x3_ngroups_;
    }
    if (ri_) {  // RI layout: tiles by global index through the tensor maps
      p.tmap_cost = tmaps_ + (costs == d_ ? 0 : 128);
      p.tmap_pi = tmaps_ + 256;
    }
    kbegin(QAPB_K_ZLAP, st_);
    kcheck(launch_lap_batch(p, st_), "z-stage");
    kend(st_);
    ++launches_;
  };
  if (!is_two_phase()) {
    zlaps(theta_, nullptr, S, it > 0);
  } else {  // rlt2.cpp:328-336 across the ranks
    zlaps(theta1_, nullptr, S, it > 0);
    kbegin(QAPB_K_XCHG, st_);
    barrier();  // every rank's phase-1 pi has landed in the fold owners' buffers
    kend(st_);
    FoldParams f = fold_params(-1);
    f.nchunks = chunks_me_;
    f.shard = shard_dev_;
    f.costs = costs;
    kbegin(QAPB_K_PHASE2, st_);
    kcheck(launch_phase2_ri(f, costs == d_, st_), "phase-2");
    kend(st_);
    kbegin(QAPB_K_XCHG, st_);
    barrier();  // the redistributed X3 costs have landed in their owners' buffers
    kend(st_);
    launches_ += 2;
    zlaps(theta_, theta1_, S + 1, true);
    kbegin(QAPB_K_XCHG, st_);  // one verdict on a phase-2 regression for every rank
    nccl_check(nccl().AllReduce(&S_->err_tile, &S_->err_tile, 1, ncclInt, ncclMin, comm_, st_),
               "allreduce err_tile");
    kcheck(launch_err_to_stop(S_, st_), "phase-2 verdict");
    kend(st_);
    ++launches_;
  }
  kbegin(QAPB_K_XCHG, st_);
  kcheck(launch_theta_xfer(m_, theta_, theta_buf_, shard_, 1, st_), "theta pack");
  nccl_check(nccl().GroupStart(), "group");
  for (int r = 0, seg = 0; r < world_; ++r) {
    const int c = fpairs_ * (shard_.pbound[r + 1] - shard_.pbound[r]) * (m_ - 1);
    nccl_check(nccl().Broadcast(theta_buf_ + seg, theta_buf_ + seg, c, ncclDouble, r, comm_, st_),
               "theta broadcast");
    seg += c;
  }
  nccl_check(nccl().GroupEnd(), "group");
  kcheck(launch_theta_xfer(m_, theta_, theta_buf_, shard_, 0, st_), "theta unpack");
  kend(st_);
  launches_ += 2;
}

void Engine::plan_pipeline() {
  // Stage k folds the triples whose first facility is in [A_k, A_k+1)
  // (contiguous in lexicographic order) and then completes every facility
  // pair (i, j) with i in that range: no later triple touches those tiles, so
  // their Z-LAPs may overwrite pi(z) in place while stage k+1 folds.
  const int m = m_;
  const int K = std::max(1, std::min(m - 1, env_int("QAPB_ZSTAGES", 1)));
  const int total = (m - 1) * m / 2;  // facility pairs
  stage_a_.assign(1, 0);
  int acc = 0;
  for (int a = 0; a < m - 1; ++a) {
    acc += m - 1 - a;
    if ((int)stage_a_.size() < K && acc * K >= total * (int)stage_a_.size() && a + 1 < m - 1)
      stage_a_.push_back(a + 1);
  }
  stage_a_.push_back(m - 1);
  auto c2 = [](int x) { return x >= 2 ? x * (x - 1) / 2 : 0; };
  auto tri_before = [&](int a) {  // triples whose first facility is < a
    int t = 0;
    for (int x = 0; x < a; ++x) t += c2(m - 1 - x);
    return t;
  };
  auto fp_first = [&](int i) { return i * m - i * (i + 1) / 2; };  // fpair(i, i+1)
  const int S = (int)stage_a_.size() - 1;
  stage_t0_.resize(S);
  stage_tiles_.resize(S);
  stage_z0_.resize(S);
  stage_zn_.resize(S);
  for (int k = 0; k < S; ++k) {
    const int A0 = stage_a_[k], A1 = stage_a_[k + 1];
    stage_t0_[k] = tri_before(A0);
    stage_tiles_[k] = tri_before(A1) - stage_t0_[k];
    stage_z0_[k] = fp_first(A0) * lpairs_;
    stage_zn_[k] = fp_first(A1) * lpairs_ - stage_z0_[k];
  }
  stage_ev_.resize(S);
  for (auto& e : stage_ev_)
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming), "event");
}

void Engine::split_gather() {
  if (!split_) return;
  kcheck(launch_x3_sync(m_, chunk_, world_ > 1 ? chunks_me_ : nchunks_, triples_, ntriples_,
                            p_lo_, p_hi_, d_, d3_, 1, st_, ri_ ? 1 : 0),
             "x3 gather");
  d_stale_ = false;
}

// the tile-layout D' of the X3 members is stale after a split fold
void Engine::split_scatter() const {
  if (!split_ || !d_stale_) return;
  kcheck(launch_x3_sync(m_, chunk_, world_ > 1 ? chunks_me_ : nchunks_, triples_, ntriples_,
                            p_lo_, p_hi_, d_, d3_, 0, st_, ri_ ? 1 : 0),
             "x3 scatter");
  cuda_check(cudaStreamSynchronize(st_), "x3 scatter");
  d_stale_ = false;
}

void Engine::enqueue_zlap(double* costs, int t0, int count, double* values,
                          const double* theta_ref, int slot, cudaStream_t st) {
  if (count <= 0) return;
  const size_t esz = (size_t)esz_;
  BatchLapParams p{};
  p.costs = costs + (size_t)t0 * esz;
  p.m = m_ - 2;
  p.count = count;
  p.counter = counter_ + slot;
  p.stop = &S_->stop;
  p.stop_w = &S_->stop;
  p.values = values + t0;
  p.pi = piz_ + (size_t)t0 * esz;
  p.theta_ref = theta_ref ? theta_ref + t0 : nullptr;
  p.err_tile = &S_->err_tile;
  p.tile_base = t0;
  if (t0 == 0 && !theta_ref) {  // the iteration's first Z-LAP launch: z_ms starts here
    p.tstamp = hist_t_;
    p.iter = &S_->iter;
  }
  if (ri_) {  // tiles by global index through the tensor maps
    p.costs = costs;
    p.pi = piz_;
    p.tmap_cost = tmaps_ + (costs == d_ ? 0 : 128);
    p.tmap_pi = tmaps_ + 256;
  }
  if (split_) {  // X3 split (FoldParams::x3buf)
    p.nx3 = (size_t)ntriples_ * x3_ngroups_ * lpairs_ * x3_group_;
    p.x3buf = x3buf_;
    p.costs_w = costs + (size_t)t0 * esz;
    p.x3_group = x3_group_;
    p.x3_ngroups = x3_ngroups_;
    p.fpair_ij = fpair_ij_;
    p.patch = (cur_iter_ > 0 && split_mode_ == 1) ? 1 : 0;
  }
  kbegin(QAPB_K_ZLAP, st);
  kcheck(launch_lap_batch(p, st), "z-stage");
  kend(st);
  ++launches_;
}

FoldParams Engine::fold_params(int stage) const {
  FoldParams f{};
  f.m = m_;
  f.triples = triples_ + 3 * (size_t)(stage < 0 ? 0 : stage_t0_[stage]);
  f.ntriples = stage < 0 ? ntriples_ : stage_tiles_[stage];
  f.tri0 = stage < 0 ? 0 : stage_t0_[stage];
  f.chunk = chunk_;
  f.nchunks = nchunks_;
  f.kz = cfg_.kappa_z_upper;
  f.phi = cfg_.phi_split;
  f.fast = is_fast();
  f.d = d_;
  f.piz = piz_;
  f.incz = incz_;
  f.push = push_;
  f.sa_fac = sa_fac_;
  f.sa_loc = sa_loc_;
  f.stop = &S_->stop;
  if (split_) {
    f.x3buf = x3buf_;
    f.d3 = d3_;
    f.x3mode = split_mode_;
    f.x3_group = x3_group_;
    f.x3_ngroups = x3_ngroups_;
  }
  if (f.tri0 == 0 && f.ntriples == ntriples_) f.order = order_;
  f.ri = ri_ ? 1 : 0;
  f.tmap_rows = (ri_ && tmaps_) ? tmaps_ + 384 : nullptr;
  f.rows_cp = (world_ > 1 && is_two_phase()) ? 1 : 0;  // see launch_zfold
  f.nz = nd_;
  if (split_) {
    const int nch = world_ > 1 ? chunks_me_ : nchunks_;
    f.nx3 = (size_t)ntriples_ * x3_ngroups_ * lpairs_ * x3_group_;
    f.nd3 = (size_t)ntriples_ * nch * lpairs_ * chunk_;
  }
  return f;
}

// stage_z, rlt2.cpp:301-338.  Steady F/S iterations run fold+Z-LAP as the
// stage pipeline; iteration 0 (no fold) solves every tile at once.
void Engine::enqueue_stage_z(int it) {
  double* costs = (is_fast() && it > 0) ? incz_ : d_;
  double* vals1 = is_two_phase() ? theta1_ : theta_;
  const int S = (int)stage_ev_.size();
  cuda_check(cudaMemsetAsync(counter_, 0, (S + 2) * sizeof(int), st_), "memset counters");
  if (it > 0) {
    for (int k = 0; k < S; ++k) {
      if (stage_tiles_[k] > 0) {  // z-level fold of this stage, rlt2.cpp:269-298
        const FoldParams f = fold_params(k);
        kbegin(QAPB_K_ZFOLD, st_);
        kcheck(launch_zfold(f, st_), "z-fold");
        kend(st_);
        ++launches_;
      }
      cuda_check(cudaEventRecord(stage_ev_[k], st_), "event record");
      cuda_check(cudaStreamWaitEvent(st2_, stage_ev_[k], 0), "stream wait");
      enqueue_zlap(costs, stage_z0_[k], stage_zn_[k], vals1, nullptr, k, st2_);
    }
    cuda_check(cudaEventRecord(join_ev_, st2_), "event record");
    cuda_check(cudaStreamWaitEvent(st_, join_ev_, 0), "stream wait");
  } else {
    enqueue_zlap(costs, 0, tiles_, vals1, nullptr, S, st_);
  }
  if (is_two_phase()) {  // rlt2.cpp:328-336
    FoldParams f = fold_params(-1);
    f.costs = costs;
    kbegin(QAPB_K_PHASE2, st_);
    cuda_check(ri_ ? launch_phase2_ri(f, costs == d_, st_) : launch_phase2(f, st_), "phase-2");
    kend(st_);
    ++launches_;
    enqueue_zlap(costs, 0, tiles_, theta_, theta1_, S + 1, st_);
  }
}

void Engine::enqueue_iteration(int it) {  // rlt2.cpp:515-530
  const bool inc = is_fast() && it > 0;
  const bool steady = it > 0;
  cur_iter_ = it;
  if (split_ && steady) d_stale_ = true;  // graph replays skip enqueue_stage_z
  if (steady && graph_ && !profiling_) {
    cuda_check(cudaGraphLaunch(graph_, st_), "graph launch");
    launches_ += graph_launches_;
    return;
  }
  const bool capture = steady && it >= 2 && !graph_ && !profiling_ && world_ == 1 &&
                       !env_flag("QAPB_NO_GRAPH") && !sync_check_enabled();
  cudaGraph_t g = nullptr;
  const long long l0 = launches_;
  if (capture)
    cuda_check(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal), "capture");
  if (steady) {  // ascent_update x/y levels, rlt2.cpp:244-262 (z level: enqueue_stage_z)
    XYFoldParams x{};
    x.m = m_;
    x.kx = cfg_.kappa_x;
    x.ky = cfg_.kappa_y;
    x.vph = cfg_.varphi;
    x.pix = pix_;
    x.sa_fac = sa_fac_;
    x.sa_loc = sa_loc_;
    x.dx = dx_;
    x.b = b_;
    x.c = c_;
    x.piy = piy_;
    x.ybar = ybar_;
    x.push = push_;
    x.fpair_ij = fpair_ij_;
    x.stop = &S_->stop;
    kbegin(QAPB_K_XYFOLD, st_);
    kcheck(launch_xyfold(x, tiles_, st_), "xy-fold");
    kend(st_);
    ++launches_;
  }
  if (world_ > 1)
    enqueue_sharded_z(it);
  else
    enqueue_stage_z(it);
  YStageParams y{};
  y.m = m_;
  y.c = c_;
  y.theta = theta_;
  y.ybar = ybar_;
  y.dx = dx_;
  y.inc = inc;
  y.delta = delta_;
  y.piy = piy_;
  y.stop = &S_->stop;
  y.tstamp = hist_t_;
  y.iter = &S_->iter;
  kbegin(QAPB_K_YSTAGE, st_);
  kcheck(launch_ystage(y, st_), "y-stage");
  kend(st_);
  ++launches_;
  XStageParams xs{};
  xs.m = m_;
  xs.delta = delta_;
  xs.b = b_;
  xs.inc = inc;
  xs.fast = is_fast();
  xs.pix = pix_;
  xs.xrow = xrow_;
  xs.xcol = xcol_;
  xs.piy = piy_;
  xs.piz = piz_;
  xs.S = S_;
  xs.hist_bound = hist_bound_;
  xs.hist_best = hist_best_;
  xs.cert = cert_;
  xs.upper_bound = cfg_.upper_bound;
  xs.min_gap = cfg_.min_gap;
  xs.fathom = cfg_.fathom_threshold;
  xs.es_delta = cfg_.early_stop_delta;
  xs.es_window = cfg_.early_stop_window;
  xs.iter_limit = cfg_.iter_limit;
  xs.feas_bad = feas_bad_;
  xs.zp_lo = p_lo_;
  xs.zp_hi = p_hi_;
  xs.ri = ri_ ? 1 : 0;
  xs.tstamp = hist_t_;
  kbegin(QAPB_K_XSTAGE, st_);
  kcheck(launch_xstage(xs, st_), "x-stage");
  if (world_ > 1)  // feasibility needs every rank's pi(z) tiles
    nccl_check(nccl().AllReduce(feas_bad_, feas_bad_, 1, ncclInt, ncclMax, comm_, st_), "allreduce");
  kcheck(launch_xfinish(xs, st_), "x-finish");
  kend(st_);
  launches_ += 2;
  if (sa_dev_) {  // rlt2.cpp:521-523 on the device (kernels.cu sa_device_kernel)
    SaParams sp{};
    sp.m = m_;
    sp.cool_period = cfg_.sa_cool_period;
    sp.fast = is_fast() ? 1 : 0;
    sp.exp_fma = exp_fma_;
    sp.t0_fraction = cfg_.sa_t0_fraction;
    sp.kappa_cap = cfg_.sa_kappa_lb_cap;
    sp.cool_factor = cfg_.sa_cool_factor;
    sp.upper_bound = cfg_.upper_bound;
    kcheck(launch_sa_device(sp, b_, S_, sa_state_, sa_fac_, sa_loc_, st_), "sa step");
    ++launches_;
  }
  if (capture) {
    cuda_check(cudaStreamEndCapture(st_, &g), "end capture");
    cuda_check(cudaGraphInstantiate(&graph_, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    graph_launches_ = (int)(launches_ - l0);
    launches_ = l0;
    cuda_check(cudaGraphLaunch(graph_, st_), "graph launch");
    launches_ += graph_launches_;
  }
}

void Engine::check_phase2() {
  if (hS_.err_tile != INT_MAX) {
    const int t = hS_.err_tile;
    hS_.err_tile = INT_MAX;
    hS_.stop = 0;
    push_scalars();
    throw std::logic_error("phase-2 theta regressed on tile " + std::to_string(t));
  }
}

double Engine::gap() const {  // rlt2.cpp:532-535
  if (!std::isfinite(cfg_.upper_bound) || cfg_.upper_bound == 0) return kInf;
  return (cfg_.upper_bound - hS_.best) / cfg_.upper_bound;
}

// Type-4 SA (rlt2.cpp:477-513).  Draws with std::mt19937_64 /
// uniform_real_distribution / std::exp exactly as the reference; the b drain
// and running update run on the device.
void Engine::sa_perturb() {
  const double nu = hS_.best;
  if (nu <= 0) return;
  if (temp_ <= 0) {
    const double ub = std::isfinite(cfg_.upper_bound) ? cfg_.upper_bound : 1.05 * nu + 1.0;
    temp_ = cfg_.sa_t0_fraction * ub;
  }
  const double cap = cfg_.sa_kappa_lb_cap * nu;
  const int m = m_;
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> amt(2 * m, 0.0);
  double total = 0;
  for (int s = 0; s < 2 * m; ++s) {
    const double kap = U(rng_) * cap;
    const bool accept = U(rng_) < std::exp(-kap / temp_);
    if (accept) {
      amt[s] = kap;
      total += kap;
    }
  }
  if (total > cap)
    for (double& a : amt) a *= cap / total;
  std::vector<double> fac(m), loc(m);
  for (int i = 0; i < m; ++i) fac[i] = amt[i] / m;
  for (int p = 0; p < m; ++p) loc[p] = amt[m + p] / m;
  double drained = 0;
  for (int i = 0; i < m; ++i) drained += fac[i] + loc[i];
  cuda_check(cudaMemcpyAsync(sa_fac_, fac.data(), m * 8, cudaMemcpyHostToDevice, st_), "H2D sa");
  cuda_check(cudaMemcpyAsync(sa_loc_, loc.data(), m * 8, cudaMemcpyHostToDevice, st_), "H2D sa");
  kcheck(launch_sa_apply(m, b_, sa_fac_, sa_loc_, S_, drained, is_fast(), st_), "sa");
  ++launches_;
  const int iter_before = hS_.iter - 1;  // sa_perturb runs before ++iter_
  if ((iter_before + 1) % cfg_.sa_cool_period == 0) temp_ *= cfg_.sa_cool_factor;
  pull_scalars();
}

double Engine::iterate() {
  const DeviceGuard dg(dev_);
  hS_.run_mode = 0;
  hS_.stop = 0;
  push_scalars();
  ensure_hist(hS_.iter + 1);
  enqueue_iteration(hS_.iter);
  pull_scalars();
  if (profiling_) collect_events();
  check_phase2();
  if (cfg_.sa_enabled && !sa_dev_ && !hS_.has_cert) sa_perturb();
  last_rec_ = qapb_record{hS_.iter, hS_.last_bound, gap(), 0, 0, 0};
  stage_times(hS_.iter - 1, &last_rec_.z_ms, &last_rec_.y_ms, &last_rec_.x_ms);
  return hS_.last_bound;
}

// IterationRecord::{z,y,x}_ms of iteration k (0-based), as rlt2.cpp:302-448
// times stage_z / stage_y / stage_x: the CUDA-event timings when profiling is
// on, else the device timestamps the stage kernels store (kernels.h tstamp).
void Engine::stage_times(int k, double* z, double* y, double* x) const {
  if (k < 0) return;
  if ((int)stage_ms_.size() >= 3 * (k + 1)) {
    *z = stage_ms_[3 * k];
    *y = stage_ms_[3 * k + 1];
    *x = stage_ms_[3 * k + 2];
    return;
  }
  if (!hist_t_ || k >= hist_cap_) return;
  unsigned long long t[4] = {0, 0, 0, 0};
  cuda_check(cudaMemcpyAsync(t, hist_t_ + 4 * (size_t)k, sizeof t, cudaMemcpyDeviceToHost, st_),
             "D2H t");
  cuda_check(cudaStreamSynchronize(st_), "D2H t");
  auto ms = [](unsigned long long a, unsigned long long b) {
    return (a && b && b >= a) ? (double)(b - a) * 1e-6 : 0.0;
  };
  *z = ms(t[0], t[1]);
  *y = ms(t[1], t[2]);
  *x = ms(t[2], t[3]);
}

void Engine::fill_records(int from, int to, std::vector<qapb_record>* recs) const {
  if (!recs || to <= from) return;
  std::vector<double> bnd(to - from), bst(to - from);
  cuda_check(cudaMemcpyAsync(bnd.data(), hist_bound_ + from, (to - from) * 8,
                             cudaMemcpyDeviceToHost, st_),
             "D2H hist");
  cuda_check(cudaMemcpyAsync(bst.data(), hist_best_ + from, (to - from) * 8,
                             cudaMemcpyDeviceToHost, st_),
             "D2H hist");
  std::vector<unsigned long long> ts;  // device stage timestamps of these iterations
  if (hist_t_ && to <= hist_cap_) {
    ts.resize(4 * (size_t)(to - from));
    cuda_check(cudaMemcpyAsync(ts.data(), hist_t_ + 4 * (size_t)from, ts.size() * 8,
                               cudaMemcpyDeviceToHost, st_),
               "D2H stage times");
  }
  cuda_check(cudaStreamSynchronize(st_), "D2H hist");
  for (int k = from; k < to; ++k) {
    qapb_record r{};
    r.iteration = k + 1;
    r.bound = bnd[k - from];
    const double best = bst[k - from];
    r.gap = (!std::isfinite(cfg_.upper_bound) || cfg_.upper_bound == 0)
                ? kInf
                : (cfg_.upper_bound - best) / cfg_.upper_bound;
    if ((int)stage_ms_.size() >= 3 * (k + 1)) {
      r.z_ms = stage_ms_[3 * k];
      r.y_ms = stage_ms_[3 * k + 1];
      r.x_ms = stage_ms_[3 * k + 2];
    } else if (!ts.empty()) {
      const unsigned long long* t = ts.data() + 4 * (size_t)(k - from);
      auto ms = [](unsigned long long a, unsigned long long b) {
        return (a && b && b >= a) ? (double)(b - a) * 1e-6 : 0.0;
      };
      r.z_ms = ms(t[0], t[1]);
      r.y_ms = ms(t[1], t[2]);
      r.x_ms = ms(t[2], t[3]);
    }
    recs->push_back(r);
  }
}

void Engine::run(qapb_report* rep, std::vector<qapb_record>* recs, std::vector<int>* cert) {
  const DeviceGuard dg(dev_);
  const auto t0 = std::chrono::steady_clock::now();
  const int from = hS_.iter;
  hS_.run_mode = 1;
  hS_.run_start = hS_.iter;
  hS_.stop = 0;
  hS_.term = QAPB_TERM_ITERATION_LIMIT;
  push_scalars();
  if (hS_.iter < cfg_.iter_limit) {
    int batch = 4;
    while (true) {
      const int remaining = cfg_.iter_limit - hS_.iter;
      const int B = (cfg_.sa_enabled && !sa_dev_) ? 1 : std::max(1, std::min(remaining, batch));
      ensure_hist(hS_.iter + B);
      for (int k = 0; k < B; ++k) enqueue_iteration(hS_.iter + k);
      pull_scalars();
      check_phase2();
      if (cfg_.sa_enabled && !sa_dev_ && !hS_.has_cert) sa_perturb();
      if (hS_.stop || hS_.iter >= cfg_.iter_limit) break;
      batch = std::min(batch * 2, 64);
    }
  }
  const int to = hS_.iter;
  if (profiling_) collect_events();
  if (recs && cfg_.record_history) fill_records(from, to, recs);
  hS_.run_mode = 0;
  hS_.stop = 0;
  push_scalars();
  if (rep) {
    rep->best_bound = hS_.best;
    rep->upper_bound = cfg_.upper_bound;
    rep->gap = gap();
    rep->termination = hS_.term;
    rep->iterations = hS_.iter;
    rep->has_certificate = hS_.has_cert;
    rep->certificate_value = hS_.has_cert ? hS_.cert_val : 0.0;
    rep->n_records = recs ? (int)recs->size() : 0;
    rep->wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  if (cert && hS_.has_cert) *cert = certificate();
  if (to > from) {
    const int k = to - 1;
    double bnd = 0;
    cuda_check(cudaMemcpyAsync(&bnd, hist_bound_ + k, 8, cudaMemcpyDeviceToHost, st_), "D2H");
    cuda_check(cudaStreamSynchronize(st_), "D2H");
    last_rec_ = qapb_record{to, bnd, gap(), 0, 0, 0};
  }
}

std::vector<int> Engine::certificate() const {
  const DeviceGuard dg(dev_);
  std::vector<int> out;
  if (!hS_.has_cert) return out;
  out.resize(m_);
  cuda_check(cudaMemcpyAsync(out.data(), cert_, m_ * sizeof(int), cudaMemcpyDeviceToHost, st_),
             "D2H cert");
  cuda_check(cudaStreamSynchronize(st_), "D2H cert");
  return out;
}

std::vector<int> Engine::x_assignment() const {
  const DeviceGuard dg(dev_);
  std::vector<int> out(m_);
  cuda_check(cudaMemcpyAsync(out.data(), xrow_, m_ * sizeof(int), cudaMemcpyDeviceToHost, st_),
             "D2H xrow");
  cuda_check(cudaStreamSynchronize(st_), "D2H xrow");
  return out;
}

size_t Engine::array_size(int which) const {
  switch (which) {
    case QAPB_ARR_PI_Z: return nd_;
    case QAPB_ARR_PI_Y: return nc_;
    case QAPB_ARR_PI_X: return nb_;
    case QAPB_ARR_STORE_B: return nb_;
    case QAPB_ARR_STORE_C: return nc_;
    case QAPB_ARR_STORE_D: return nd_;
    case QAPB_ARR_THETA: return tiles_;
    case QAPB_ARR_DELTA: return nb_;
    case QAPB_ARR_INCZ: return incz_ ? nd_ : 0;
  }
  throw std::invalid_argument("unknown engine array");
}

// Sharded engines hold pi(z), D' and incz partially (kernels.cu,
// shard_state_mask_kernel): assemble the full array on every rank.  Collective:
// every rank must call it for the same array.
void Engine::assemble_sharded(int which, double* dst) const {
  const DeviceGuard dg(dev_);
  cuda_check(cudaStreamSynchronize(st_), "assemble");
  double* src = which == QAPB_ARR_PI_Z ? piz_ : (which == QAPB_ARR_INCZ ? incz_ : d_);
  if (which == QAPB_ARR_STORE_D) split_scatter();  // local split D' -> tiles
  double* ref = nullptr;  // RI: this rank's array in the reference layout
  if (ri_) {
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&ref), nd_ * sizeof(double), st_),
               "cudaMallocAsync");
    kcheck(launch_z_relayout(m_, src, ref, 0, st_), "relayout");
    src = ref;
  }
  if (which == QAPB_ARR_STORE_D) {
    kcheck(launch_shard_state_scatter(m_, shard_, triples_, src, 0, st_), "d3 scatter");
  } else if (which == QAPB_ARR_INCZ && hS_.iter >= 2) {  // a fold has stored costs
    kcheck(launch_shard_state_scatter(m_, shard_, triples_, src, 1, st_), "cost scatter");
  }
  unsigned long long* buf = nullptr;
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&buf), nd_ * sizeof(double), st_),
             "cudaMallocAsync");
  kcheck(launch_shard_state_mask(m_, shard_, src, buf, which == QAPB_ARR_STORE_D ? 1 : 0, st_),
             "state mask");
  nccl_check(nccl().AllReduce(buf, buf, nd_, ncclUint64, ncclSum, comm_, st_), "assemble");
  cuda_check(cudaMemcpyAsync(dst, buf, nd_ * sizeof(double), cudaMemcpyDefault, st_), "D2H");
  cuda_check(cudaFreeAsync(buf, st_), "cudaFreeAsync");
  if (ref) cuda_check(cudaFreeAsync(ref, st_), "cudaFreeAsync");
  cuda_check(cudaStreamSynchronize(st_), "assemble");
}

void Engine::get_array(int which, double* dst, size_t count) const {
  const DeviceGuard dg(dev_);
  const size_t n = array_size(which);
  if (count != n) throw std::invalid_argument("array size mismatch");
  if (world_ > 1 && n &&
      (which == QAPB_ARR_PI_Z || which == QAPB_ARR_STORE_D || which == QAPB_ARR_INCZ)) {
    assemble_sharded(which, dst);
    return;
  }
  const double* src = nullptr;
  switch (which) {
    case QAPB_ARR_PI_Z: src = piz_; break;
    case QAPB_ARR_PI_Y: src = piy_; break;
    case QAPB_ARR_PI_X: src = pix_; break;
    case QAPB_ARR_STORE_B: src = b_; break;
    case QAPB_ARR_STORE_C: src = c_; break;
    case QAPB_ARR_STORE_D:
      split_scatter();
      src = d_;
      break;
    case QAPB_ARR_THETA: src = theta_; break;
    case QAPB_ARR_DELTA: src = delta_; break;
    case QAPB_ARR_INCZ: src = incz_; break;
  }
  // dst may be host or device memory (device snapshots, store.cu)
  if (n && ri_ && (which == QAPB_ARR_PI_Z || which == QAPB_ARR_STORE_D || which == QAPB_ARR_INCZ)) {
    // back to the reference layout (StoreIndex) on the way out
    double* tmp = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * sizeof(double), st_),
               "cudaMallocAsync");
    kcheck(launch_z_relayout(m_, src, tmp, 0, st_), "relayout");
    cuda_check(cudaMemcpyAsync(dst, tmp, n * sizeof(double), cudaMemcpyDefault, st_), "D2H array");
    cuda_check(cudaFreeAsync(tmp, st_), "cudaFreeAsync");
    cuda_check(cudaStreamSynchronize(st_), "D2H array");
    return;
  }
  // on the engine's stream and completed before return: dst may be device
  // memory (a device store), where a legacy-stream copy would return early
  if (n) {
    cuda_check(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDefault, st_),
               "D2H array");
    cuda_check(cudaStreamSynchronize(st_), "D2H array");
  }
}

// ---- measurement hooks ---------------------------------------------------
void Engine::kbegin(int kind, cudaStream_t st) {
  if (!profiling_) return;
  if (ev_pool_.size() < 2) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "cudaEventCreate");
      ev_pool_.push_back(e);
    }
  }
  ev_open_ = ev_pool_.back();
  ev_pool_.pop_back();
  kind_open_ = kind;
  cuda_check(cudaEventRecord(ev_open_, st), "cudaEventRecord");
}

void Engine::kend(cudaStream_t st) {
  if (!profiling_ || kind_open_ < 0) return;
  cudaEvent_t b = ev_pool_.back();
  ev_pool_.pop_back();
  cuda_check(cudaEventRecord(b, st), "cudaEventRecord");
  pending_.push_back(PendingEvent{kind_open_, cur_iter_, ev_open_, b});
  kind_open_ = -1;
}

void Engine::collect_events() {
  for (auto& pe : pending_) {
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, pe.a, pe.b), "cudaEventElapsedTime");
    kms_[pe.kind] += ms;
    kcnt_[pe.kind] += 1;
    const int stage = (pe.kind == QAPB_K_ZLAP || pe.kind == QAPB_K_PHASE2)
                          ? 0
                          : (pe.kind == QAPB_K_YSTAGE ? 1 : (pe.kind == QAPB_K_XSTAGE ? 2 : -1));
    if (stage >= 0) {
      if ((int)stage_ms_.size() < 3 * (pe.iter + 1)) stage_ms_.resize(3 * (pe.iter + 1), 0.0);
      stage_ms_[3 * pe.iter + stage] += ms;
    }
    ev_pool_.push_back(pe.a);
    ev_pool_.push_back(pe.b);
  }
  pending_.clear();
}

void Engine::enqueue(int iters) {
  const DeviceGuard dg(dev_);
  if (cfg_.sa_enabled && !sa_dev_)
    throw std::invalid_argument("enqueue: SA needs a host step per iteration; use iterate()");
  if (iters <= 0) return;
  if (hS_.run_mode || hS_.stop) {
    hS_.run_mode = 0;
    hS_.stop = 0;
    push_scalars();
  }
  ensure_hist(hS_.iter + iters);
  for (int k = 0; k < iters; ++k) enqueue_iteration(hS_.iter + k);
  hS_.iter += iters;  // host view; refreshed by synchronize()
}

void Engine::synchronize() {
  const DeviceGuard dg(dev_);
  pull_scalars();
  if (profiling_) collect_events();
  check_phase2();
}

void Engine::history(int from, int count, double* bounds, double* best) const {
  const DeviceGuard dg(dev_);
  if (from < 0 || count < 0 || from + count > hS_.iter)
    throw std::invalid_argument("history: range outside completed iterations");
  if (!count) return;
  if (bounds)
    cuda_check(cudaMemcpyAsync(bounds, hist_bound_ + from, count * 8, cudaMemcpyDeviceToHost,
                               st_),
               "D2H");
  if (best)
    cuda_check(cudaMemcpyAsync(best, hist_best_ + from, count * 8, cudaMemcpyDeviceToHost, st_),
               "D2H");
  cuda_check(cudaStreamSynchronize(st_), "D2H");
}

double Engine::time_kernel(int kind, int reps) {
  const DeviceGuard dg(dev_);
  cuda_check(cudaStreamSynchronize(st_), "sync");
  cudaEvent_t a, b;
  cuda_check(cudaEventCreate(&a), "event");
  cuda_check(cudaEventCreate(&b), "event");
  hS_.stop = 0;
  hS_.run_mode = 0;
  push_scalars();
  const int S = (int)stage_ev_.size();
  double* costs = is_fast() ? incz_ : d_;
  auto one = [&]() {
    switch (kind) {
      case QAPB_K_ZFOLD: {
        FoldParams f = fold_params(-1);
        kcheck(launch_zfold(f, st_), "z-fold");
        break;
      }
      case QAPB_K_PHASE2: {
        FoldParams f = fold_params(-1);
        f.costs = costs;
        kcheck(launch_phase2(f, st_), "phase-2");
        break;
      }
      case QAPB_K_ZLAP:
        cuda_check(cudaMemsetAsync(counter_, 0, (S + 2) * sizeof(int), st_), "memset");
        enqueue_zlap(costs, 0, tiles_, theta_, nullptr, S, st_);
        break;
      default:
        throw std::invalid_argument("time_kernel: unsupported kernel kind");
    }
  };
  one();  // warm
  cuda_check(cudaEventRecord(a, st_), "event");
  for (int r = 0; r < reps; ++r) one();
  cuda_check(cudaEventRecord(b, st_), "event");
  cuda_check(cudaEventSynchronize(b), "sync");
  float ms = 0;
  cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / std::max(1, reps);
}

void Engine::set_profiling(bool on) {
  const DeviceGuard dg(dev_);
  if (on == profiling_) return;
  cuda_check(cudaStreamSynchronize(st_), "sync");
  if (profiling_) collect_events();
  profiling_ = on;
}

void Engine::kernel_times(double* ms, long long* launches, bool reset) {
  const DeviceGuard dg(dev_);
  cuda_check(cudaStreamSynchronize(st_), "sync");
  cuda_check(cudaStreamSynchronize(st2_), "sync");
  collect_events();
  for (int k = 0; k < QAPB_K_COUNT; ++k) {
    if (ms) ms[k] = kms_[k];
    if (launches) launches[k] = kcnt_[k];
    if (reset) {
      kms_[k] = 0;
      kcnt_[k] = 0;
    }
  }
}

}  // namespace qapb

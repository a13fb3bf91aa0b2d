// engine.h — device-resident RLT2 dual-ascent engine (host side, C++).
//
// Mirrors qap::AscentEngine (rlt2.hpp:151-213): same state, same stage order
// (iterate, rlt2.cpp:515-530), same run() termination (rlt2.cpp:544-588), but
// all O(n^4)..O(n^6) state lives in HBM and a run() enqueues batches of
// iterations with no host round trip (device-side stop flag); the host only
// touches the device between batches, or once per iteration when SA is on
// (the Type-4 draws use the reference's own RNG, rlt2.cpp:477-513).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/qapb200.h"
#include "kernels.h"

namespace qapb {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

// Sets the engine's device for the scope of an entry point and restores the
// caller's current device afterwards (engines of several devices may be
// driven from one thread).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

class Engine {
 public:
  // AscentEngine(CoefficientStore, cfg) (rlt2.cpp:207-230); d == nullptr
  // means D' = 0.
  Engine(int m, const double* b, const double* c, const double* d, double offset,
         const qapb_config& cfg);
  // AscentEngine(init_coefficients(inst), cfg): store built on the device.
  Engine(int n, const double* flow, const double* dist, const double* linear,
         const qapb_config& cfg, int rank = 0, int world = 1,
         const unsigned char* nccl_id = nullptr);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  double iterate();                                  // rlt2.cpp:515-530
  void run(qapb_report* rep, std::vector<qapb_record>* recs, std::vector<int>* cert);

  int m() const { return m_; }
  int device() const { return dev_; }
  int iteration() const { return hS_.iter; }
  double best_bound() const { return hS_.best; }
  double gap() const;                                // rlt2.cpp:532-535
  bool has_certificate() const { return hS_.has_cert != 0; }
  double certificate_value() const { return hS_.cert_val; }
  double offset() const { return hS_.offset; }
  bool is_fast() const { return cfg_.variant == QAPB_F1 || cfg_.variant == QAPB_F2; }
  bool is_two_phase() const { return cfg_.variant == QAPB_F2 || cfg_.variant == QAPB_S2; }
  std::vector<int> certificate() const;
  std::vector<int> x_assignment() const;
  size_t array_size(int which) const;
  void get_array(int which, double* dst, size_t count) const;
  qapb_record last_record() const { return last_rec_; }
  long long launches() const { return launches_; }

  // measurement / device-loop hooks (qapb_engine_enqueue & co.)
  void enqueue(int iters);
  void synchronize();
  void set_profiling(bool on);
  void kernel_times(double* ms, long long* launches, bool reset);
  void history(int from, int count, double* bounds, double* best) const;
  double time_kernel(int kind, int reps);

  // device pointers for in-process consumers (bench / multi-GPU layer)
  double* dev_d() const { return d_; }
  double* dev_piz() const { return piz_; }
  cudaStream_t stream() const { return st_; }

 private:
  void alloc();
  void init_state();
  void enqueue_iteration(int iter_index);
  void enqueue_stage_z(int iter_index);
  void enqueue_zlap(double* costs, int t0, int count, double* values, const double* theta_ref,
                    int counter_slot, cudaStream_t st);
  void plan_pipeline();
  void ensure_hist(int need);
  void pull_scalars();
  void push_scalars();
  void sa_perturb();                                 // rlt2.cpp:477-513 (host draws)
  void check_phase2();
  void fill_records(int from, int to, std::vector<qapb_record>* recs) const;
  void build_graph();
  void kbegin(int kind, cudaStream_t st);
  void kend(cudaStream_t st);
  FoldParams fold_params(int stage) const;
  void collect_events();

  struct PendingEvent {
    int kind, iter;
    cudaEvent_t a, b;
  };
  bool profiling_ = false;
  int cur_iter_ = 0;
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<PendingEvent> pending_;
  cudaEvent_t ev_open_ = nullptr;
  int kind_open_ = -1;
  double kms_[QAPB_K_COUNT] = {0};
  long long kcnt_[QAPB_K_COUNT] = {0};
  std::vector<double> stage_ms_;  // per iteration: z, y, x

  // multi-GPU: facility-range ownership + NCCL exchanges
  int rank_ = 0, world_ = 1;
  ncclComm_t comm_ = nullptr;
  ShardInfo shard_{};
  ShardInfo* shard_dev_ = nullptr;
  std::vector<double*> xbufs_;  // all exchange buffers (owned)
  std::vector<long long> xcount_;  // doubles per peer in one exchange
  int* feas_bad_ = nullptr;
  int p_lo_ = 0, p_hi_ = 0, chunks_me_ = 0;  // my first locations / fold chunks
  int* rows_before_ = nullptr;
  double* theta_buf_ = nullptr;
  void barrier();
  void assemble_sharded(int which, double* dst) const;
  // single-GPU X3 split (kernels.h FoldParams::x3buf)
  void split_gather();
  void split_scatter() const;
  bool split_ = false;
  int split_mode_ = 0;
  // z arrays in the row-interleaved layout (kernels.h z_ri_offset); Z-LAP
  // tiles move by 3-D TMA tensor copies: tmaps_ = {d, incz, pi(z)} maps + the fold's 2-D pi(z) row map
  bool ri_ = false;
  unsigned char* tmaps_ = nullptr;
  bool cost_scatter_ = false;  // sharded: scatter remote X3 costs before the Z-LAPs
  int x3_group_ = 0, x3_ngroups_ = 0;
  mutable bool d_stale_ = false;
  double* x3buf_ = nullptr;
  double* d3_ = nullptr;
  std::vector<void*> peer_maps_;  // IPC-mapped peer receive buffers
  int* barrier_ = nullptr;
  void setup_shards(const unsigned char* nccl_id);
  void enqueue_sharded_z(int it);
  void nccl_check(ncclResult_t r, const char* what) const;

  int m_, dev_;
  qapb_config cfg_;
  int tiles_, esz_, fpairs_, lpairs_, ntriples_, chunk_, nchunks_;
  size_t nb_, nc_, nd_;
  cudaStream_t st_ = nullptr;
  // Z pipeline: fold stage k (triples with first facility in [A_k, A_k+1)) on
  // st_, then the Z-LAPs of the facility pairs it completed on st2_, which
  // overlap fold stage k+1.
  cudaStream_t st2_ = nullptr;
  std::vector<int> stage_a_;                 // stage boundaries in first facility
  std::vector<int> stage_t0_, stage_tiles_;  // triple range per stage
  std::vector<int> stage_z0_, stage_zn_;     // tile range per stage
  std::vector<cudaEvent_t> stage_ev_;
  cudaEvent_t join_ev_ = nullptr;
  double *b_ = nullptr, *c_ = nullptr, *d_ = nullptr, *piz_ = nullptr, *incz_ = nullptr;
  double *piy_ = nullptr, *pix_ = nullptr, *theta_ = nullptr, *theta1_ = nullptr;
  double *delta_ = nullptr, *ybar_ = nullptr, *dx_ = nullptr, *push_ = nullptr;
  double *sa_fac_ = nullptr, *sa_loc_ = nullptr;
  int *xrow_ = nullptr, *xcol_ = nullptr, *cert_ = nullptr, *triples_ = nullptr;
  int* order_ = nullptr;  // fold processing order (FoldParams::order); null = lexicographic
  int *fpair_ij_ = nullptr, *counter_ = nullptr;  // counter_: one per Z launch
  DevScalars* S_ = nullptr;
  double *hist_bound_ = nullptr, *hist_best_ = nullptr;
  unsigned long long* hist_t_ = nullptr;  // 4 device timestamps per iteration (kernels.h)
  int hist_cap_ = 0;
  void stage_times(int k, double* z, double* y, double* x) const;
  void kcheck(cudaError_t e, const char* what) const;
  DevScalars* hSpin_ = nullptr;  // pinned mirror for async copies
  DevScalars hS_{};
  std::mt19937_64 rng_;  // host SA (QAPB_HOST_SA=1); the device SA keeps its own state
  bool sa_dev_ = false;
  int exp_fma_ = 1;  // glibc exp build the device SA restates (kernels.h)
  SaState* sa_state_ = nullptr;
  double temp_ = 0;
  qapb_record last_rec_{};
  long long launches_ = 0;
  cudaGraphExec_t graph_ = nullptr;
  int graph_launches_ = 0;
};

}  // namespace qapb

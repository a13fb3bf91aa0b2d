// store.cu — device-resident CoefficientStore and collapse_store on the B200
// (branch-and-bound node evaluation without host round
// trips).  A parent's warm-start snapshot stays in HBM; each child store is
// folded from it on the device (collapse_store, rlt2.cpp:109-182) and handed
// to a new engine device-to-device.
//
// Parity: collapse_store accumulates into C' in tile order; every output C'
// entry receives at most two contributions (one from the tile pairing the
// fixed facility with its first facility, one from its own tile's cell
// (fac, loc)), so the kernel adds them in the same tile order and keeps the
// reference's zero-skip rules, which makes the result bitwise identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "store.h"

namespace qapb {

namespace {

__device__ __forceinline__ void unfpair(int m, int fp, int* i, int* j) {
  int a = 0, acc = 0;
  while (fp >= acc + (m - 1 - a)) {
    acc += m - 1 - a;
    ++a;
  }
  *i = a;
  *j = a + 1 + (fp - acc);
}

// b' = (b + c[i,p,fac,loc]) + c[fac,loc,i,p]          rlt2.cpp:119-127
__global__ void collapse_b_kernel(int m, int fac, int loc, const double* __restrict__ b,
                                  const double* __restrict__ c, double* __restrict__ ob) {
  const int mc = m - 1;
  const DIdx ix(m);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= mc * mc) return;
  const int I = e / mc, P = e - I * mc;
  const int i = I + (I >= fac), p = P + (P >= loc);
  ob[e] = dadd(dadd(b[(size_t)i * m + p], c[ix.cidx(i, p, fac, loc)]), c[ix.cidx(fac, loc, i, p)]);
}

// C' entries: copy-through (rlt2.cpp:128-141) plus the two folds of D' cells
// (rlt2.cpp:150-162 and 166-170), added in tile order
__global__ void collapse_c_kernel(int m, int fac, int loc, const double* __restrict__ c,
                                  const double* __restrict__ d, double* __restrict__ oc) {
  const int mc = m - 1;
  const DIdx ix(m), ox(mc);
  const size_t total = (size_t)mc * mc * (mc - 1) * (mc - 1);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    // e = cidx(I,P,J,Q) in the child: ((I*mc+P)*(mc-1) + Jl)*(mc-1) + Ql
    const int Ql = (int)(e % (mc - 1));
    const size_t r1 = e / (mc - 1);
    const int Jl = (int)(r1 % (mc - 1));
    const int IP = (int)(r1 / (mc - 1));
    const int I = IP / mc, P = IP - I * mc;
    const int J = Jl + (Jl >= I), Q = Ql + (Ql >= P);
    const int i = I + (I >= fac), p = P + (P >= loc), j = J + (J >= fac), q = Q + (Q >= loc);
    double v = c[ix.cidx(i, p, j, q)];
    if (m >= 3) {
      // fold 1: tile of facility pair {fac, i} with fac at loc, i at p; cell (j, q)
      const int t2 = fac < i ? ix.tile(fac, i, loc, p) : ix.tile(i, fac, p, loc);
      const double v2 = fac < i ? d[(size_t)t2 * ix.esz + ix.cell(fac, i, loc, p, j, q)]
                                : d[(size_t)t2 * ix.esz + ix.cell(i, fac, p, loc, j, q)];
      // fold 2: tile (i, j, p, q) itself (i < j only), cell (fac, loc); added even if 0
      if (i < j) {
        const int t3 = ix.tile(i, j, p, q);
        const double v3 = d[(size_t)t3 * ix.esz + ix.cell(i, j, p, q, fac, loc)];
        if (t2 < t3) {
          if (v2 != 0) v = dadd(v, v2);
          v = dadd(v, v3);
        } else {
          v = dadd(v, v3);
          if (v2 != 0) v = dadd(v, v2);
        }
      } else if (v2 != 0) {
        v = dadd(v, v2);
      }
    }
    oc[e] = v;
  }
}

// D' cells of surviving tiles: reindexed copy, zeros as +0 (rlt2.cpp:163-178)
__global__ void collapse_d_kernel(int m, int fac, int loc, const double* __restrict__ d,
                                  double* __restrict__ od) {
  const int mc = m - 1;
  const DIdx ix(m), ox(mc);
  const int otiles = mc * (mc - 1) / 2 * ox.lpairs;
  for (int t = blockIdx.x; t < otiles; t += gridDim.x) {
    const int fp = t / ox.lpairs, lp = t - fp * ox.lpairs;
    int I, J, P, Q;
    unfpair(mc, fp, &I, &J);
    ox.unlpair(lp, &P, &Q);
    const int i = I + (I >= fac), j = J + (J >= fac), p = P + (P >= loc), q = Q + (Q >= loc);
    const double* src = d + (size_t)ix.tile(i, j, p, q) * ix.esz;
    double* dst = od + (size_t)t * ox.esz;
    const int lo = min(P, Q), hi = max(P, Q);
    for (int e = threadIdx.x; e < ox.esz; e += blockDim.x) {
      const int Kl = e / (mc - 2), Rl = e - Kl * (mc - 2);
      // child cell (Kl, Rl) -> child (K, R) -> parent (k, r)
      int K = Kl + (Kl >= I);
      K += (K >= J);
      int R = Rl + (Rl >= lo);
      R += (R >= hi);
      const int k = K + (K >= fac), r = R + (R >= loc);
      const double v = src[ix.cell(i, j, p, q, k, r)];
      dst[e] = (v != 0) ? v : 0.0;
    }
  }
}

// store_evaluate (rlt2.cpp:91-107): the terms in the reference's summation
// order -- b[i,perm i] (i ascending), C'[i,perm i,j,perm j] (i, then j != i),
// D' cells (i<j lexicographic, then k != i,j ascending) -- gathered in
// parallel into `terms`; one thread then adds them in that order from offset.
__global__ void store_terms_kernel(int m, const double* __restrict__ b,
                                   const double* __restrict__ c, const double* __restrict__ d,
                                   const int* __restrict__ perm, double* __restrict__ terms) {
  const DIdx ix(m);
  const int nb = m, ncl = m * (m - 1);
  const int nd = m >= 3 ? m * (m - 1) / 2 * (m - 2) : 0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nb + ncl + nd;
       e += gridDim.x * blockDim.x) {
    double v;
    if (e < nb) {
      v = b[(size_t)e * m + perm[e]];
    } else if (e < nb + ncl) {
      const int x = e - nb, i = x / (m - 1), jj = x - i * (m - 1), j = jj + (jj >= i);
      v = c[ix.cidx(i, perm[i], j, perm[j])];
    } else {
      const int x = e - nb - ncl, pair = x / (m - 2), kk = x - pair * (m - 2);
      int i, j;
      unfpair(m, pair, &i, &j);  // pairs in fpair (lexicographic) order
      const int k = kk + (kk >= i) + (kk + (kk >= i) >= j);
      const int t = ix.tile(i, j, perm[i], perm[j]);
      v = d[(size_t)t * ix.esz + ix.cell(i, j, perm[i], perm[j], k, perm[k])];
    }
    terms[e] = v;
  }
}
__global__ void ordered_sum_kernel(const double* __restrict__ terms, int count, double offset,
                                   double* out) {
  double v = offset;
  for (int e = 0; e < count; ++e) v = dadd(v, terms[e]);
  *out = v;
}

// redistribute_family (rlt2.cpp:184-205) on the device: the same rule the
// phase-2 kernel applies per family, exposed for the reference API
__global__ void redistribute_kernel(const double* pi, double* add, int vslots, double tol,
                                    int* ok) {
  int nb = vslots;
  double total = 0.0;
  double a[3];
  for (int s = 0; s < 3; ++s) {
    if (pi[s] > tol)
      total = dadd(total, pi[s]);
    else
      ++nb;
  }
  const bool zero = total <= 0.0 || nb == 0;
  const double share = zero ? 0.0 : __ddiv_rn(total, (double)nb);
  for (int s = 0; s < 3; ++s) a[s] = zero ? 0.0 : ((pi[s] > tol) ? -pi[s] : share);
  for (int s = 0; s < 3; ++s) add[s] = a[s];
  *ok = (total <= 0.0 || nb != 0) ? 1 : 0;
}

int sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// the calling thread's current device, restored on scope exit
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

size_t store_nb(int m) { return (size_t)m * m; }
size_t store_nc(int m) { return (size_t)m * m * (m - 1) * (m - 1); }
size_t store_nd(int m) {
  return m >= 3 ? (size_t)m * (m - 1) / 2 * m * (m - 1) * (m - 2) * (m - 2) : 0;
}

// Each store owns a stream and takes its arrays from the device's
// stream-ordered pool: creating, folding and freeing the stores of several
// branch-and-bound banks never serialises the device (cudaMalloc/cudaFree and
// legacy-stream work would).
DeviceStore::DeviceStore(int m_, int device_) : m(m_), device(device_) {
  DeviceGuard g(device);
  check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
  check(cudaMallocAsync(&b, std::max<size_t>(1, store_nb(m)) * sizeof(double), stream), "alloc b");
  check(cudaMallocAsync(&c, std::max<size_t>(1, store_nc(m)) * sizeof(double), stream), "alloc c");
  check(cudaMallocAsync(&d, std::max<size_t>(1, store_nd(m)) * sizeof(double), stream), "alloc d");
  synchronize();  // usable from any stream from here on
}

DeviceStore::~DeviceStore() {
  DeviceGuard g(device);
  cudaFreeAsync(b, stream);
  cudaFreeAsync(c, stream);
  cudaFreeAsync(d, stream);
  cudaStreamSynchronize(stream);
  cudaStreamDestroy(stream);
}

void DeviceStore::synchronize() const { check(cudaStreamSynchronize(stream), "store stream"); }

std::unique_ptr<DeviceStore> collapse_store_device(const DeviceStore& s, int fac, int loc) {
  return collapse_store_device(s, fac, loc, s.offset);
}

std::unique_ptr<DeviceStore> collapse_store_device(const DeviceStore& s, int fac, int loc,
                                                   double offset) {
  const int m = s.m, mc = m - 1;
  if (mc < 2) throw std::invalid_argument("collapse_store: store too small");  // rlt2.cpp:111
  if (fac < 0 || fac >= m || loc < 0 || loc >= m)
    throw std::invalid_argument("collapse_store: facility/location out of range");
  DeviceGuard g(s.device);
  auto out = std::make_unique<DeviceStore>(mc, s.device);
  // the child's stream follows everything already queued on the parent's
  cudaEvent_t ev;
  check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  check(cudaEventRecord(ev, s.stream), "event");
  check(cudaStreamWaitEvent(out->stream, ev, 0), "wait");
  cudaEventDestroy(ev);
  double bfl = 0.0;
  check(cudaMemcpyAsync(&bfl, s.b + (size_t)fac * m + loc, sizeof(double),
                        cudaMemcpyDeviceToHost, out->stream),
        "D2H b");
  collapse_b_kernel<<<(mc * mc + 255) / 256, 256, 0, out->stream>>>(m, fac, loc, s.b, s.c, out->b);
  check(cudaGetLastError(), "collapse b");
  collapse_c_kernel<<<4 * sms(), 256, 0, out->stream>>>(m, fac, loc, s.c, s.d, out->c);
  check(cudaGetLastError(), "collapse c");
  if (mc >= 3) {
    collapse_d_kernel<<<8 * sms(), 256, 0, out->stream>>>(m, fac, loc, s.d, out->d);
    check(cudaGetLastError(), "collapse d");
  }
  out->synchronize();
  out->offset = offset + bfl;  // rlt2.cpp:116
  return out;
}

double store_evaluate_device(const DeviceStore& s, const int* perm, double offset) {
  const int m = s.m;
  if (m < 3) throw std::invalid_argument("store_evaluate: m >= 3 required");
  DeviceGuard g(s.device);
  const int count = m + m * (m - 1) + m * (m - 1) / 2 * (m - 2);
  int* dperm = nullptr;
  double *terms = nullptr, *dv = nullptr;
  check(cudaMallocAsync(reinterpret_cast<void**>(&dperm), m * sizeof(int), s.stream), "alloc");
  check(cudaMallocAsync(reinterpret_cast<void**>(&terms), count * sizeof(double), s.stream),
        "alloc");
  check(cudaMallocAsync(reinterpret_cast<void**>(&dv), sizeof(double), s.stream), "alloc");
  check(cudaMemcpyAsync(dperm, perm, m * sizeof(int), cudaMemcpyHostToDevice, s.stream), "H2D");
  store_terms_kernel<<<std::max(1, std::min(4 * sms(), (count + 255) / 256)), 256, 0, s.stream>>>(
      m, s.b, s.c, s.d, dperm, terms);
  check(cudaGetLastError(), "store terms");
  ordered_sum_kernel<<<1, 1, 0, s.stream>>>(terms, count, offset, dv);
  check(cudaGetLastError(), "ordered sum");
  double v = 0.0;
  check(cudaMemcpyAsync(&v, dv, sizeof(double), cudaMemcpyDeviceToHost, s.stream), "D2H");
  cudaFreeAsync(dperm, s.stream);
  cudaFreeAsync(terms, s.stream);
  cudaFreeAsync(dv, s.stream);
  s.synchronize();
  return v;
}

bool redistribute_family_device(const double pi[3], double add[3], int virtual_slots, double tol,
                                int device) {
  DeviceGuard g(device);
  cudaStream_t st = cudaStreamPerThread;
  double* buf = nullptr;
  check(cudaMallocAsync(reinterpret_cast<void**>(&buf), 7 * sizeof(double), st), "alloc");
  check(cudaMemcpyAsync(buf, pi, 3 * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
  redistribute_kernel<<<1, 1, 0, st>>>(buf, buf + 3, virtual_slots, tol,
                                       reinterpret_cast<int*>(buf + 6));
  check(cudaGetLastError(), "redistribute");
  double h[7];
  check(cudaMemcpyAsync(h, buf, sizeof h, cudaMemcpyDeviceToHost, st), "D2H");
  cudaFreeAsync(buf, st);
  check(cudaStreamSynchronize(st), "redistribute");
  for (int k = 0; k < 3; ++k) add[k] = h[3 + k];
  int ok = 0;
  std::memcpy(&ok, &h[6], sizeof ok);
  return ok != 0;
}

}  // namespace qapb

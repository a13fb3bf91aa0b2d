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

}  // namespace

size_t store_nb(int m) { return (size_t)m * m; }
size_t store_nc(int m) { return (size_t)m * m * (m - 1) * (m - 1); }
size_t store_nd(int m) {
  return m >= 3 ? (size_t)m * (m - 1) / 2 * m * (m - 1) * (m - 2) * (m - 2) : 0;
}

DeviceStore::DeviceStore(int m_, int device_) : m(m_), device(device_) {
  check(cudaSetDevice(device), "cudaSetDevice");
  check(cudaMalloc(&b, std::max<size_t>(1, store_nb(m)) * sizeof(double)), "cudaMalloc b");
  check(cudaMalloc(&c, std::max<size_t>(1, store_nc(m)) * sizeof(double)), "cudaMalloc c");
  check(cudaMalloc(&d, std::max<size_t>(1, store_nd(m)) * sizeof(double)), "cudaMalloc d");
}

DeviceStore::~DeviceStore() {
  cudaSetDevice(device);
  cudaFree(b);
  cudaFree(c);
  cudaFree(d);
}

std::unique_ptr<DeviceStore> collapse_store_device(const DeviceStore& s, int fac, int loc) {
  const int m = s.m, mc = m - 1;
  if (mc < 2) throw std::invalid_argument("collapse_store: store too small");  // rlt2.cpp:111
  if (fac < 0 || fac >= m || loc < 0 || loc >= m)
    throw std::invalid_argument("collapse_store: facility/location out of range");
  auto out = std::make_unique<DeviceStore>(mc, s.device);
  double bfl = 0.0;
  check(cudaMemcpy(&bfl, s.b + (size_t)fac * m + loc, sizeof(double), cudaMemcpyDeviceToHost),
        "D2H b");
  out->offset = s.offset + bfl;  // rlt2.cpp:116
  collapse_b_kernel<<<(mc * mc + 255) / 256, 256>>>(m, fac, loc, s.b, s.c, out->b);
  check(cudaGetLastError(), "collapse b");
  collapse_c_kernel<<<4 * sms(), 256>>>(m, fac, loc, s.c, s.d, out->c);
  check(cudaGetLastError(), "collapse c");
  if (mc >= 3) {
    collapse_d_kernel<<<8 * sms(), 256>>>(m, fac, loc, s.d, out->d);
    check(cudaGetLastError(), "collapse d");
  }
  check(cudaDeviceSynchronize(), "collapse_store");
  return out;
}

}  // namespace qapb

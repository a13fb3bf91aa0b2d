// common.cuh — device helpers shared by the RLT2 kernels (sm_100a).
//
// Arithmetic contract: every floating-point operation on the path is a
// separately rounded IEEE fp64 op in the reference's evaluation order
// (SURVEY.md Appendix A).  The explicit __d*_rn intrinsics are never fused
// into FMAs by nvcc; the library is additionally compiled with --fmad=false.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define QAPB_FULL 0xffffffffu

namespace qapb {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// StoreIndex (rlt2.hpp:25-69) on the device.  m = problem size.
struct DIdx {
  int m, lpairs, esz;
  __host__ __device__ DIdx() : m(0), lpairs(0), esz(0) {}
  __host__ __device__ explicit DIdx(int m_)
      : m(m_), lpairs(m_ * (m_ - 1)), esz((m_ - 2) * (m_ - 2)) {}
  __device__ __forceinline__ int fpair(int i, int j) const {  // rlt2.hpp:37-39
    return i * m - i * (i + 1) / 2 + (j - i - 1);
  }
  __device__ __forceinline__ int lpair(int p, int q) const {  // rlt2.hpp:40-42
    return p * (m - 1) + q - (q > p);
  }
  __device__ __forceinline__ int tile(int i, int j, int p, int q) const {  // :43-45
    return fpair(i, j) * lpairs + lpair(p, q);
  }
  __device__ __forceinline__ int cell(int i, int j, int p, int q, int k, int r) const {
    const int kl = k - (k > i) - (k > j);  // rlt2.hpp:47-52
    const int lo = p < q ? p : q, hi = p < q ? q : p;
    const int rl = r - (r > lo) - (r > hi);
    return kl * (m - 2) + rl;
  }
  __device__ __forceinline__ size_t cidx(int i, int p, int j, int q) const {  // :65-68
    return ((size_t)i * m + p) * (m - 1) * (m - 1) + (size_t)(j - (j > i)) * (m - 1) +
           (q - (q > p));
  }
  // lpair id -> (p, q), inverse of lpair()
  __device__ __forceinline__ void unlpair(int lp, int* p, int* q) const {
    const int pp = lp / (m - 1), qq = lp - pp * (m - 1);
    *p = pp;
    *q = qq + (qq >= pp);
  }
};

// x / d for 0 <= x < 2^22 and 0 < d < 2^12 through a float reciprocal and one
// correction step (the compiler's 32-bit division by a runtime divisor is ~20
// instructions)
__device__ __forceinline__ int small_udiv(int x, int d) {
  int q = __float2int_rz(__fmul_rz((float)x, __frcp_rn((float)d)));
  const int r = x - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// r-th free index of {0..n-1} \ {lo, hi} (lo < hi): uncell's column rule.
__device__ __forceinline__ int skip2(int r, int lo, int hi) {
  if (r >= lo) ++r;
  if (r >= hi) ++r;
  return r;
}

// Debug builds (make EXTRA=-DQAPB_BOUNDS): index checks that print and trap.
#ifdef QAPB_BOUNDS
#define QAPB_CHECK(cond, tag, v, lim)                                                        \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("QAPB_BOUNDS %s: %llu >= %llu (block %d thread %d)\n", tag,                     \
             (unsigned long long)(v), (unsigned long long)(lim), (int)blockIdx.x,           \
             (int)threadIdx.x);                                                             \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define QAPB_CHECK(cond, tag, v, lim) \
  do {                                \
  } while (0)
#endif

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- async copy / mbarrier primitives (TMA bulk path) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// expect `bytes` more transaction bytes in the current phase (no arrival)
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// One TMA bulk copy global -> shared, completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 eviction-priority policies and their cache-hinted loads / stores
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// TMA bulk copy shared -> global (bulk-group completion), its commit and the
// wait that makes the source shared memory reusable.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// every committed bulk store of this thread has completed (writes performed)
__device__ __forceinline__ void bulk_wait_all0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// 3-D TMA tensor copies through a CUtensorMap in global memory (64-byte
// aligned), coordinates innermost first.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const void* tmap, int c0, int c1,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* tmap, int c0, int c1, int c2,
                                             const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          tmap),
      "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
      : "memory");
}
// TMA bulk prefetch of [src, src+bytes) into L2 (no completion tracking).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// 16-byte LDGSTS, L2 only (.cg): rows that are 16-byte aligned.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
// 8-byte LDGSTS (cp.async): global -> shared without a register round trip,
// so a thread can keep dozens of loads in flight.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "QAPB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra QAPB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace qapb

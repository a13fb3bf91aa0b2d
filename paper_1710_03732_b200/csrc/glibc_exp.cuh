// Bit-exact restatement of the double exp that the reference's SA step calls
// (std::exp, rlt2.cpp:494): glibc >= 2.28, sysdeps/ieee754/dbl-64/e_exp.c (the
// ARM optimized-routines algorithm; this image ships GLIBC 2.39).
//
//   x = k ln2/128 + r,  |r| <= ln2/256
//   exp(x) = 2^(k/128) (1 + tmp),  tmp = tail + r + C2 r^2 + ... + C5 r^5
//
// glibc picks one of several builds of that file at load time (an IFUNC on
// x86-64): with FMA+AVX2 the compiler contracted the polynomial into fused
// multiply-adds; without it (SSE2/AVX builds) every product is rounded.  The
// results differ in the last bit for some arguments, so both are restated here
// op for op, and the host decides which one its libm uses (exp_variant_host()).
// The operation order below follows the x86-64 objects of GLIBC 2.39
// (__exp_fma and __exp_sse2); tests/test_exp_glibc.py pins both variants
// bitwise against the host libm and tests/test_gpu_exp.py pins the device
// against the host on 1e8 arguments.
#pragma once
#include <cstdint>
#include <cstring>

#include "exp_table.h"

#if defined(__CUDACC__)
#define QAPB_EXP_HD __host__ __device__ __forceinline__
#else
#define QAPB_EXP_HD inline
#endif

namespace qapb_exp {

// constants of e_exp_data.c (N = 128, EXP_POLY_ORDER = 5)
constexpr double kInvLn2N = 0x1.71547652b82fep7;     // 128 / ln2
constexpr double kShift = 0x1.8p52;                   // round-to-int shift
constexpr double kNegLn2hiN = -0x1.62e42fefa0000p-8;  // -ln2/128, 36 bits
constexpr double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
constexpr double kC2 = 0x1.ffffffffffdbdp-2;  // minimax on |r| <= ln2/256
constexpr double kC3 = 0x1.555555555543cp-3;
constexpr double kC4 = 0x1.55555cf172b91p-5;
constexpr double kC5 = 0x1.1111167a4d017p-7;

QAPB_EXP_HD uint64_t as_u64(double x) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}
QAPB_EXP_HD double as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

// separately rounded primitives (the device TU is built with --fmad=false,
// the host one without -mfma, but the intrinsics make it explicit)
QAPB_EXP_HD double add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
QAPB_EXP_HD double sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
QAPB_EXP_HD double mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
QAPB_EXP_HD double fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}

// 2^(k/128) scaling for results near the overflow / subnormal range
// (e_exp.c specialcase)
template <bool FMA>
QAPB_EXP_HD double special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {  // k > 0: scale may overflow by <= 460
    const double scale = as_f64(sbits - (1009ULL << 52));
    const double y = FMA ? fma(scale, tmp, scale) : add(scale, mul(scale, tmp));
    return mul(0x1p1009, y);
  }
  const double scale = as_f64(sbits + (1022ULL << 52));  // k < 0: subnormal care
  const double st = mul(scale, tmp);  // not contracted in either build
  double y = add(scale, st);
  if (y < 1.0) {
    const double hi = add(y, 1.0);
    double lo = add(sub(scale, y), st);
    lo = add(add(sub(1.0, hi), y), lo);
    y = sub(add(lo, hi), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return mul(0x1p-1022, y);
}

// `tab` = the 256-entry table of exp_table.h (device: global, host: static)
template <bool FMA>
QAPB_EXP_HD double exp(double x, const uint64_t* tab) {
  const uint64_t ux = as_u64(x);
  uint32_t abstop = static_cast<uint32_t>(ux >> 52) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {  // |x| < 2^-54 or |x| >= 512 or not finite
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return add(1.0, x);
    if (abstop >= 0x409u) {
      if (ux == 0xfff0000000000000ULL) return 0.0;
      if (abstop >= 0x7ffu) return add(1.0, x);
      return (ux >> 63) ? 0.0 : as_f64(0x7ff0000000000000ULL);  // __math_uflow/oflow
    }
    abstop = 0;  // large |x|: may over/underflow, scale in special()
  }
  double kd = FMA ? fma(x, kInvLn2N, kShift) : add(mul(kInvLn2N, x), kShift);
  const uint64_t ki = as_u64(kd);
  kd = sub(kd, kShift);
  const double r = FMA ? fma(kd, kNegLn2loN, fma(kd, kNegLn2hiN, x))
                       : add(add(x, mul(kd, kNegLn2hiN)), mul(kd, kNegLn2loN));
  const uint32_t idx = 2u * static_cast<uint32_t>(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = as_f64(tab[idx]);
  const uint64_t sbits = tab[idx + 1] + top;
  const double r2 = mul(r, r);
  double tmp;
  if (FMA) {
    tmp = fma(mul(r2, r2), fma(r, kC5, kC4), fma(fma(r, kC3, kC2), r2, add(tail, r)));
  } else {
    tmp = add(add(add(tail, r), mul(r2, add(kC2, mul(r, kC3)))),
              mul(mul(r2, r2), add(kC4, mul(r, kC5))));
  }
  if (abstop == 0) return special<FMA>(tmp, sbits, ki);
  const double scale = as_f64(sbits);
  return FMA ? fma(scale, tmp, scale) : add(scale, mul(scale, tmp));
}

}  // namespace qapb_exp

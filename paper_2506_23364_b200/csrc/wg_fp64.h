// Strict IEEE-754 binary64 primitives shared by device kernels and host-side
// checks.  Every operation the reference performs through numpy ufuncs is a
// separately rounded + - * / sqrt (no fused multiply-add), so parity code
// spells each one out: on the device through the _rn intrinsics (which nvcc
// never contracts, independent of -fmad), on the host as plain C operators
// compiled with -ffp-contract=off.  WG_FMA is used ONLY where the third-party
// code being mirrored itself fuses (glibc's __sin_fma/__cos_fma).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define WG_HD __host__ __device__ __forceinline__
#else
#define WG_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define WG_ADD(a, b) __dadd_rn((a), (b))
#define WG_SUB(a, b) __dsub_rn((a), (b))
#define WG_MUL(a, b) __dmul_rn((a), (b))
#define WG_DIV(a, b) __ddiv_rn((a), (b))
#define WG_SQRT(a) __dsqrt_rn((a))
#define WG_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#include <math.h>
#include <string.h>
#define WG_ADD(a, b) ((a) + (b))
#define WG_SUB(a, b) ((a) - (b))
#define WG_MUL(a, b) ((a) * (b))
#define WG_DIV(a, b) ((a) / (b))
#define WG_SQRT(a) sqrt((a))
#define WG_FMA(a, b, c) fma((a), (b), (c))
#endif

WG_HD uint64_t wg_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}

WG_HD double wg_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}

WG_HD double wg_fabs(double x) { return wg_from_bits(wg_bits(x) & 0x7fffffffffffffffULL); }

WG_HD double wg_copysign(double mag, double sgn) {
  return wg_from_bits((wg_bits(mag) & 0x7fffffffffffffffULL) | (wg_bits(sgn) & 0x8000000000000000ULL));
}

// IEEE negation is an exact sign flip (also for zeros); on the device it folds
// into the consuming instruction as an operand modifier.
WG_HD double wg_neg(double x) { return -x; }

// numpy.minimum / numpy.maximum on non-NaN operands (the operands on the
// parity paths are never NaN).  Ties return the first operand like numpy.
WG_HD double wg_min(double a, double b) { return (b < a) ? b : a; }
WG_HD double wg_max(double a, double b) { return (b > a) ? b : a; }

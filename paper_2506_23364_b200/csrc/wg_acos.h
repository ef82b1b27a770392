// Bit-exact restatement of the float64 arccos numpy 2.3.5 computes on AVX-512
// hosts: Intel SVML's __svml_acos8_ha, which numpy dispatches np.arccos to
// there (the reference's steepness node, terrain.py:99-102, and through it
// the release mask, simulate.py:207-225, and the snow alpha,
// simulate.py:520-537).  Matching it bit for bit makes the slope field, and
// so every threshold decision on it, identical to the reference's.
//
// The SVML routine is straight-line code (one lane shown): every operation
// below is one instruction of __svml_acos8_ha in numpy's
// _multiarray_umath.so, in program order -- WG_FMA for each vfmadd/vfmsub
// (all {rn-sae}), WG_MUL/WG_ADD/WG_SUB for vmulpd/vaddpd/vsubpd, selects for
// the mask-register blends.  Its one non-IEEE step, VRSQRT14PD, is a table
// (svml_acos_tables.inc, generated with the constants by
// tools/gen_svml_acos.py from the CPU instruction and numpy's data block).
// Inputs with |x| > 1 or NaN take SVML's scalar "rare" path, which this
// restatement does not model: the callers clip to [-1, 1] first
// (terrain.py:101), so they never reach it.
#pragma once

#include "wg_fp64.h"

#if defined(__CUDA_ARCH__) || defined(__CUDACC__)
#define WG_ACOS_TABLE static __device__ const __align__(16)
#else
#define WG_ACOS_TABLE static const
#endif
#include "svml_acos_tables.inc"
#undef WG_ACOS_TABLE

// VRSQRT14PD of a positive normal s: the result depends on the exponent
// parity and the top 15 mantissa bits only, and scales exactly by powers of
// 4 -- except that exact powers of 4 get their exact root.
WG_HD double wg_rsqrt14(double s) {
  const uint64_t u = wg_bits(s);
  const int e = (int)(u >> 52) - 1023;
  if ((u & 0x000fffffffffffffULL) == 0 && (e & 1) == 0) return wg_from_bits((uint64_t)(1023 - e / 2) << 52);
  const uint32_t par = (uint32_t)e & 1u;
  const uint32_t idx = (par << 15) | (uint32_t)((u >> 37) & 0x7fffu);
  const uint32_t g = idx >> 3, k = idx & 7u;
  // record g: (value of entry 0, nibble word of backward differences)
#if defined(__CUDA_ARCH__)
  const uint2 rec = __ldg(reinterpret_cast<const uint2*>(wg_rsq14_tab) + g);
  const uint32_t base = rec.x, word = rec.y;
#else
  const uint32_t base = wg_rsq14_tab[2 * g], word = wg_rsq14_tab[2 * g + 1];
#endif
  // sum of nibbles 1..k (nibble 0 is zero): mask, then a SWAR byte sum
  const uint32_t x = word & (k == 7u ? 0xffffffffu : ((1u << (4 * (k + 1))) - 1u));
  const uint32_t b = (x & 0x0f0f0f0fu) + ((x >> 4) & 0x0f0f0f0fu);
  const uint32_t tot = (b * 0x01010101u) >> 24;
  const int q = par ? -16 - (e + 1) / 2 : -17 - e / 2;
  return (double)(int)(base - tot) * wg_from_bits((uint64_t)(q + 1023) << 52);
}

// np.arccos(x) for x in [-1, 1], bit for bit (AVX-512 numpy).
WG_HD double wg_acos(double x) {
  const uint64_t sgn = wg_bits(x) & 0x8000000000000000ULL;
  const double na = wg_from_bits(wg_bits(x) | 0x8000000000000000ULL);  // -|x|
  const double s = WG_FMA(0.5, na, 0.5);                                // (1 - |x|) / 2
  const double x2 = WG_MUL(na, na);
  double y = wg_rsqrt14(s);
  if (s < wg_from_bits(0x3000000000000000ULL)) y = 0.0;
  const double t = x2 < s ? x2 : s;  // vminpd: second operand on ties
  const double s2 = WG_ADD(s, s);
  const int k1 = !(t < s);  // |x| >= 1/2 branch: acos = 2 asin(sqrt(s))
  const int k3 = !(t < x);  // ... with x negative: pi - that
  const double h = WG_MUL(s2, y);
  const double e = WG_FMA(WG_MUL(y, y), s2, -2.0);
  const double lo = WG_FMA(y, s2, -h);
  double p = WG_FMA(wg_from_bits(WG_ACOS_E3), e, wg_from_bits(WG_ACOS_E2));
  const double he = WG_MUL(h, e);
  p = WG_FMA(e, p, wg_from_bits(WG_ACOS_E1));
  p = WG_FMA(e, p, wg_from_bits(WG_ACOS_E0));
  const double q0 = WG_FMA(wg_from_bits(WG_ACOS_P10), t, wg_from_bits(WG_ACOS_P9));
  const double corr = WG_FMA(he, p, -lo);
  double q1 = WG_FMA(wg_from_bits(WG_ACOS_P12), t, wg_from_bits(WG_ACOS_P11));
  const double q10 = WG_FMA(wg_from_bits(WG_ACOS_P4), t, wg_from_bits(WG_ACOS_P3));
  const double t2 = WG_MUL(t, t);
  double q8 = WG_FMA(wg_from_bits(WG_ACOS_P8), t, wg_from_bits(WG_ACOS_P7));
  q1 = WG_FMA(t2, q1, q0);
  const double t4 = WG_MUL(t2, t2);
  const double q11 = WG_FMA(wg_from_bits(WG_ACOS_P6), t, wg_from_bits(WG_ACOS_P5));
  q8 = WG_FMA(t2, q8, q11);
  q1 = WG_FMA(t4, q1, q8);
  q1 = WG_FMA(t2, q1, q10);
  const double c2 = k1 ? corr : 0.0;
  q1 = WG_FMA(t, q1, wg_from_bits(WG_ACOS_P2));
  q1 = WG_FMA(t, q1, wg_from_bits(WG_ACOS_P1));
  const double pt = WG_MUL(t, q1);
  double a_lo = k1 ? 0.0 : wg_from_bits(WG_ACOS_HPI_LO);
  double a_hi = k1 ? 0.0 : wg_from_bits(WG_ACOS_HPI_HI);
  if (k1 && k3) {
    a_lo = wg_from_bits(WG_ACOS_PI_LO);
    a_hi = wg_from_bits(WG_ACOS_PI_HI);
  }
  const double z9 = wg_from_bits(wg_bits(a_lo) ^ sgn);
  const double z4 = k1 ? h : na;
  const double z6 = WG_SUB(z9, c2);
  const double z3 = WG_SUB(z4, c2);
  double r = WG_ADD(WG_FMA(z3, pt, z6), z4);
  r = wg_from_bits(wg_bits(r) ^ sgn);
  return WG_ADD(r, a_hi);
}

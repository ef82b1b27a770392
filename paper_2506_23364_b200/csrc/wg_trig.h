// Bit-exact port of glibc 2.39's x86-64 __sin_fma / __cos_fma for |x| < 2.426265
// (sysdeps/ieee754/dbl-64/s_sin.c built with -mfma -mavx2, the ifunc variant
// numpy's np.sin/np.cos reach on FMA hosts).  The reference jitters every
// particle step through them (simulate.py:358-361), so the trajectory kernel
// must reproduce their exact bits, not merely be accurate.
//
// Ported from the instruction stream of libm.so.6 (glibc 2.39-0ubuntu8.5):
//   __sin_fma @ 0x7b2d0, __cos_fma @ 0x7bad0.  Each fused operation below
//   corresponds to one vfmadd/vfnmadd/vfmsub in that stream (GCC contracted
//   the C source with -ffp-contract=fast); every other operation is a
//   separately rounded vaddsd/vsubsd/vmulsd.
// The jitter angle is theta = (2u-1) * randomness * pi/2 with randomness in
// [0, 1] (simulate.py:91-94, 358), so |theta| <= pi/2 < 2.426265 and the
// large-argument range reduction (reduce_sincos/__branred) is never reached.
// Outside that domain these functions return NaN (never hit on the path).
#pragma once

#include "wg_fp64.h"

#if defined(__CUDA_ARCH__)
// table lives in shared memory inside the kernels that use it (see traj.cu);
// this header takes the table pointer as an argument.
#endif

// polynomial / split constants, IEEE bit patterns from libm .rodata
#define WG_SC_BIG 52776558133248.0                         /* 0x42c8000000000000: 1.5 * 2^45 */
#define WG_SC_TINY 0.126                                   /* 0x3fc020c49ba5e354 */
#define WG_SC_HP0 1.5707963267948966                       /* 0x3ff921fb54442d18 */
#define WG_SC_HP1 6.123233995736766e-17                    /* 0x3c91a62633145c07 */
#define WG_SC_SN3 (-0.16666666666666488)                   /* 0xbfc5555555555515 */
#define WG_SC_SN5 0.008333332142857223                     /* 0x3f811110e829872f */
#define WG_SC_CS2 0.5                                      /* 0x3fe0000000000000 */
#define WG_SC_CS4 (-0.04166666666666644)                   /* 0xbfa5555555555535 */
#define WG_SC_CS6 0.001388888740079376                     /* 0x3f56c16bedd9e239 */
#define WG_SC_S1 (-0.16666666666666666)                    /* 0xbfc5555555555555 */
#define WG_SC_S2 0.008333333333332329                      /* 0x3f81111111110ece */
#define WG_SC_S3 (-0.00019841269834414642)                 /* 0xbf2a01a019db08b8 */
#define WG_SC_S4 2.755729806860771e-06                     /* 0x3ec71de27b9a7ed9 */
#define WG_SC_S5 (-2.5022014848318398e-08)                 /* 0xbe5addffc2fcdf59 */

// do_sin(x, dx) of s_sin.c; tab = __sincostab as doubles (4 per entry).
WG_HD double wg_do_sin(const double* tab, double x, double dx) {
  double ax = wg_fabs(x);
  if (ax < WG_SC_TINY) {
    // TAYLOR_SIN(x*x, x, dx)
    double xx = WG_MUL(x, x);
    double p = WG_FMA(xx, WG_SC_S5, WG_SC_S4);
    p = WG_FMA(xx, p, WG_SC_S3);
    p = WG_FMA(xx, p, WG_SC_S2);
    p = WG_FMA(xx, p, WG_SC_S1);
    double t = WG_FMA(p, x, wg_neg(WG_MUL(dx, 0.5)));
    t = WG_FMA(xx, t, dx);
    return WG_ADD(x, t);
  }
  if (x <= 0.0) dx = wg_neg(dx);
  double u = WG_ADD(WG_SC_BIG, ax);
  int k = (int)((uint32_t)wg_bits(u) << 2);
  double xr = WG_SUB(ax, WG_SUB(u, WG_SC_BIG));
  double xx = WG_MUL(xr, xr);
  double ps = WG_FMA(xx, WG_SC_SN5, WG_SC_SN3);
  double s = WG_ADD(xr, WG_FMA(WG_MUL(xr, xx), ps, dx));
  double pc = WG_FMA(xx, WG_SC_CS6, WG_SC_CS4);
  pc = WG_FMA(xx, pc, WG_SC_CS2);
  double c = WG_FMA(xr, dx, WG_MUL(xx, pc));
  double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  double cor = WG_FMA(s, ccs, ssn);
  cor = WG_FMA(wg_neg(c), sn, cor);
  cor = WG_FMA(s, cs, cor);
  return wg_copysign(WG_ADD(sn, cor), x);
}

// do_cos(x, dx) of s_sin.c.
WG_HD double wg_do_cos(const double* tab, double x, double dx) {
  if (x < 0.0) dx = wg_neg(dx);
  double ax = wg_fabs(x);
  double u = WG_ADD(WG_SC_BIG, ax);
  int k = (int)((uint32_t)wg_bits(u) << 2);
  double xr = WG_ADD(WG_SUB(ax, WG_SUB(u, WG_SC_BIG)), dx);
  double xx = WG_MUL(xr, xr);
  double ps = WG_FMA(xx, WG_SC_SN5, WG_SC_SN3);
  double s = WG_FMA(WG_MUL(xr, xx), ps, xr);
  double pc = WG_FMA(xx, WG_SC_CS6, WG_SC_CS4);
  pc = WG_FMA(xx, pc, WG_SC_CS2);
  double c = WG_MUL(xx, pc);
  double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  double cor = WG_FMA(wg_neg(s), ssn, ccs);
  cor = WG_FMA(wg_neg(c), cs, cor);
  cor = WG_FMA(wg_neg(s), sn, cor);
  return WG_ADD(cs, cor);
}

// __sin (s_sin.c) restricted to |x| < 2.426265.
WG_HD double wg_glibc_sin(const double* tab, double x) {
  uint32_t k = (uint32_t)(wg_bits(x) >> 32) & 0x7fffffffu;
  if (k <= 0x3e4fffffu) return x;
  if (k <= 0x3feb5fffu) return wg_do_sin(tab, x, 0.0);
  if (k <= 0x400368fcu) {
    double t = WG_SUB(WG_SC_HP0, wg_fabs(x));
    return wg_copysign(wg_do_cos(tab, t, WG_SC_HP1), x);
  }
  return wg_from_bits(0x7ff8000000000000ULL);
}

// __cos (s_sin.c) restricted to |x| < 2.426265.
WG_HD double wg_glibc_cos(const double* tab, double x) {
  uint32_t k = (uint32_t)(wg_bits(x) >> 32) & 0x7fffffffu;
  if (k <= 0x3e3fffffu) return 1.0;
  if (k <= 0x3feb5fffu) return wg_do_cos(tab, x, 0.0);
  if (k <= 0x400368fcu) {
    double y = WG_SUB(WG_SC_HP0, wg_fabs(x));
    double a = WG_ADD(y, WG_SC_HP1);
    double da = WG_ADD(WG_SUB(y, a), WG_SC_HP1);
    return wg_do_sin(tab, a, da);
  }
  return wg_from_bits(0x7ff8000000000000ULL);
}

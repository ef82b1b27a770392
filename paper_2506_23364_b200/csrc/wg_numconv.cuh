// Decimal <-> binary64 conversion with Python's semantics, for the device
// ESRI ASCII grid reader/writer (asciigrid.cu; reference:
// /root/reference/pkg/src/demflow/asciigrid.py).
//
//   nc_parse(s, n, &v)  == float(token) of CPython (the reference parses with
//                          np.array(tokens, dtype=float64), which calls it):
//                          [+-] digits/'.'/exponent with PEP 515 underscores,
//                          inf / infinity / nan (any case); correctly rounded
//                          (round half to even), overflow -> inf.
//   nc_format(v, buf)   == asciigrid.format_number(v): str(int(v)) for integral
//                          |v| < 1e16, else repr(v) -- the shortest digit
//                          string that round-trips (Ryu), laid out like
//                          CPython's float_repr ('r': exponent iff decpt <= -4
//                          or decpt > 16).
//
// Parsing: the Eisel-Lemire algorithm on up to 19 significant digits, whose
// 128-bit product is always sufficient (Mushtak & Lemire 2023); with more
// digits the truncated significand w and w + 1 are both converted and, when
// they disagree, an exact big-decimal conversion decides (the classic
// "decimal shift" algorithm, 800 digits + sticky bit).  Formatting: Ryu
// (Adams 2018).  Tables: pow5_tables.inc (tools/gen_pow5_tables.py).
//
// Host+device: tools/numconv_check.cu compiles the same code for the CPU and
// checks it against CPython on millions of inputs.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define NC_HD __host__ __device__ inline
#else
#define NC_HD inline
#endif

namespace nc {

NC_HD void mul128(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

NC_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

NC_HD double bits_to_double(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  __builtin_memcpy(&d, &b, 8);
  return d;
#endif
}

NC_HD uint64_t double_to_bits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t b;
  __builtin_memcpy(&b, &d, 8);
  return b;
#endif
}

// ---- parsing -------------------------------------------------------------

// Eisel-Lemire: w * 10^q (w != 0, normalised inside) -> IEEE bits without
// sign.  fast_float's compute_float<binary64> restated.
NC_HD uint64_t el_convert(int64_t q, uint64_t w, const uint64_t (*tab)[2]) {
  if (w == 0 || q < -342) return 0;
  if (q > 308) return 0x7FF0000000000000ULL;
  const int lz = clz64(w);
  w <<= lz;
  const int idx = (int)(q + 342);
  uint64_t lo, hi;
  mul128(w, tab[idx][1], lo, hi);
  const uint64_t precision_mask = 0xFFFFFFFFFFFFFFFFULL >> 55;
  if ((hi & precision_mask) == precision_mask) {  // the product's low bits matter: add the next 64
    uint64_t lo2, hi2;
    mul128(w, tab[idx][0], lo2, hi2);
    lo += hi2;
    if (hi2 > lo) hi++;
  }
  const int upperbit = (int)(hi >> 63);
  const int shift = upperbit + 64 - 52 - 3;
  uint64_t mantissa = hi >> shift;
  int32_t power2 = (int32_t)((((152170 + 65536) * (int32_t)q) >> 16) + 63) + upperbit - lz + 1023;
  if (power2 <= 0) {  // subnormal
    if (-power2 + 1 >= 64) return 0;
    mantissa >>= -power2 + 1;
    mantissa += (mantissa & 1);
    mantissa >>= 1;
    power2 = (mantissa < (1ULL << 52)) ? 0 : 1;
    return (mantissa & ((1ULL << 52) - 1)) | ((uint64_t)power2 << 52);
  }
  if (lo <= 1 && q >= -4 && q <= 23 && (mantissa & 3) == 1) {
    // exactly halfway between two doubles: round to even
    if ((mantissa << shift) == hi) mantissa &= ~1ULL;
  }
  mantissa += (mantissa & 1);
  mantissa >>= 1;
  if (mantissa >= (2ULL << 52)) {
    mantissa = 1ULL << 52;
    power2++;
  }
  mantissa &= ~(1ULL << 52);
  if (power2 >= 0x7FF) return 0x7FF0000000000000ULL;
  return mantissa | ((uint64_t)power2 << 52);
}

// Exact big-decimal conversion (the "decimal shift" algorithm): digits d[0..nd)
// with the decimal point after dp digits, trunc = nonzero digits were dropped.
struct BigDec {
  static constexpr int kMax = 800;
  unsigned char d[kMax];
  int nd, dp;
  bool trunc;
};

NC_HD void bd_trim(BigDec& a) {
  while (a.nd > 0 && a.d[a.nd - 1] == 0) a.nd--;
  if (a.nd == 0) a.dp = 0;
}

NC_HD void bd_rshift(BigDec& a, unsigned k) {  // a /= 2^k, k <= 60
  int r = 0, w = 0;
  uint64_t n = 0;
  for (; (n >> k) == 0; r++) {
    if (r >= a.nd) {
      if (n == 0) {
        a.nd = 0;
        return;
      }
      while ((n >> k) == 0) {
        n *= 10;
        r++;
      }
      break;
    }
    n = n * 10 + a.d[r];
  }
  a.dp -= r - 1;
  const uint64_t mask = (1ULL << k) - 1;
  for (; r < a.nd; r++) {
    const uint64_t c = a.d[r];
    const uint64_t dig = n >> k;
    n &= mask;
    a.d[w++] = (unsigned char)dig;
    n = n * 10 + c;
  }
  while (n > 0) {
    const uint64_t dig = n >> k;
    n &= mask;
    if (w < BigDec::kMax) {
      a.d[w++] = (unsigned char)dig;
    } else if (dig > 0) {
      a.trunc = true;
    }
    n *= 10;
  }
  a.nd = w;
  bd_trim(a);
}

NC_HD void bd_lshift(BigDec& a, unsigned k) {  // a *= 2^k, k <= 60
  // multiply from the right into a right-aligned temporary; the integer
  // part grows by the carry digits (at most 19 for k <= 60)
  int extra = 0;
  unsigned char tmp[BigDec::kMax + 20];
  int w = BigDec::kMax + 20;
  uint64_t n = 0;
  for (int r = a.nd - 1; r >= 0; r--) {
    n += (uint64_t)a.d[r] << k;
    const uint64_t quo = n / 10, rem = n - 10 * quo;
    tmp[--w] = (unsigned char)rem;
    n = quo;
  }
  while (n > 0) {
    const uint64_t quo = n / 10, rem = n - 10 * quo;
    tmp[--w] = (unsigned char)rem;
    n = quo;
    extra++;
  }
  int len = BigDec::kMax + 20 - w;
  a.dp += extra;
  if (len > BigDec::kMax) {
    for (int i = BigDec::kMax; i < len; i++)
      if (tmp[w + i] != 0) a.trunc = true;
    len = BigDec::kMax;
  }
  for (int i = 0; i < len; i++) a.d[i] = tmp[w + i];
  a.nd = len;
  bd_trim(a);
}

NC_HD bool bd_round_up(const BigDec& a, int nd) {
  if (nd < 0 || nd >= a.nd) return false;
  if (a.d[nd] == 5 && nd + 1 == a.nd) {  // exactly halfway: round to even
    if (a.trunc) return true;
    return nd > 0 && (a.d[nd - 1] % 2) == 1;
  }
  return a.d[nd] >= 5;
}

NC_HD uint64_t bd_rounded_integer(const BigDec& a) {
  if (a.dp > 20) return 0xFFFFFFFFFFFFFFFFULL;
  int i = 0;
  uint64_t n = 0;
  for (; i < a.dp && i < a.nd; i++) n = n * 10 + a.d[i];
  for (; i < a.dp; i++) n *= 10;
  if (bd_round_up(a, a.dp)) n++;
  return n;
}

// IEEE bits (no sign) of the decimal, correctly rounded (Go's floatBits).
NC_HD uint64_t bd_to_bits(BigDec& a) {
  const int powtab[9] = {1, 3, 6, 9, 13, 16, 19, 23, 26};
  const int bias = -1023;
  int exp = 0;
  uint64_t mant = 0;
  if (a.nd == 0) return 0;
  if (a.dp > 310) return 0x7FF0000000000000ULL;
  if (a.dp < -330) return 0;
  while (a.dp > 0) {
    const int n = a.dp >= 9 ? 27 : powtab[a.dp];
    bd_rshift(a, (unsigned)n);
    exp += n;
  }
  while (a.dp < 0 || (a.dp == 0 && a.d[0] < 5)) {
    const int n = -a.dp >= 9 ? 27 : powtab[-a.dp];
    bd_lshift(a, (unsigned)n);
    exp -= n;
  }
  exp--;  // [0.5, 1) -> [1, 2)
  if (exp < bias + 1) {
    const int n = bias + 1 - exp;
    bd_rshift(a, (unsigned)(n > 60 ? 60 : n));
    // (n > 60 only for results that round to zero; shift the rest)
    for (int rest = n - 60; rest > 0; rest -= 60) bd_rshift(a, (unsigned)(rest > 60 ? 60 : rest));
    exp += n;
  }
  if (exp - bias >= 0x7FF) return 0x7FF0000000000000ULL;
  bd_lshift(a, 53);
  mant = bd_rounded_integer(a);
  if (mant == (2ULL << 52)) {
    mant >>= 1;
    exp++;
    if (exp - bias >= 0x7FF) return 0x7FF0000000000000ULL;
  }
  if ((mant & (1ULL << 52)) == 0) exp = bias;
  return (mant & ((1ULL << 52) - 1)) | ((uint64_t)((exp - bias) & 0x7FF) << 52);
}

NC_HD bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

NC_HD unsigned char lower(unsigned char c) { return (c >= 'A' && c <= 'Z') ? (unsigned char)(c + 32) : c; }

// Returns 0 and sets *out, or -1 for a token CPython's float() rejects.
NC_HD int nc_parse(const unsigned char* s, int n, double* out, const uint64_t (*tab)[2]) {
  int i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) {
    neg = s[i] == '-';
    i++;
  }
  if (i >= n) return -1;
  const uint64_t sign = neg ? 0x8000000000000000ULL : 0;
  {
    const unsigned char c0 = lower(s[i]);
    if (c0 == 'i' || c0 == 'n') {
      const int r = n - i;
      const char* words[3] = {"inf", "infinity", "nan"};
      const int lens[3] = {3, 8, 3};
      for (int k = 0; k < 3; k++) {
        if (r != lens[k]) continue;
        bool eq = true;
        for (int j = 0; j < r; j++) eq = eq && lower(s[i + j]) == (unsigned char)words[k][j];
        if (eq) {
          *out = bits_to_double(sign | (k < 2 ? 0x7FF0000000000000ULL : 0x7FF8000000000000ULL));
          return 0;
        }
      }
      return -1;
    }
  }
  const int body = i;
  uint64_t w = 0;
  int kept = 0;          // significant digits in w
  int64_t exp10 = 0;     // value = w * 10^(exp10 + e)
  bool many = false;     // nonzero digits beyond the 19 kept
  bool any = false;
  // integer part
  bool prev_digit = false;
  for (; i < n; i++) {
    const unsigned char c = s[i];
    if (is_digit(c)) {
      any = true;
      prev_digit = true;
      if (kept < 19) {
        if (w != 0 || c != '0') {
          w = w * 10 + (c - '0');
          kept++;
        }
      } else {
        exp10++;
        many = many || c != '0';
      }
    } else if (c == '_') {
      if (!prev_digit || i + 1 >= n || !is_digit(s[i + 1])) return -1;
      prev_digit = false;
    } else {
      break;
    }
  }
  if (i < n && s[i] == '.') {
    i++;
    prev_digit = false;
    for (; i < n; i++) {
      const unsigned char c = s[i];
      if (is_digit(c)) {
        any = true;
        prev_digit = true;
        if (kept < 19) {
          if (w != 0 || c != '0') {
            w = w * 10 + (c - '0');
            kept++;
          }
          exp10--;
        } else {
          many = many || c != '0';
        }
      } else if (c == '_') {
        if (!prev_digit || i + 1 >= n || !is_digit(s[i + 1])) return -1;
        prev_digit = false;
      } else {
        break;
      }
    }
  }
  if (!any) return -1;
  int64_t e = 0;
  if (i < n && lower(s[i]) == 'e') {
    i++;
    bool eneg = false;
    if (i < n && (s[i] == '+' || s[i] == '-')) {
      eneg = s[i] == '-';
      i++;
    }
    bool edig = false;
    prev_digit = false;
    for (; i < n; i++) {
      const unsigned char c = s[i];
      if (is_digit(c)) {
        edig = true;
        prev_digit = true;
        if (e < 100000000) e = e * 10 + (c - '0');
      } else if (c == '_') {
        if (!prev_digit || i + 1 >= n || !is_digit(s[i + 1])) return -1;
        prev_digit = false;
      } else {
        break;
      }
    }
    if (!edig) return -1;
    if (eneg) e = -e;
  }
  if (i != n) return -1;
  if (w == 0) {
    *out = bits_to_double(sign);
    return 0;
  }
  const int64_t q = exp10 + e;
  uint64_t bits = el_convert(q, w, tab);
  if (many && bits != el_convert(q, w + 1, tab)) {
    // exact conversion from all the digits
    BigDec a;
    a.nd = 0;
    a.dp = 0;
    a.trunc = false;
    bool seen_point = false;
    for (int j = body; j < n; j++) {
      const unsigned char c = s[j];
      if (c == '.') {
        seen_point = true;
        continue;
      }
      if (c == '_') continue;
      if (!is_digit(c)) break;
      if (c == '0' && a.nd == 0) {  // leading zeros
        if (seen_point) a.dp--;
        continue;
      }
      if (!seen_point) a.dp++;
      if (a.nd < BigDec::kMax) {
        a.d[a.nd++] = (unsigned char)(c - '0');
      } else if (c != '0') {
        a.trunc = true;
      }
    }
    int64_t dp = (int64_t)a.dp + e;
    if (dp > 100000) dp = 100000;
    if (dp < -100000) dp = -100000;
    a.dp = (int)dp;
    bd_trim(a);
    bits = bd_to_bits(a);
  }
  *out = bits_to_double(sign | bits);
  return 0;
}

// ---- SWAR fast path for plain numerals --------------------------------------
// [+-]digits[.digits] with <= 19 digits in all, no exponent or underscore: the
// token's (<= 24) bytes arrive as three little-endian words; digit runs are
// validated and converted eight at a time (Lemire's eight-digit trick) and
// the value goes through the same Eisel-Lemire step as nc_parse.  Returns
// false for any other shape (the caller then runs nc_parse).

NC_HD int ctz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __ffsll((long long)x) - 1;
#else
  return __builtin_ctzll(x);
#endif
}

// bytes [off, off + 8) of the 24-byte token (W[3] must be 0), off in [-8, 16];
// bytes before 0 read as '0'
NC_HD uint64_t bytes8(const uint64_t* W, int off) {
  if (off < 0) {
    const int k = -off;  // 1..8 leading fill bytes
    const uint64_t x = k >= 8 ? 0 : (W[0] << (8 * k));
    const uint64_t fill = k >= 8 ? ~0ULL : ((1ULL << (8 * k)) - 1);
    return x | (0x3030303030303030ULL & fill);
  }
  // word selection by compare/select on constant indices (W stays in
  // registers; a dynamic W[q] would place the array in local memory)
  const int q = off >> 3, r = off & 7;
  const uint64_t lo = q == 0 ? W[0] : (q == 1 ? W[1] : W[2]);
  const uint64_t hi = q == 0 ? W[1] : (q == 1 ? W[2] : W[3]);
  return (lo >> (8 * r)) | ((hi << 1) << (63 - 8 * r));  // r == 0: hi << 64 -> 0
}

NC_HD bool eight_digits(uint64_t x) {
  return (((x + 0x4646464646464646ULL) | (x - 0x3030303030303030ULL)) & 0x8080808080808080ULL) == 0;
}

NC_HD uint64_t parse8(uint64_t x) {
  x = (x & 0x0F0F0F0F0F0F0F0FULL) * 2561 >> 8;
  x = (x & 0x00FF00FF00FF00FFULL) * 6553601 >> 16;
  return (x & 0x0000FFFF0000FFFFULL) * 42949672960001ULL >> 32;
}

// digits [a, a + n) (0 <= n <= 8) right-aligned: bytes before the run read '0'
NC_HD bool digits8(const uint64_t* W, int a, int n, uint64_t& v) {
  uint64_t x = bytes8(W, a + n - 8);
  const int k = 8 - n;
  if (k > 0) {
    const uint64_t fill = k >= 8 ? ~0ULL : ((1ULL << (8 * k)) - 1);
    x = (x & ~fill) | (0x3030303030303030ULL & fill);
  }
  if (!eight_digits(x)) return false;
  v = parse8(x);
  return true;
}

// digits [a, a + n) (0 <= n <= 16) as an integer; false if a byte is not a
// digit (no recursion: device stacks are sized statically)
NC_HD bool digits_value(const uint64_t* W, int a, int n, uint64_t& v) {
  v = 0;
  if (n == 0) return true;
  if (n <= 8) return digits8(W, a, n, v);
  uint64_t hi, lo;
  if (!digits8(W, a, n - 8, hi) || !digits8(W, a + n - 8, 8, lo)) return false;
  v = hi * 100000000ULL + lo;
  return true;
}

NC_HD bool nc_parse_simple(const uint64_t* W, int len, double* out, const uint64_t (*tab)[2]) {
  if (len < 1 || len > 24) return false;
  const unsigned c0 = (unsigned)(W[0] & 255u);
  const int s0 = (c0 == '-' || c0 == '+') ? 1 : 0;
  // first '.' (zero-byte test on W ^ '.')
  int p = len;
  for (int q = 0; q < 3; q++) {
    const uint64_t t = W[q] ^ 0x2E2E2E2E2E2E2E2EULL;
    const uint64_t z = (t - 0x0101010101010101ULL) & ~t & 0x8080808080808080ULL;
    if (z) {
      const int pos = 8 * q + (ctz64(z) >> 3);
      if (pos < len) p = pos;
      break;
    }
  }
  const int ni = p - s0, nf = p < len ? len - p - 1 : 0;
  if (ni < 0 || ni + nf < 1 || ni > 16 || nf > 16 || ni + nf > 19) return false;
  uint64_t iv, fv;
  if (!digits_value(W, s0, ni, iv) || !digits_value(W, p + 1, nf, fv)) return false;
  uint64_t scale = (nf & 1) ? 10 : 1;  // 10^nf, nf <= 16
  if (nf & 2) scale *= 100;
  if (nf & 4) scale *= 10000;
  if (nf & 8) scale *= 100000000;
  if (nf & 16) scale *= 10000000000000000ULL;
  const uint64_t m = iv * scale + fv;
  const uint64_t bits = m == 0 ? 0 : el_convert(-(int64_t)nf, m, tab);
  *out = bits_to_double(bits | (c0 == '-' ? 0x8000000000000000ULL : 0));
  return true;
}

// ---- formatting ----------------------------------------------------------

NC_HD uint32_t pow5bits(int32_t e) { return (uint32_t)(((uint32_t)e * 1217359) >> 19) + 1; }
NC_HD uint32_t log10pow2(int32_t e) { return ((uint32_t)e * 78913) >> 18; }
NC_HD uint32_t log10pow5(int32_t e) { return ((uint32_t)e * 732923) >> 20; }

NC_HD uint32_t pow5factor(uint64_t v) {
  uint32_t count = 0;
  for (;;) {
    const uint64_t q = v / 5;
    if (v - 5 * q != 0) break;
    v = q;
    ++count;
  }
  return count;
}

NC_HD uint64_t mul_shift64(uint64_t m, const uint64_t* mul, int32_t j) {
  // mul = {lo, hi}; (m * mul) >> j, j >= 64
  uint64_t high1, low1, high0, low0;
  mul128(m, mul[1], low1, high1);
  mul128(m, mul[0], low0, high0);
  (void)low0;
  const uint64_t sum = high0 + low1;
  if (sum < high0) ++high1;
  const int d = j - 64;
  return (high1 << (64 - d)) | (sum >> d);
}

// Ryu's d2d: shortest decimal (output * 10^exp) of a finite nonzero double.
NC_HD void ryu_d2d(uint64_t ieee_m, uint32_t ieee_e, uint64_t& output, int32_t& exp10, const uint64_t (*pow5inv)[2],
                   const uint64_t (*pow5)[2]) {
  int32_t e2;
  uint64_t m2;
  if (ieee_e == 0) {
    e2 = 1 - 1023 - 52 - 2;
    m2 = ieee_m;
  } else {
    e2 = (int32_t)ieee_e - 1023 - 52 - 2;
    m2 = (1ULL << 52) | ieee_m;
  }
  const bool even = (m2 & 1) == 0;
  const bool accept_bounds = even;
  const uint64_t mv = 4 * m2;
  const uint32_t mm_shift = ieee_m != 0 || ieee_e <= 1;
  uint64_t vr, vp, vm;
  int32_t e10;
  bool vm_tz = false, vr_tz = false;
  if (e2 >= 0) {
    const uint32_t q = log10pow2(e2) - (e2 > 3);
    e10 = (int32_t)q;
    const int32_t k = 125 + (int32_t)pow5bits((int32_t)q) - 1;
    const int32_t i = -e2 + (int32_t)q + k;
    vr = mul_shift64(4 * m2, pow5inv[q], i);
    vp = mul_shift64(4 * m2 + 2, pow5inv[q], i);
    vm = mul_shift64(4 * m2 - 1 - mm_shift, pow5inv[q], i);
    if (q <= 21) {
      const uint32_t mv_mod5 = (uint32_t)(mv - 5 * (mv / 5));
      if (mv_mod5 == 0) {
        vr_tz = pow5factor(mv) >= q;
      } else if (accept_bounds) {
        vm_tz = pow5factor(mv - 1 - mm_shift) >= q;
      } else {
        vp -= pow5factor(mv + 2) >= q;
      }
    }
  } else {
    const uint32_t q = log10pow5(-e2) - (-e2 > 1);
    e10 = (int32_t)q + e2;
    const int32_t i = -e2 - (int32_t)q;
    const int32_t k = (int32_t)pow5bits(i) - 125;
    const int32_t j = (int32_t)q - k;
    vr = mul_shift64(4 * m2, pow5[i], j);
    vp = mul_shift64(4 * m2 + 2, pow5[i], j);
    vm = mul_shift64(4 * m2 - 1 - mm_shift, pow5[i], j);
    if (q <= 1) {
      vr_tz = true;
      if (accept_bounds) {
        vm_tz = mm_shift == 1;
      } else {
        --vp;
      }
    } else if (q < 63) {
      vr_tz = (mv & ((1ULL << q) - 1)) == 0;
    }
  }
  int32_t removed = 0;
  uint8_t last = 0;
  if (vm_tz || vr_tz) {
    for (;;) {
      const uint64_t vp10 = vp / 10, vm10 = vm / 10;
      if (vp10 <= vm10) break;
      const uint32_t vm_mod = (uint32_t)(vm - 10 * vm10);
      const uint64_t vr10 = vr / 10;
      const uint32_t vr_mod = (uint32_t)(vr - 10 * vr10);
      vm_tz &= vm_mod == 0;
      vr_tz &= last == 0;
      last = (uint8_t)vr_mod;
      vr = vr10;
      vp = vp10;
      vm = vm10;
      ++removed;
    }
    if (vm_tz) {
      for (;;) {
        const uint64_t vm10 = vm / 10;
        const uint32_t vm_mod = (uint32_t)(vm - 10 * vm10);
        if (vm_mod != 0) break;
        const uint64_t vp10 = vp / 10, vr10 = vr / 10;
        const uint32_t vr_mod = (uint32_t)(vr - 10 * vr10);
        vr_tz &= last == 0;
        last = (uint8_t)vr_mod;
        vr = vr10;
        vp = vp10;
        vm = vm10;
        ++removed;
      }
    }
    if (vr_tz && last == 5 && vr % 2 == 0) last = 4;  // round even on an exact ...50..0
    output = vr + ((vr == vm && (!accept_bounds || !vm_tz)) || last >= 5);
  } else {
    bool round_up = false;
    const uint64_t vp100 = vp / 100, vm100 = vm / 100;
    if (vp100 > vm100) {
      const uint64_t vr100 = vr / 100;
      const uint32_t vr_mod = (uint32_t)(vr - 100 * vr100);
      round_up = vr_mod >= 50;
      vr = vr100;
      vp = vp100;
      vm = vm100;
      removed += 2;
    }
    for (;;) {
      const uint64_t vp10 = vp / 10, vm10 = vm / 10;
      if (vp10 <= vm10) break;
      const uint64_t vr10 = vr / 10;
      const uint32_t vr_mod = (uint32_t)(vr - 10 * vr10);
      round_up = vr_mod >= 5;
      vr = vr10;
      vp = vp10;
      vm = vm10;
      ++removed;
    }
    output = vr + (vr == vm || round_up);
  }
  exp10 = e10 + removed;
}

NC_HD int decimal_length(uint64_t v) {  // digits of v (>= 1)
  int n = 1;
  while (v >= 10) {
    v /= 10;
    n++;
  }
  return n;
}

// v's nd decimal digits into dst[0, nd), written from the right (no
// temporary: dst may be shared memory)
NC_HD void put_digits(uint64_t v, int nd, char* dst) {
  for (int i = nd - 1; i >= 0; i--) {
    const uint64_t q = v / 10;
    dst[i] = (char)('0' + (v - 10 * q));
    v = q;
  }
}

// format_number(v) in two steps so a caller can place the text before
// producing it: nc_prepare decides the form and its length, nc_emit writes
// exactly that many characters.
struct Fmt {
  uint64_t m;   // integer value, or the shortest decimal significand
  int32_t e10;  // repr: value = m * 10^e10
  int nd;       // digits of m
  int kind;     // 0 integer, 1 repr exponent form, 2 repr 0.000ddd, 3 repr ddd000.0, 4 repr ddd.ddd, 5 inf, 6 nan
  bool neg;
  int len;
};

NC_HD Fmt nc_prepare(double v, const uint64_t (*pow5inv)[2], const uint64_t (*pow5)[2]) {
  Fmt f{};
  const uint64_t bits = double_to_bits(v);
  f.neg = (bits >> 63) != 0;
  const uint32_t ieee_e = (uint32_t)((bits >> 52) & 0x7FF);
  const uint64_t ieee_m = bits & ((1ULL << 52) - 1);
  if (ieee_e == 0x7FF) {
    f.kind = ieee_m != 0 ? 6 : 5;
    f.len = ieee_m != 0 ? 3 : 3 + (f.neg ? 1 : 0);
    return f;
  }
  const double a = f.neg ? -v : v;
  if (a < 1e16 && a == (double)(int64_t)a) {  // integral: str(int(v)); -0.0 -> "0"
    f.kind = 0;
    f.m = (uint64_t)(int64_t)a;
    f.nd = decimal_length(f.m);
    f.neg = f.neg && f.m != 0;
    f.len = f.nd + (f.neg ? 1 : 0);
    return f;
  }
  ryu_d2d(ieee_m, ieee_e, f.m, f.e10, pow5inv, pow5);
  f.nd = decimal_length(f.m);
  const int decpt = f.nd + f.e10;
  int n = f.neg ? 1 : 0;
  if (decpt <= -4 || decpt > 16) {
    f.kind = 1;
    int x = decpt - 1;
    if (x < 0) x = -x;
    n += 1 + (f.nd > 1 ? f.nd : 0) + 2 + (x < 10 ? 2 : decimal_length((uint64_t)x));
  } else if (decpt <= 0) {
    f.kind = 2;
    n += 2 + (-decpt) + f.nd;
  } else if (decpt >= f.nd) {
    f.kind = 3;
    n += decpt + 2;
  } else {
    f.kind = 4;
    n += f.nd + 1;
  }
  f.len = n;
  return f;
}

NC_HD void nc_emit(const Fmt& f, char* dst) {
  int n = 0;
  if (f.kind == 6) {
    dst[0] = 'n', dst[1] = 'a', dst[2] = 'n';
    return;
  }
  if (f.neg) dst[n++] = '-';
  if (f.kind == 5) {
    dst[n++] = 'i', dst[n++] = 'n', dst[n++] = 'f';
    return;
  }
  if (f.kind == 0) {
    put_digits(f.m, f.nd, dst + n);
    return;
  }
  const int nd = f.nd, decpt = nd + f.e10;
  if (f.kind == 1) {
    // d[.ddd]e[+-]xx
    if (nd > 1) {
      put_digits(f.m, nd, dst + n + 1);  // digits at n+1 .. n+nd, then move the first one left
      dst[n] = dst[n + 1];
      dst[n + 1] = '.';
      n += nd + 1;
    } else {
      dst[n++] = (char)('0' + f.m);
    }
    dst[n++] = 'e';
    int x = decpt - 1;
    dst[n++] = x < 0 ? '-' : '+';
    if (x < 0) x = -x;
    if (x < 10) {
      dst[n++] = '0';
      dst[n++] = (char)('0' + x);
    } else {
      put_digits((uint64_t)x, decimal_length((uint64_t)x), dst + n);
    }
  } else if (f.kind == 2) {
    dst[n++] = '0';
    dst[n++] = '.';
    for (int i = 0; i < -decpt; i++) dst[n++] = '0';
    put_digits(f.m, nd, dst + n);
  } else if (f.kind == 3) {
    put_digits(f.m, nd, dst + n);
    n += nd;
    for (int i = nd; i < decpt; i++) dst[n++] = '0';
    dst[n++] = '.';
    dst[n++] = '0';
  } else {
    // ddd.ddd: digits at n .. n+nd, then open the point at decpt
    put_digits(f.m / 1, nd, dst + n);  // all digits, shifted below
    for (int i = nd; i > decpt; i--) dst[n + i] = dst[n + i - 1];
    dst[n + decpt] = '.';
  }
}

// format_number(v) (asciigrid.py:160-167) into buf (>= 25 bytes); returns
// the length.  Non-finite values print as CPython's repr ('inf', 'nan').
NC_HD int nc_format(double v, char* buf, const uint64_t (*pow5inv)[2], const uint64_t (*pow5)[2]) {
  const Fmt f = nc_prepare(v, pow5inv, pow5);
  nc_emit(f, buf);
  return f.len;
}

}  // namespace nc

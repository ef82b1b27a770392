/* Dumps the AVX-512 VRSQRT14PD result for every (exponent parity, top-15
 * mantissa bits) class of the input, and checks that those 16 bits (plus an
 * exact power-of-4 scaling) determine the result -- except exact powers of
 * four, whose reciprocal square root is returned exact (1.0 for 1.0, while
 * the rest of its class gives 0x1.fffap-1).
 * Build: gcc -O2 -mavx512f rsqrt14_probe.c -o rsqrt14_probe
 * Output (stdout, binary): 65536 little-endian uint64 result bit patterns,
 * index = parity * 32768 + m, input = (parity ? 0.5 : 1.0) * (1 + m / 2^15 + 2^-52). */
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double rs(double x) {
  double r[8];
  _mm512_storeu_pd(r, _mm512_rsqrt14_pd(_mm512_set1_pd(x)));
  return r[0];
}
static double from_bits(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
static uint64_t bits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static uint64_t rnd(void) { return ((uint64_t)rand() << 42) ^ ((uint64_t)rand() << 21) ^ (uint64_t)rand(); }

int main(void) {
  srand(12345);
  long bad = 0;
  for (long t = 0; t < 4000000; t++) {
    uint64_t u = rnd() & 0x000fffffffffffffULL;
    int e = 0x3c0 + (int)(rnd() % 0x40);  /* exponents 2^-63 .. 2^0 */
    double x = from_bits(((uint64_t)e << 52) | u);
    double x2 = from_bits(((uint64_t)e << 52) | (u & ~((1ULL << 37) - 1)) | (rnd() & ((1ULL << 37) - 1)));
    if (bits(rs(x)) != bits(rs(x2))) bad++;         /* only the top 15 mantissa bits matter */
    if (bits(rs(4.0 * x)) != bits(0.5 * rs(x))) bad++; /* power-of-4 scaling is exact */
  }
  for (int par = 0; par < 2; par++)
    for (uint64_t m = 0; m < 32768; m++) {  /* every class: lowest, second and highest member */
      const uint64_t b = ((uint64_t)(0x3ff - par) << 52) | (m << 37);
      const double lo = rs(from_bits(b)), lo1 = rs(from_bits(b | 1)), hi = rs(from_bits(b | ((1ULL << 37) - 1)));
      if (bits(lo1) != bits(hi)) bad++;
      if (bits(lo) != bits(lo1) && !(par == 0 && m == 0 && lo == 1.0)) bad++;
    }
  for (int e = -60; e <= 60; e += 2)  /* exact powers of four */
    if (rs(from_bits((uint64_t)(0x3ff + e) << 52)) != from_bits((uint64_t)(0x3ff - e / 2) << 52)) bad++;
  if (bad) { fprintf(stderr, "rsqrt14 model violated %ld times\n", bad); return 1; }
  for (int par = 0; par < 2; par++)
    for (uint64_t m = 0; m < 32768; m++) {
      uint64_t o = bits(rs(from_bits(((uint64_t)(0x3ff - par) << 52) | (m << 37) | 1)));
      fwrite(&o, 8, 1, stdout);
    }
  return 0;
}

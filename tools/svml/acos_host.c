/* Host build of csrc/wg_acos.h (the device arccos restated in C) for the CPU
 * tests: gcc -O2 -fPIC -shared -ffp-contract=off acos_host.c -o libacos_host.so -lm */
#include <stdint.h>

#include "../../paper_2506_23364_b200/csrc/wg_acos.h"

void wg_acos_host(const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; i++) out[i] = wg_acos(x[i]);
}

void wg_rsqrt14_host(const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; i++) out[i] = wg_rsqrt14(x[i]);
}

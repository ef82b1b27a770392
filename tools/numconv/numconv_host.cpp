// Host build of csrc/wg_numconv.cuh (the device ASCII-grid number parser and
// formatter) for checking it against CPython on millions of inputs:
//   g++ -O2 -shared -fPIC -o tools/numconv/libnumconv.so tools/numconv/numconv_host.cpp
// (tools/numconv/check.py builds and drives it).
#include <stdint.h>

#define NC_TABLE static const
#include "../../paper_2506_23364_b200/csrc/pow5_tables.inc"
#include "../../paper_2506_23364_b200/csrc/wg_numconv.cuh"

extern "C" {

void nc_parse_many(const unsigned char* text, const int64_t* offs, const int32_t* lens, int64_t n, double* out,
                   int32_t* status) {
  for (int64_t i = 0; i < n; i++) status[i] = nc::nc_parse(text + offs[i], lens[i], &out[i], (const uint64_t(*)[2])kEL);
}

// the SWAR fast path: status 1 = handled (out set), 0 = declined
void nc_parse_simple_many(const unsigned char* text, const int64_t* offs, const int32_t* lens, int64_t n, double* out,
                          int32_t* status) {
  for (int64_t i = 0; i < n; i++) {
    uint64_t W[4] = {0, 0, 0, 0};
    const int len = lens[i];
    if (len > 24) {
      status[i] = 0;
      continue;
    }
    __builtin_memcpy(W, text + offs[i], len);
    status[i] = nc::nc_parse_simple(W, len, &out[i], (const uint64_t(*)[2])kEL) ? 1 : 0;
  }
}

void nc_format_many(const double* v, int64_t n, char* out, int32_t* lens) {
  for (int64_t i = 0; i < n; i++)
    lens[i] = nc::nc_format(v[i], out + 32 * i, (const uint64_t(*)[2])kPow5Inv, (const uint64_t(*)[2])kPow5);
}
}

// Content digest of device-resident payloads for the executor's
// content-addressed cache (replaces the reference's host SHA-256 over
// .tobytes(), workflow.py:465-529, which runs at ~0.33 GiB/s and dominated
// cold and warm latency at scale -- SURVEY.md 0.7 / 8(f) rank 1).
//
// 256-bit result = four independent 64-bit lanes.  The payload is cut into
// 256-byte chunks; each chunk is folded by a SplitMix-style nonlinear absorb
// with its chunk index mixed in, and the four lane values of all chunks are
// summed mod 2^64.  The sum is commutative, so the digest is independent of
// launch geometry and thread scheduling, while the index mixing keeps it
// position-sensitive.  SPEC.md:444 asks only for a stable hash of >= 128 bits;
// the executor feeds these 32 bytes (plus type tags and headers) into a host
// SHA-256 to form the 64-hex cache keys.
#include "wg_internal.cuh"

namespace {

__device__ const unsigned long long kSeeds[4] = {0x243F6A8885A308D3ULL, 0x13198A2E03707344ULL, 0xA4093822299F31D0ULL,
                                          0x082EFA98EC4E6C89ULL};
constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// One pass over `rows` rows of `row_bytes` bytes each, row r starting at
// data + r*ld: chunk (r, c) is the c-th 256-byte piece of row r and is mixed
// with its global index r*cpr + c (cpr = chunks per row), so a strided window
// hashes exactly like the same rows stored contiguously.
__global__ void digest_kernel(const unsigned char* __restrict__ data, int64_t rows, int64_t row_bytes, int64_t ld,
                              unsigned long long* __restrict__ out) {
  const int64_t cpr = (row_bytes + 255) / 256;
  const int64_t nchunks = rows * cpr;
  unsigned long long acc[4] = {0, 0, 0, 0};
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = c / cpr, k = c - r * cpr;
    const unsigned char* row = data + r * ld;
    const int64_t nbytes = row_bytes;
    unsigned long long h[4];
#pragma unroll
    for (int l = 0; l < 4; l++) h[l] = mix(kSeeds[l] ^ ((unsigned long long)c * kGolden));
    const int64_t base = k * 256;
    const bool full = base + 256 <= nbytes && ((((uintptr_t)(row + base)) & 15) == 0);
    if (full) {
      const ulonglong2* p = reinterpret_cast<const ulonglong2*>(row + base);
#pragma unroll 4
      for (int q = 0; q < 16; q++) {
        const ulonglong2 v = __ldg(p + q);
        h[q & 3] = mix(h[q & 3] ^ v.x) + v.y;
        h[(q + 1) & 3] ^= mix(v.y + kGolden * (unsigned long long)(q + 1));
      }
    } else {
      // ragged or unaligned chunk: byte-wise little-endian words, zero padded
      for (int q = 0; q < 16; q++) {
        unsigned long long x = 0, y = 0;
        for (int b = 0; b < 8; b++) {
          const int64_t i0 = base + 16 * q + b, i1 = i0 + 8;
          if (i0 < nbytes) x |= (unsigned long long)row[i0] << (8 * b);
          if (i1 < nbytes) y |= (unsigned long long)row[i1] << (8 * b);
        }
        h[q & 3] = mix(h[q & 3] ^ x) + y;
        h[(q + 1) & 3] ^= mix(y + kGolden * (unsigned long long)(q + 1));
      }
    }
#pragma unroll
    for (int l = 0; l < 4; l++) acc[l] += mix(h[l] + (unsigned long long)l);
  }
#pragma unroll
  for (int l = 0; l < 4; l++) {
    unsigned long long v = acc[l];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + l, v);
  }
}

}  // namespace

extern "C" int wg_digest2d(const void* data, int64_t rows, int64_t row_bytes, int64_t ld_bytes, uint64_t* out,
                           void* stream) {
  if (!out) return wg::set_error(WG_EARG, "null digest buffer");
  if (rows <= 0 || row_bytes <= 0) return WG_OK;
  if (!data || ld_bytes < row_bytes) return wg::set_error(WG_EARG, "bad digest arguments");
  const int64_t nchunks = rows * ((row_bytes + 255) / 256);
  digest_kernel<<<wg::stream_grid(nchunks, 256, 4), 256, 0, wg::as_stream(stream)>>>(
      reinterpret_cast<const unsigned char*>(data), rows, row_bytes, ld_bytes,
      reinterpret_cast<unsigned long long*>(out));
  WG_LAUNCH_CHECK("digest_kernel");
  return WG_OK;
}

extern "C" int wg_digest(const void* data, int64_t nbytes, uint64_t* out, void* stream) {
  return wg_digest2d(data, 1, nbytes, nbytes, out, stream);
}

// ESRI ASCII grid reader/writer on the device:
// /root/reference/pkg/src/demflow/asciigrid.py -- parse_ascii_grid (42-143)
// tokenises the body with str.split() and converts every token with
// np.array(tokens, dtype=float64); write_ascii_grid (146-157) joins
// format_number(v) (160-167) with single spaces, one raster row per line.
//
// Reader: (1) tokenise -- one pass over the body marks token starts (a
// non-whitespace byte after whitespace; str.split()'s ASCII whitespace is
// \t \n \v \f \r \x1c-\x1f and space), per-4-KiB-tile counts, a scan of the
// tile counts, and a scatter of the start offsets; (2) parse -- one thread per
// token runs nc_parse (wg_numconv.cuh: CPython float() semantics, correctly
// rounded) and records the first invalid token.  Writer: one thread per value
// runs nc_format (format_number: int digits or shortest round-trip repr);
// pass 1 sums the formatted lengths per block, a scan places the blocks,
// pass 2 formats again into shared memory and streams each block's bytes out.
#include "wg_internal.cuh"

#define NC_TABLE __device__ const
#include "pow5_tables.inc"
#include "wg_numconv.cuh"

namespace {

constexpr int kTokThreads = 256;
constexpr int kTokBytes = 16;  // per thread
constexpr int64_t kTokTile = (int64_t)kTokThreads * kTokBytes;
constexpr int kFmtThreads = 256;
constexpr int kFmtMax = 25;  // longest format_number output (24) + separator
constexpr int kFmtPer = 4;   // values per thread in the one-pass writer

__device__ __forceinline__ bool is_ws(unsigned c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }

// whitespace bytes of a 32-bit word as 0xFF bytes (SWAR): space, \t..\r,
// \x1c..\x1f
__device__ __forceinline__ unsigned ws_bytes(unsigned w) {
  return __vcmpeq4(w, 0x20202020u) | __vcmpltu4(__vsub4(w, 0x09090909u), 0x05050505u) |
         __vcmpltu4(__vsub4(w, 0x1c1c1c1cu), 0x04040404u);
}

// one bit per byte (byte k -> bit k) of a 0x00/0xFF byte mask
__device__ __forceinline__ unsigned byte_bits(unsigned m) { return ((m & 0x01010101u) * 0x01020408u) >> 24; }

// token-start bits of this thread's 16 bytes [p0, p0 + 16) within [lo, n):
// SWAR classification of four words; bytes outside [lo, n) count as
// whitespace; the byte before p0 comes from the previous lane (lane 0 loads it)
__device__ __forceinline__ unsigned start_bits(const unsigned char* __restrict__ t, int64_t p0, int64_t lo, int64_t n,
                                               unsigned& nonascii) {
  uint4 v;
  if (p0 + kTokBytes <= n) {
    v = __ldg(reinterpret_cast<const uint4*>(t + p0));
  } else {
    unsigned char b[kTokBytes];
    for (int k = 0; k < kTokBytes; k++) b[k] = (p0 + k < n) ? __ldg(t + p0 + k) : ' ';
    v = *reinterpret_cast<const uint4*>(b);
  }
  unsigned ws = byte_bits(ws_bytes(v.x)) | (byte_bits(ws_bytes(v.y)) << 4) | (byte_bits(ws_bytes(v.z)) << 8) |
                (byte_bits(ws_bytes(v.w)) << 12);
  unsigned hi = (v.x | v.y | v.z | v.w) & 0x80808080u;
  if (p0 < lo) {  // header bytes: neither tokens nor body
    const int64_t k = lo - p0;
    const unsigned out = k >= kTokBytes ? 0xFFFFu : ((1u << k) - 1u);
    ws |= out;
    if (k >= kTokBytes) hi = 0;
    else {
      const unsigned char* pb = reinterpret_cast<const unsigned char*>(&v);
      hi = 0;
      for (int q = (int)k; q < kTokBytes; q++) hi |= pb[q] & 0x80u;
    }
  }
  if (p0 + kTokBytes > n) {
    const int64_t k = n - p0;  // in-range bytes (< 16)
    ws |= k <= 0 ? 0xFFFFu : (0xFFFFu << k) & 0xFFFFu;
  }
  nonascii |= hi ? 1u : 0u;
  const int lane = threadIdx.x & 31;
  unsigned prev = __shfl_up_sync(0xffffffffu, ws >> 15, 1);
  if (lane == 0) prev = (p0 <= lo) ? 1u : (is_ws(__ldg(t + p0 - 1)) ? 1u : 0u);
  return ~ws & ((ws << 1) | prev) & 0xFFFFu;
}

__global__ void tok_count_kernel(const unsigned char* __restrict__ t, int64_t lo, int64_t n,
                                 unsigned long long* __restrict__ tile_counts, unsigned* __restrict__ flags) {
  const int64_t p0 = (int64_t)blockIdx.x * kTokTile + (int64_t)threadIdx.x * kTokBytes;
  unsigned nonascii = 0;
  const unsigned bits = start_bits(t, p0, lo, n, nonascii);
  unsigned c = __popc(bits);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ unsigned s[kTokThreads / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  if (__any_sync(0xffffffffu, nonascii) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int w = 0; w < kTokThreads / 32; w++) tot += s[w];
    tile_counts[blockIdx.x] = tot;
  }
}

// exclusive scan of n counts in place (one block of 1024); total to *total.
// Per 1024-element chunk: warp shuffles, one shared pass over the 32 warp
// sums, a running carry.
__global__ void scan_kernel(unsigned long long* __restrict__ v, int64_t n, unsigned long long* __restrict__ total) {
  __shared__ unsigned long long s_warp[32];
  __shared__ unsigned long long s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const unsigned long long x = i < n ? v[i] : 0;
    unsigned long long y = x;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    if (lane == 31) s_warp[warp] = y;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long w = s_warp[lane];
      unsigned long long z = w;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += t;
      }
      s_warp[lane] = z - w;  // exclusive warp offsets
    }
    __syncthreads();
    const unsigned long long carry = s_carry;
    if (i < n) v[i] = carry + s_warp[warp] + y - x;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_warp[31] + y;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s_carry;
}

__global__ void tok_scatter_kernel(const unsigned char* __restrict__ t, int64_t lo, int64_t n,
                                   const unsigned long long* __restrict__ tile_offsets, int64_t* __restrict__ starts,
                                   int64_t cap, int64_t base) {
  const int64_t p0 = (int64_t)blockIdx.x * kTokTile + (int64_t)threadIdx.x * kTokBytes;
  unsigned dummy = 0;
  unsigned bits = start_bits(t, p0, lo, n, dummy);
  const unsigned c = __popc(bits);
  // block exclusive scan of c
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __shared__ unsigned ws[kTokThreads / 32];
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  unsigned woff = 0;
  for (int w = 0; w < warp; w++) woff += ws[w];
  int64_t idx = (int64_t)tile_offsets[blockIdx.x] + woff + x - c;
  while (bits) {
    const int k = __ffs(bits) - 1;
    bits &= bits - 1;
    if (idx < cap) starts[idx] = base + p0 + k;
    idx++;
  }
}

// Fast path for the common numeral shape [+-]digits[.digits] (no exponent,
// no underscore, <= 19 significant digits): the token's bytes come from six
// word loads held in registers, the token end from a SWAR whitespace scan,
// and the value from the same Eisel-Lemire conversion nc_parse uses.  Any
// other shape (or a token near the end of the text) returns false and the
// caller runs the general nc_parse.
__device__ __forceinline__ bool parse_fast(const unsigned char* __restrict__ t, int64_t s, int64_t n, double* v,
                                           int64_t* len_out) {
  if (s + 28 > n) return false;
  uint32_t w[6];
  const uint32_t* base = reinterpret_cast<const uint32_t*>(t) + (s >> 2);
  const unsigned sh = (unsigned)(s & 3) * 8;
#pragma unroll
  for (int k = 0; k < 6; k++) w[k] = __funnelshift_r(__ldg(base + k), __ldg(base + k + 1), sh);
  unsigned wsm = 0;
#pragma unroll
  for (int k = 0; k < 6; k++) wsm |= byte_bits(ws_bytes(w[k])) << (4 * k);
  if (wsm == 0) return false;  // token of 24+ bytes
  const int len = __ffs(wsm) - 1;
  *len_out = len;
  // the token's bytes as three little-endian words (+ a zero word)
  uint64_t W[4];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const int b0 = 8 * k;  // bytes beyond the token are masked to 0 below
    W[k] = (uint64_t)w[2 * k] | ((uint64_t)w[2 * k + 1] << 32);
    if (len < b0 + 8) W[k] &= len <= b0 ? 0ULL : (~0ULL >> (64 - 8 * (len - b0)));
  }
  W[3] = 0;
  return nc::nc_parse_simple(W, len, v, (const uint64_t(*)[2])kEL);
}

__global__ void parse_kernel(const unsigned char* __restrict__ t, int64_t n, const int64_t* __restrict__ starts,
                             int64_t count, double* __restrict__ out, unsigned long long* __restrict__ first_bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = starts[i];
    double v = 0.0;
    int64_t len;
    if (!parse_fast(t, s, n, &v, &len)) {
      int64_t e = s;
      while (e < n && !is_ws(__ldg(t + e))) e++;
      len = e - s;
      const int rc = len > 0x7fffffff ? -1 : nc::nc_parse(t + s, (int)len, &v, (const uint64_t(*)[2])kEL);
      if (rc != 0) atomicMin(first_bad, (unsigned long long)i);
    }
    out[i] = v;
  }
}


// One pass with a decoupled look-back: block b (ids taken in execution
// order from a counter, so every predecessor is running or done) formats its
// 256 values once into shared memory, publishes its byte count, sums its
// predecessors' counts (stopping at the first inclusive prefix) and streams
// its bytes to their final offset.  Status word: 2 flag bits (1 = block
// total, 2 = inclusive prefix) over a 62-bit count.
constexpr unsigned long long kFlagAgg = 1ULL << 62, kFlagIncl = 2ULL << 62, kValMask = (1ULL << 62) - 1;

__global__ void __launch_bounds__(kFmtThreads) fmt_kernel(const double* __restrict__ v, int64_t count, int64_t cols,
                                                          unsigned char* __restrict__ out,
                                                          unsigned long long* __restrict__ status,
                                                          unsigned long long* __restrict__ counter,
                                                          unsigned long long* __restrict__ nbytes, int64_t nblocks) {
  __shared__ unsigned char stage[kFmtThreads * kFmtPer * kFmtMax];
  __shared__ unsigned ws[kFmtThreads / 32];
  __shared__ unsigned long long s_bid, s_off;
  __shared__ int64_t s_col0;
  if (threadIdx.x == 0) {
    const unsigned long long bid = atomicAdd(counter, 1ULL);
    s_bid = bid;
    s_col0 = (int64_t)(bid * kFmtThreads * kFmtPer) % cols;
  }
  __syncthreads();
  const unsigned long long bid = s_bid;
  // kFmtPer consecutive values per thread
  const int64_t i0 = ((int64_t)bid * kFmtThreads + threadIdx.x) * kFmtPer;
  nc::Fmt f[kFmtPer];
  unsigned lens[kFmtPer];
  unsigned nl = 0;  // '\n' after value k <=> bit k
  unsigned len = 0;
  int64_t col = (s_col0 + (int64_t)threadIdx.x * kFmtPer) % cols;
#pragma unroll
  for (int k = 0; k < kFmtPer; k++) {
    lens[k] = 0;
    if (i0 + k < count) {
      f[k] = nc::nc_prepare(v[i0 + k], (const uint64_t(*)[2])kPow5Inv, (const uint64_t(*)[2])kPow5);
      lens[k] = (unsigned)f[k].len + 1;
      if (col == cols - 1) nl |= 1u << k;
    }
    col = col + 1 == cols ? 0 : col + 1;
    len += lens[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = len;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  unsigned woff = 0, total = 0;
  for (int w = 0; w < kFmtThreads / 32; w++) {
    if (w < warp) woff += ws[w];
    total += ws[w];
  }
  if (warp == 0) {
    // warp-parallel look-back: lane l inspects block j - l of a 32-block
    // window; the window is consumed up to its nearest inclusive prefix once
    // every status up to it is published
    volatile unsigned long long* vs = status;
    if (lane == 0) {
      __threadfence();
      vs[bid] = (bid == 0 ? kFlagIncl : kFlagAgg) | total;
    }
    unsigned long long prefix = 0;
    long long j = (long long)bid - 1;
    while (j >= 0) {
      const long long jj = j - lane;
      const unsigned long long st = jj >= 0 ? vs[jj] : (2ULL << 62);  // before block 0: an empty inclusive prefix
      const unsigned ready = __ballot_sync(0xffffffffu, (st & ~kValMask) != 0);
      const unsigned incl = __ballot_sync(0xffffffffu, (st & kFlagIncl) != 0);
      const int first_incl = incl ? __ffs(incl) - 1 : 32;  // nearest inclusive in the window
      const unsigned need = first_incl >= 31 ? 0xffffffffu : ((2u << first_incl) - 1u);
      if ((ready & need) != need) continue;  // a predecessor in range has not published yet
      unsigned long long add = (lane <= first_incl && jj >= 0) ? (st & kValMask) : 0;
      for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
      prefix += add;
      if (first_incl < 32) break;
      j -= 32;
    }
    if (lane == 0) {
      if (bid != 0) {
        __threadfence();
        vs[bid] = kFlagIncl | (prefix + total);
      }
      s_off = prefix;
      if (bid == (unsigned long long)nblocks - 1) *nbytes = prefix + total;
    }
  }
  __syncthreads();
  unsigned off = woff + x - len;
#pragma unroll
  for (int k = 0; k < kFmtPer; k++) {
    if (lens[k]) {
      nc::nc_emit(f[k], reinterpret_cast<char*>(stage) + off);  // straight into shared memory
      stage[off + lens[k] - 1] = (nl >> k) & 1u ? '\n' : ' ';
      off += lens[k];
    }
  }
  __syncthreads();
  unsigned char* dst = out + s_off;
  for (unsigned k = threadIdx.x; k < total; k += kFmtThreads) dst[k] = stage[k];
}

int64_t ntiles_of(int64_t n) { return (n + kTokTile - 1) / kTokTile; }

}  // namespace

extern "C" {

size_t wg_ascii_tokenize_scratch_bytes(int64_t n) { return 256 + (size_t)(ntiles_of(n) + 1) * 8; }

int wg_ascii_tokenize(const uint8_t* text, int64_t n, int64_t body_off, int64_t* starts, int64_t cap,
                      uint64_t* count_flags, void* scratch, void* stream) {
  if (n < 0 || body_off < 0 || body_off > n || cap < 0) return wg::set_error(WG_EARG, "bad text range");
  if (!count_flags || !scratch || (n > 0 && !text) || (cap > 0 && !starts)) return wg::set_error(WG_EARG, "null buffer");
  cudaStream_t st = wg::as_stream(stream);
  // count_flags[0] = number of tokens, count_flags[1] = 1 if a byte >= 0x80
  WG_CUDA_TRY(cudaMemsetAsync(count_flags, 0, 2 * sizeof(uint64_t), st));
  if (n == body_off) return WG_OK;
  const int64_t first_tile = body_off / kTokTile;
  const int64_t tiles = ntiles_of(n) - first_tile;
  unsigned long long* tile = reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(scratch) + 256);
  // tiles are indexed from the body's first tile: shift the text base
  const unsigned char* t0 = text + first_tile * kTokTile;
  const int64_t lo = body_off - first_tile * kTokTile, len = n - first_tile * kTokTile;
  if (tiles > 0x7fffffff) return wg::set_error(WG_ELIMIT, "text too large");
  tok_count_kernel<<<(unsigned)tiles, kTokThreads, 0, st>>>(t0, lo, len, tile,
                                                            reinterpret_cast<unsigned*>(count_flags + 1));
  WG_LAUNCH_CHECK("tok_count_kernel");
  scan_kernel<<<1, 1024, 0, st>>>(tile, tiles, reinterpret_cast<unsigned long long*>(count_flags));
  WG_LAUNCH_CHECK("scan_kernel");
  if (cap > 0) {
    tok_scatter_kernel<<<(unsigned)tiles, kTokThreads, 0, st>>>(t0, lo, len, tile, starts, cap,
                                                                first_tile * kTokTile);
    WG_LAUNCH_CHECK("tok_scatter_kernel");
  }
  return WG_OK;
}

int wg_ascii_parse(const uint8_t* text, int64_t n, const int64_t* starts, int64_t count, double* out,
                   uint64_t* first_bad, void* stream) {
  if (n < 0 || count < 0) return wg::set_error(WG_EARG, "bad text range");
  if (!first_bad || (count > 0 && (!text || !starts || !out))) return wg::set_error(WG_EARG, "null buffer");
  cudaStream_t st = wg::as_stream(stream);
  WG_CUDA_TRY(cudaMemsetAsync(first_bad, 0xff, sizeof(uint64_t), st));
  if (count == 0) return WG_OK;
  parse_kernel<<<wg::stream_grid(count, 256, 8), 256, 0, st>>>(text, n, starts, count, out,
                                                               reinterpret_cast<unsigned long long*>(first_bad));
  WG_LAUNCH_CHECK("parse_kernel");
  return WG_OK;
}

size_t wg_ascii_format_scratch_bytes(int64_t count) {
  return 256 + (size_t)((count + kFmtThreads - 1) / kFmtThreads + 1) * 8;
}

int64_t wg_ascii_format_capacity(int64_t count) { return count < 0 ? -1 : count * kFmtMax; }

int wg_ascii_format(const double* values, int64_t count, int64_t cols, uint8_t* out, int64_t cap, uint64_t* nbytes,
                    void* scratch, void* stream) {
  if (count < 0 || cols < 1 || !scratch || !nbytes || (count > 0 && (!values || !out)))
    return wg::set_error(WG_EARG, "bad args");
  if (cap < count * kFmtMax) return wg::set_error(WG_EARG, "capacity %lld < %lld", (long long)cap,
                                                  (long long)(count * kFmtMax));
  cudaStream_t st = wg::as_stream(stream);
  if (count == 0) {
    WG_CUDA_TRY(cudaMemsetAsync(nbytes, 0, sizeof(uint64_t), st));
    return WG_OK;
  }
  const int64_t blocks = (count + kFmtThreads * kFmtPer - 1) / (kFmtThreads * kFmtPer);
  if (blocks > 0x7fffffff) return wg::set_error(WG_ELIMIT, "too many values");
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(scratch);
  unsigned long long* status = counter + 32;  // 256-byte offset
  WG_CUDA_TRY(cudaMemsetAsync(scratch, 0, 256 + (size_t)blocks * 8, st));
  fmt_kernel<<<(unsigned)blocks, kFmtThreads, 0, st>>>(values, count, cols, out, status, counter,
                                                     reinterpret_cast<unsigned long long*>(nbytes), blocks);
  WG_LAUNCH_CHECK("fmt_kernel");
  return WG_OK;
}

}  // extern "C"

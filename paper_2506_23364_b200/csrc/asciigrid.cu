// ESRI ASCII grid reader/writer on the device:
// /root/reference/pkg/src/demflow/asciigrid.py -- parse_ascii_grid (42-143)
// tokenises the body with str.split() and converts every token with
// np.array(tokens, dtype=float64); write_ascii_grid (146-157) joins
// format_number(v) (160-167) with single spaces, one raster row per line.
//
// Reader: two passes (tok_kernel, parse_kernel): token starts by SWAR
// whitespace classification (str.split()'s ASCII whitespace is \t \n \v
// \f \r \x1c-\x1f and space) scattered to their global index found by a
// decoupled look-back over 4 KiB tiles, then the conversion (wg_numconv.cuh:
// CPython float() semantics, correctly rounded) of every token, one thread
// each, straight into its slot.
// Writer: one fused pass (fmt_kernel): four values per thread sized and
// formatted once (format_number: int digits or shortest round-trip repr,
// Ryu), block byte offsets by the same look-back, bytes staged in shared
// memory and streamed out.
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

constexpr unsigned long long kFlagAgg = 1ULL << 62, kFlagIncl = 2ULL << 62, kValMask = (1ULL << 62) - 1;

// lane 0: publish block bid's own total (block 0: its inclusive prefix)
__device__ __forceinline__ void publish_aggregate(unsigned long long* status, unsigned long long bid,
                                                  unsigned long long total) {
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    reinterpret_cast<volatile unsigned long long*>(status)[bid] = (bid == 0 ? kFlagIncl : kFlagAgg) | total;
  }
}

// one warp: the sum of the totals of blocks 0 .. bid-1, then publishes block
// bid's inclusive prefix.  Warp-parallel look-back: lane l inspects block
// j - l of a 32-block window; the window is consumed up to its nearest
// inclusive prefix once every status up to it is published.
__device__ __forceinline__ unsigned long long resolve_prefix(unsigned long long* status, unsigned long long bid,
                                                             unsigned long long total) {
  const int lane = threadIdx.x & 31;
  volatile unsigned long long* vs = status;
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
  if (lane == 0 && bid != 0) {
    __threadfence();
    vs[bid] = kFlagIncl | (prefix + total);
  }
  return prefix;
}

// Reader, pass 1 (tok_kernel): one block per 64 KiB of the body, block
// ids in execution order (so the look-back only waits on running or finished
// blocks): SWAR token-start bits of 16 bytes per thread, a block scan, the
// tile's count published for the look-back, and the absolute offsets of the
// tile's tokens scattered to starts[] at their global index.  Pass 2
// (parse_kernel): one thread per token (parse_fast, else nc_parse), values
// straight into out[].  info[0] = tokens in the body, info[1] = 1 if a body
// byte is >= 0x80, info[2] = offset of token #expected (the first extra
// token) if any, info[3] = offset of the first token < expected that float()
// rejects (UINT64_MAX if none); pass 2 runs only when info[0] == expected.
// kTokSub sub-tiles of 4 KiB per block: the look-back runs once per 64 KiB
// (one look-back per 4 KiB serialises on the chain of published prefixes)
#ifndef WG_TOK_SUB
#define WG_TOK_SUB 16
#endif
constexpr int kTokSub = WG_TOK_SUB;

__device__ __forceinline__ unsigned block_scan(unsigned c, unsigned* ws, unsigned& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // ws reuse across calls
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  unsigned woff = 0;
  total = 0;
  for (int w = 0; w < kTokThreads / 32; w++) {
    if (w < warp) woff += ws[w];
    total += ws[w];
  }
  return woff + x - c;  // exclusive
}

__global__ void __launch_bounds__(kTokThreads) tok_kernel(const unsigned char* __restrict__ t, int64_t lo, int64_t n,
                                                          int64_t base, int64_t* __restrict__ starts,
                                                          int64_t expected, unsigned long long* __restrict__ status,
                                                          unsigned long long* __restrict__ counter,
                                                          unsigned long long* __restrict__ info, int64_t nblocks) {
  __shared__ unsigned ws[kTokThreads / 32];
  __shared__ unsigned long long s_bid, s_off;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_bid = atomicAdd(counter, 1ULL);
  __syncthreads();
  const unsigned long long bid = s_bid;
  const int64_t b0 = (int64_t)bid * kTokTile * kTokSub + (int64_t)threadIdx.x * kTokBytes;
  // pass A: the block's token count
  unsigned nonascii = 0, c = 0;
  for (int k = 0; k < kTokSub; k++) c += __popc(start_bits(t, b0 + k * kTokTile, lo, n, nonascii));
  if (__any_sync(0xffffffffu, nonascii) && lane == 0) atomicOr(info + 1, 1ULL);
  unsigned total;
  block_scan(c, ws, total);
  if (warp == 0) {
    publish_aggregate(status, bid, total);
    const unsigned long long prefix = resolve_prefix(status, bid, total);
    if (lane == 0) {
      s_off = prefix;
      if (bid == (unsigned long long)nblocks - 1) info[0] = prefix + total;
    }
  }
  __syncthreads();
  // pass B: sub-tile by sub-tile (document order), scatter the offsets
  // (the bits are recomputed from the L2-resident tile: keeping all 16 in
  // registers measured slower, 111 registers)
  int64_t run = (int64_t)s_off;
  for (int k = 0; k < kTokSub; k++) {
    const int64_t p0 = b0 + k * kTokTile;
    unsigned dummy = 0;
    unsigned bits = start_bits(t, p0, lo, n, dummy);
    unsigned sub;
    int64_t idx = run + block_scan(__popc(bits), ws, sub);
    run += sub;
    while (bits) {
      const int q = __ffs(bits) - 1;
      bits &= bits - 1;
      if (idx < expected) starts[idx] = base + p0 + q;
      else if (idx == expected) info[2] = (unsigned long long)(base + p0 + q);
      idx++;
    }
  }
}

__global__ void parse_kernel(const unsigned char* __restrict__ t, int64_t n, const int64_t* __restrict__ starts,
                             int64_t count, double* __restrict__ out, unsigned long long* __restrict__ info) {
  if ((int64_t)info[0] != count) return;  // the host reports the count mismatch
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = starts[i];
    double v = 0.0;
    int64_t len;
    if (!parse_fast(t, s, n, &v, &len)) {
      int64_t e = s;
      while (e < n && !is_ws(__ldg(t + e))) e++;
      len = e - s;
      const int rc = len > 0x7fffffff ? -1 : nc::nc_parse(t + s, (int)len, &v, (const uint64_t(*)[2])kEL);
      if (rc != 0) atomicMin(info + 3, (unsigned long long)s);
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

#ifndef WG_FMT_MINB
#define WG_FMT_MINB 4  // 64 registers, 4 blocks/SM (A/B: 13.6 -> 12.5 ms at 16384^2)
#endif
__global__ void __launch_bounds__(kFmtThreads, WG_FMT_MINB) fmt_kernel(const double* __restrict__ v, int64_t count, int64_t cols,
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
    publish_aggregate(status, bid, total);
    const unsigned long long prefix = resolve_prefix(status, bid, total);
    if (lane == 0) {
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

size_t wg_ascii_read_scratch_bytes(int64_t n, int64_t expected) {
  return 256 + (size_t)(ntiles_of(n) + 1) * 8 + (size_t)(expected > 0 ? expected : 0) * 8;
}

int wg_ascii_read(const uint8_t* text, int64_t n, int64_t body_off, double* out, int64_t expected, uint64_t* info,
                  void* scratch, void* stream) {
  if (n < 0 || body_off < 0 || body_off > n || expected < 0) return wg::set_error(WG_EARG, "bad text range");
  if (!info || !scratch || (n > 0 && !text) || (expected > 0 && !out)) return wg::set_error(WG_EARG, "null buffer");
  cudaStream_t st = wg::as_stream(stream);
  WG_CUDA_TRY(cudaMemsetAsync(info, 0, 2 * sizeof(uint64_t), st));
  WG_CUDA_TRY(cudaMemsetAsync(info + 2, 0xff, 2 * sizeof(uint64_t), st));
  if (n == body_off) return WG_OK;
  // tiles are counted from the body's first tile: shift the text base
  const int64_t first_tile = body_off / kTokTile;
  const int64_t tiles = ntiles_of(n) - first_tile;
  const int64_t blocks = (tiles + kTokSub - 1) / kTokSub;
  if (blocks > 0x7fffffff) return wg::set_error(WG_ELIMIT, "text too large");
  const unsigned char* t0 = text + first_tile * kTokTile;
  const int64_t lo = body_off - first_tile * kTokTile, len = n - first_tile * kTokTile;
  // scratch: [claim counter (256 B)] [tile status x tiles] [token starts x expected]
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(scratch);
  unsigned long long* status = counter + 32;
  int64_t* starts = reinterpret_cast<int64_t*>(status + ntiles_of(n) + 1);
  WG_CUDA_TRY(cudaMemsetAsync(scratch, 0, 256 + (size_t)blocks * 8, st));
  tok_kernel<<<(unsigned)blocks, kTokThreads, 0, st>>>(t0, lo, len, first_tile * kTokTile, starts, expected, status,
                                                       counter, reinterpret_cast<unsigned long long*>(info), blocks);
  WG_LAUNCH_CHECK("tok_kernel");
  if (expected > 0) {
    parse_kernel<<<wg::resident_grid(parse_kernel, expected, 256), 256, 0, st>>>(text, n, starts, expected, out,
                                                                    reinterpret_cast<unsigned long long*>(info));
    WG_LAUNCH_CHECK("parse_kernel");
  }
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

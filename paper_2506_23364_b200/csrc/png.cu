// Tile serving on the device: extract_tile + encode_png
// (/root/reference/pkg/src/demflow/overlay.py:221-260; service.py:351-360).
//
// One CTA per tile reads its tile_px x tile_px window of a pyramid level
// (texels outside the level are transparent black, overlay.py:247-251) and
// writes a complete PNG file: signature, IHDR (8-bit RGBA, non-interlaced),
// one IDAT holding a zlib stream, IEND.  The reference encodes with Pillow
// (zlib deflate); its byte stream is not pinned, so parity is the decoded
// image (decode_png(encode_png(t)) == t) and the stream's own checksums.
//
// Encoding: per scanline, warp-parallel, the PNG filter (None/Sub/Up/Avg/
// Paeth) with the least sum of |signed residual| (libpng's heuristic); the
// residual bytes are deflated as ONE fixed-Huffman block whose matches are
// byte runs (distance 1) -- transparent and flat areas become runs of zeros
// under Sub/Up.  Each lane tokenises its 32-byte slice; pass A sums bits per
// row, a block scan places the rows, pass B writes every token's bits with
// 32-bit atomic ORs into the zeroed stream.  Adler-32 of the filtered data
// comes from per-lane position-weighted sums; CRC-32 of the IDAT chunk from
// per-lane CRCs joined with crc32_combine's GF(2) shift (zlib's method).
#include "wg_internal.cuh"

namespace {

constexpr int kPngThreads = 256;  // 8 warps per tile
constexpr int kPrefix = 8 + 25 + 8;  // signature + IHDR chunk + IDAT length/type
constexpr uint32_t kCrcPoly = 0xEDB88320u;

__device__ __forceinline__ int sabs(unsigned v) { return v < 128 ? (int)v : 256 - (int)v; }

__device__ __forceinline__ unsigned paeth(unsigned a, unsigned b, unsigned c) {
  const int p = (int)a + (int)b - (int)c;
  const int pa = abs(p - (int)a), pb = abs(p - (int)b), pc = abs(p - (int)c);
  if (pa <= pb && pa <= pc) return a;
  if (pb <= pc) return b;
  return c;
}

__device__ __forceinline__ unsigned filt(int type, unsigned x, unsigned a, unsigned b, unsigned c) {
  switch (type) {
    case 0: return x;
    case 1: return (x - a) & 255u;
    case 2: return (x - b) & 255u;
    case 3: return (x - ((a + b) >> 1)) & 255u;
    default: return (x - paeth(a, b, c)) & 255u;
  }
}

__device__ __forceinline__ uint32_t rev(uint32_t v, int n) { return __brev(v) >> (32 - n); }

// fixed-Huffman literal: (bits reversed for LSB-first packing, length)
__device__ __forceinline__ void lit_code(unsigned lit, uint32_t& code, int& len) {
  if (lit < 144) {
    code = rev(0x30 + lit, 8);
    len = 8;
  } else {
    code = rev(0x190 + (lit - 144), 9);
    len = 9;
  }
}

// length L (3..258) + distance 1: length code with extra bits, then the
// 5-bit distance code 0
__device__ __forceinline__ void match_code(unsigned L, uint32_t& code, int& len) {
  unsigned sym, extra = 0, ebits = 0;
  if (L == 258) {
    sym = 285;
  } else if (L <= 10) {
    sym = 254 + L;
  } else {
    // codes 265..284: 4 codes per extra-bit count, base lengths 11,13,..
    const unsigned l = L - 3;  // 8..254
    const int eb = 31 - __clz(l) - 2;  // extra bits (1..5)
    const unsigned grp = (l >> eb) - 4;  // 0..3 within the group
    sym = 265 + (eb - 1) * 4 + grp;
    extra = l & ((1u << eb) - 1);
    ebits = eb;
  }
  uint32_t c;
  int n;
  if (sym < 280) {
    c = rev(sym - 256, 7);
    n = 7;
  } else {
    c = rev(0xC0 + (sym - 280), 8);
    n = 8;
  }
  code = c | (extra << n);  // extra bits follow, LSB first
  len = n + (int)ebits + 5;  // + distance code 0 (five zero bits)
}

// Bit sink: count (kWrite false) or OR into the zeroed stream at bit offset.
template <bool kWrite>
struct Bits {
  uint32_t* words;
  uint64_t pos;
  __device__ __forceinline__ void put(uint32_t code, int len) {
    if (kWrite) {
      const uint64_t w = pos >> 5;
      const int s = (int)(pos & 31);
      const uint64_t v = (uint64_t)code << s;
      atomicOr(words + w, (uint32_t)v);
      if (s + len > 32) atomicOr(words + w + 1, (uint32_t)(v >> 32));
    }
    pos += (uint64_t)len;
  }
};

// Tokenise one lane's residual bytes (runs -> distance-1 matches).
template <bool kWrite>
__device__ void emit_bytes(Bits<kWrite>& out, const uint32_t* f, int nbytes, unsigned prev, bool has_prev) {
  int i = 0;
  while (i < nbytes) {
    const unsigned b = (f[i >> 2] >> (8 * (i & 3))) & 255u;
    int j = i + 1;
    while (j < nbytes && ((f[j >> 2] >> (8 * (j & 3))) & 255u) == b) j++;
    int avail = j - i;
    uint32_t code;
    int len;
    if (!(has_prev && prev == b)) {
      lit_code(b, code, len);
      out.put(code, len);
      avail -= 1;
    }
    while (avail >= 3) {
      const int L = avail > 258 ? 258 : avail;
      match_code((unsigned)L, code, len);
      out.put(code, len);
      avail -= L;
    }
    for (; avail > 0; avail--) {
      lit_code(b, code, len);
      out.put(code, len);
    }
    prev = b;
    has_prev = true;
    i = j;
  }
}

// One PNG image: W x H texels read from a level at (x0, y0); texels outside
// the level are transparent black (the tile canvas, overlay.py:247-251).
struct Img {
  const uint8_t* level;
  int64_t lw, lh;  // level size in texels
  int64_t x0, y0;  // image origin in the level
  int W, H;        // image size
};

__device__ __forceinline__ uint32_t texel(const Img& g, int r, int c) {
  const int64_t y = g.y0 + r, x = g.x0 + c;
  if (r < 0 || c < 0 || c >= g.W || y >= g.lh || x >= g.lw) return 0u;
  return __ldg(reinterpret_cast<const uint32_t*>(g.level) + (y * g.lw + x));
}

// A row is processed in chunks of 256 texels: lane l holds texels
// [256 k + 8 l, +8) of chunk k.
constexpr int kLanePx = 8;
constexpr int kChunkPx = 32 * kLanePx;

// libpng's heuristic over the whole row: the filter with the least sum of
// |signed residual| (ties -> the lower type), warp-uniform.
__device__ int choose_filter(const Img& g, int r) {
  const int lane = threadIdx.x & 31;
  int sum[5] = {0, 0, 0, 0, 0};
  for (int c0 = lane * kLanePx; c0 < g.W; c0 += kChunkPx) {
    uint32_t left = texel(g, r, c0 - 1), upleft = texel(g, r - 1, c0 - 1);
#pragma unroll
    for (int k = 0; k < kLanePx; k++) {
      const uint32_t x = texel(g, r, c0 + k), up = texel(g, r - 1, c0 + k);
      if (c0 + k < g.W) {
#pragma unroll
        for (int byte = 0; byte < 4; byte++) {
          const unsigned xb = (x >> (8 * byte)) & 255u, a = (left >> (8 * byte)) & 255u,
                         b = (up >> (8 * byte)) & 255u, c = (upleft >> (8 * byte)) & 255u;
#pragma unroll
          for (int t = 0; t < 5; t++) sum[t] += sabs(filt(t, xb, a, b, c));
        }
      }
      left = x;
      upleft = up;
    }
  }
  int best = 0, bsum = 0x7fffffff;
#pragma unroll
  for (int t = 0; t < 5; t++) {
    int v = sum[t];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (v < bsum) {
      bsum = v;
      best = t;
    }
  }
  return best;
}

// This lane's residual texels of chunk starting at texel c0 (its 8 texels);
// returns how many are inside the row.
__device__ __forceinline__ int residuals(const Img& g, int r, int c0, int ftype, uint32_t* f) {
  uint32_t left = texel(g, r, c0 - 1), upleft = texel(g, r - 1, c0 - 1);
#pragma unroll
  for (int k = 0; k < kLanePx; k++) {
    const uint32_t x = texel(g, r, c0 + k), up = texel(g, r - 1, c0 + k);
    uint32_t w = 0;
#pragma unroll
    for (int byte = 0; byte < 4; byte++) {
      const unsigned xb = (x >> (8 * byte)) & 255u, a = (left >> (8 * byte)) & 255u, b = (up >> (8 * byte)) & 255u,
                     c = (upleft >> (8 * byte)) & 255u;
      w |= filt(ftype, xb, a, b, c) << (8 * byte);
    }
    f[k] = w;
    left = x;
    upleft = up;
  }
  const int n = g.W - c0;
  return n < 0 ? 0 : (n > kLanePx ? kLanePx : n);
}

// Visit row r: the filter byte then every chunk's lane slices, chaining the
// previous byte across lanes and chunks.  kWrite false: returns the row's
// bits (lane 0 holds them) and accumulates the Adler sums; kWrite true:
// writes the bits starting at row_bit.
template <bool kWrite>
__device__ uint64_t visit_row(const Img& g, int r, uint32_t* words, uint64_t row_bit, unsigned long long& sumA,
                              unsigned long long& sumW) {
  const int lane = threadIdx.x & 31;
  const int ftype = choose_filter(g, r);
  uint32_t code;
  int len;
  lit_code((unsigned)ftype, code, len);
  if (kWrite && lane == 0) {
    Bits<true> o{words, row_bit};
    o.put(code, len);
  }
  const int64_t row_base = (int64_t)r * (4 * (int64_t)g.W + 1);
  if (!kWrite && lane == 0) {
    sumA += (unsigned)ftype;
    sumW += (unsigned long long)row_base * (unsigned)ftype;
  }
  uint64_t bits = (uint64_t)len;  // warp-uniform running total
  unsigned carry = (unsigned)ftype;  // byte before the chunk
  for (int cbase = 0; cbase < g.W; cbase += kChunkPx) {
    const int c0 = cbase + lane * kLanePx;
    uint32_t f[kLanePx];
    const int n = residuals(g, r, c0, ftype, f);
    const unsigned last = (f[(n > 0 ? n : 1) - 1] >> 24) & 255u;
    unsigned prev = __shfl_up_sync(0xffffffffu, last, 1);
    if (lane == 0) prev = carry;
    Bits<false> cnt{nullptr, 0};
    if (n > 0) emit_bytes(cnt, f, 4 * n, prev, true);
    uint64_t x = cnt.pos;  // inclusive scan of lane bits
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (kWrite && n > 0) {
      Bits<true> o{words, row_bit + bits + x - cnt.pos};
      emit_bytes(o, f, 4 * n, prev, true);
    }
    if (!kWrite) {
      for (int k = 0; k < 4 * n; k++) {
        const unsigned b = (f[k >> 2] >> (8 * (k & 3))) & 255u;
        sumA += b;
        sumW += (unsigned long long)(row_base + 1 + 4 * (int64_t)c0 + k) * b;
      }
    }
    bits += __shfl_sync(0xffffffffu, x, 31);
    const int m = min(32, (g.W - cbase + kLanePx - 1) / kLanePx);  // lanes with texels
    carry = __shfl_sync(0xffffffffu, last, m - 1);
  }
  return bits;
}

__device__ uint32_t crc_table_entry(uint32_t n) {
  uint32_t c = n;
  for (int k = 0; k < 8; k++) c = (c & 1) ? kCrcPoly ^ (c >> 1) : c >> 1;
  return c;
}

__device__ uint32_t multmodp(uint32_t a, uint32_t b) {  // a * b mod P (reflected)
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}

__device__ uint32_t x8nmodp(uint64_t n) {  // x^(8n) mod P
  uint32_t xp = 1u << 30;  // x^1
  // x^(2^k) by squaring; start at x^8 = x^(2^3)
  for (int k = 0; k < 3; k++) xp = multmodp(xp, xp);
  uint32_t p = 1u << 31;  // x^0
  while (n) {
    if (n & 1) p = multmodp(xp, p);
    n >>= 1;
    xp = multmodp(xp, xp);
  }
  return p;
}

__device__ __forceinline__ void put_be32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)(v >> 24);
  p[1] = (uint8_t)(v >> 16);
  p[2] = (uint8_t)(v >> 8);
  p[3] = (uint8_t)v;
}

// CRC-32 of bytes [0, n) of p (standard: init ~0, final xor), one warp.
__device__ uint32_t warp_crc32(const uint8_t* p, int64_t n, const uint32_t* table) {
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (n + 31) / 32;
  const int64_t lo = lane * chunk < n ? lane * chunk : n, hi = lo + chunk < n ? lo + chunk : n;
  uint32_t c = 0xFFFFFFFFu;
  for (int64_t i = lo; i < hi; i++) c = table[(c ^ __ldcg(p + i)) & 255u] ^ (c >> 8);
  c ^= 0xFFFFFFFFu;
  uint32_t crc = __shfl_sync(0xffffffffu, c, 0);
  // gather the lane CRCs through shared memory and join them in order
  // (crc32_combine: crc(A||B) = crc(A) * x^(8|B|) mod P ^ crc(B))
  __shared__ uint32_t s_crc[32];
  __shared__ int64_t s_len[32];
  s_crc[lane] = c;
  s_len[lane] = hi - lo;
  __syncwarp();
  if (lane == 0) {
    for (int l = 1; l < 32; l++)
      if (s_len[l] > 0) crc = multmodp(x8nmodp((uint64_t)s_len[l]), crc) ^ s_crc[l];
  }
  return __shfl_sync(0xffffffffu, crc, 0);
}

// One CTA per image.  txy: image origins in tile units of T (tiles), or
// null for one W x H image at (0, 0) (encode_png of a whole texture).
__global__ void __launch_bounds__(kPngThreads) png_kernel(const uint8_t* __restrict__ level, int64_t lw, int64_t lh,
                                                          int W, int H, const int32_t* __restrict__ txy,
                                                          uint8_t* __restrict__ out, int64_t cap,
                                                          int64_t* __restrict__ lens) {
  extern __shared__ uint64_t s_rows[];  // H row bit counts, then offsets
  __shared__ uint32_t s_table[256];
  __shared__ unsigned long long s_adA, s_adB;
  __shared__ uint64_t s_total;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = kPngThreads / 32;
  Img g{level, lw, lh, txy ? (int64_t)txy[2 * blockIdx.x] * W : 0, txy ? (int64_t)txy[2 * blockIdx.x + 1] * H : 0,
        W, H};
  uint8_t* img = out + (int64_t)blockIdx.x * cap;
  const int64_t nbytes = (4 * (int64_t)W + 1) * H;  // filtered data (zlib payload)
  for (int i = threadIdx.x; i < 256; i += kPngThreads) s_table[i] = crc_table_entry((uint32_t)i);
  if (threadIdx.x == 0) s_adA = s_adB = 0;
  __syncthreads();
  // ---- pass A: bits per row, Adler sums
  unsigned long long sumA = 0, sumW = 0;
  for (int r = warp; r < H; r += nw) {
    const uint64_t bits = visit_row<false>(g, r, nullptr, 0, sumA, sumW);
    if (lane == 0) s_rows[r] = bits;
  }
  for (int o = 16; o > 0; o >>= 1) {
    sumA += __shfl_xor_sync(0xffffffffu, sumA, o);
    sumW += __shfl_xor_sync(0xffffffffu, sumW, o);
  }
  if (lane == 0) {
    atomicAdd(&s_adA, sumA);
    atomicAdd(&s_adB, sumW);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan of the row bits
    uint64_t acc = 3;  // BFINAL + BTYPE
    for (int r = 0; r < H; r++) {
      const uint64_t b = s_rows[r];
      s_rows[r] = acc;
      acc += b;
    }
    s_total = acc + 7;  // + end-of-block code (seven zero bits)
  }
  __syncthreads();
  const int64_t dbytes = (int64_t)((s_total + 7) / 8);
  const int64_t zlen = 2 + dbytes + 4;
  const int64_t file_len = kPrefix + zlen + 4 + 12;
  if (file_len > cap) {  // cannot happen for cap = wg_png_capacity(W, H)
    if (threadIdx.x == 0) lens[blockIdx.x] = -1;
    return;
  }
  // zero the words the deflate bits go to, then the fixed prefix
  uint32_t* words = reinterpret_cast<uint32_t*>(img);
  const int64_t w_lo = (kPrefix + 2) / 4, w_hi = (kPrefix + 2 + dbytes + 3) / 4;
  for (int64_t w = w_lo + threadIdx.x; w < w_hi; w += kPngThreads) words[w] = 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint8_t sig[8] = {0x89, 'P', 'N', 'G', 0x0D, 0x0A, 0x1A, 0x0A};
    for (int i = 0; i < 8; i++) img[i] = sig[i];
    put_be32(img + 8, 13);
    img[12] = 'I', img[13] = 'H', img[14] = 'D', img[15] = 'R';
    put_be32(img + 16, (uint32_t)W);
    put_be32(img + 20, (uint32_t)H);
    img[24] = 8, img[25] = 6, img[26] = 0, img[27] = 0, img[28] = 0;  // 8-bit RGBA, deflate, adaptive, no interlace
    uint32_t c = 0xFFFFFFFFu;
    for (int i = 12; i < 29; i++) c = s_table[(c ^ img[i]) & 255u] ^ (c >> 8);
    put_be32(img + 29, c ^ 0xFFFFFFFFu);
    put_be32(img + 33, (uint32_t)zlen);
    img[37] = 'I', img[38] = 'D', img[39] = 'A', img[40] = 'T';
    img[41] = 0x78, img[42] = 0x01;  // zlib: deflate, 32 KiB window, no dictionary
  }
  __threadfence();
  __syncthreads();
  // ---- pass B: write the bits
  const uint64_t bit0 = (uint64_t)(kPrefix + 2) * 8;
  if (threadIdx.x == 0) {
    Bits<true> o{words, bit0};
    o.put(0x3u, 3);  // BFINAL = 1, BTYPE = 01 (fixed Huffman)
  }
  for (int r = warp; r < H; r += nw) visit_row<true>(g, r, words, bit0 + s_rows[r], sumA, sumW);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {  // Adler-32 of the filtered data
    const unsigned long long N = (unsigned long long)nbytes;
    const uint32_t A = (uint32_t)((1 + s_adA) % 65521ULL);
    // B = sum over k of (1 + bytes before k) = N + sum_i (N - i) d_i
    const uint32_t B = (uint32_t)((N + N * s_adA - s_adB) % 65521ULL);
    put_be32(img + kPrefix + 2 + dbytes, (B << 16) | A);
  }
  __threadfence();
  __syncthreads();
  if (warp == 0) {
    const uint32_t crc = warp_crc32(img + 37, 4 + zlen, s_table);
    if (lane == 0) {
      uint8_t* e = img + kPrefix + zlen;
      put_be32(e, crc);
      put_be32(e + 4, 0);
      e[8] = 'I', e[9] = 'E', e[10] = 'N', e[11] = 'D';
      put_be32(e + 12, 0xAE426082u);
      lens[blockIdx.x] = file_len;
    }
  }
}

int launch_png(const uint8_t* level, int64_t lw, int64_t lh, int64_t W, int64_t H, const int32_t* txy, int64_t n,
               uint8_t* out, int64_t cap, int64_t* lens, cudaStream_t st) {
  const size_t smem = (size_t)H * sizeof(uint64_t);
  static bool attr = false;
  if (!attr) {
    WG_CUDA_TRY(cudaFuncSetAttribute(png_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  png_kernel<<<(unsigned)n, kPngThreads, smem, st>>>(level, lw, lh, (int)W, (int)H, txy, out, cap, lens);
  WG_LAUNCH_CHECK("png_kernel");
  return WG_OK;
}

}  // namespace

extern "C" {

int64_t wg_png_capacity(int64_t width, int64_t height) {
  if (width < 1 || height < 1 || width > 0x7fffffff || height > 25000) return -1;
  const int64_t raw = (4 * width + 1) * height;
  const int64_t deflate = (raw * 9 + 3 + 7 + 7) / 8 + 8;  // <= 9 bits per byte
  return ((kPrefix + 2 + deflate + 4 + 4 + 12) + 255) / 256 * 256;
}

int wg_png_tiles(const uint8_t* level, int64_t width, int64_t height, int64_t tile_px, const int32_t* txy,
                 int64_t ntiles, uint8_t* out, int64_t cap, int64_t* lens, void* stream) {
  if (ntiles <= 0) return WG_OK;
  const int64_t need = wg_png_capacity(tile_px, tile_px);
  if (need < 0) return wg::set_error(WG_EARG, "bad tile_px %lld", (long long)tile_px);
  if (cap < need || cap % 4) return wg::set_error(WG_EARG, "per-tile capacity %lld < %lld", (long long)cap, (long long)need);
  if (!level || !txy || !out || !lens || width < 1 || height < 1) return wg::set_error(WG_EARG, "bad arguments");
  if ((((uintptr_t)level) & 3) || (((uintptr_t)out) & 3)) return wg::set_error(WG_EARG, "buffers must be 4-byte aligned");
  if (ntiles > 0x7fffffff) return wg::set_error(WG_ELIMIT, "too many tiles");
  return launch_png(level, width, height, tile_px, tile_px, txy, ntiles, out, cap, lens, wg::as_stream(stream));
}

int wg_png_encode(const uint8_t* pixels, int64_t width, int64_t height, uint8_t* out, int64_t cap, int64_t* len,
                  void* stream) {
  const int64_t need = wg_png_capacity(width, height);
  if (need < 0) return wg::set_error(WG_EARG, "bad image size %lldx%lld", (long long)width, (long long)height);
  if (cap < need || cap % 4) return wg::set_error(WG_EARG, "capacity %lld < %lld", (long long)cap, (long long)need);
  if (!pixels || !out || !len) return wg::set_error(WG_EARG, "null buffer");
  if ((((uintptr_t)pixels) & 3) || (((uintptr_t)out) & 3)) return wg::set_error(WG_EARG, "buffers must be 4-byte aligned");
  return launch_png(pixels, width, height, width, height, nullptr, 1, out, cap, len, wg::as_stream(stream));
}

}  // extern "C"

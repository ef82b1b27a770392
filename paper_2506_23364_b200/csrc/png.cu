// Tile serving on the device: extract_tile + encode_png
// (/root/reference/pkg/src/demflow/overlay.py:221-260; service.py:351-360).
//
// Each image (a tile_px x tile_px tile of a pyramid level -- texels outside
// the level are transparent black, overlay.py:247-251 -- or a whole texture)
// becomes a complete PNG file: signature, IHDR (8-bit RGBA, non-interlaced),
// one IDAT holding a zlib stream, IEND.  The reference encodes with Pillow
// (zlib deflate); its byte stream is not pinned, so parity is the decoded
// image (decode_png(encode_png(t)) == t) and the stream's own checksums.
//
// Three kernels over a batch of images:
//   filter_kernel  one CTA per image, warp per row: the PNG filter (None/Sub/
//                  Up/Avg/Paeth) with the least sum of |signed residual|
//                  (libpng's heuristic); writes the filtered stream (filter
//                  byte + residuals per row) and its Adler-32;
//   lz_kernel      one warp per ~32 KiB chunk of rows: LZ77 parse with a
//                  32-position lookahead (lane k checks position i + k; the
//                  first match ends the step), then the whole warp measures
//                  every candidate of that position -- the kRing most recent
//                  positions with the same 3-byte hash (per-chunk ring
//                  buckets in global memory, every consumed position
//                  inserted warp-parallel, deterministically) and the
//                  image-shaped distances 1, 4, row, 2 rows, row +- 4 -- and
//                  of the next one (one-step lazy evaluation); the longest
//                  wins (ties: the nearer); matches may reach back 32 KiB
//                  into earlier chunks.  Tokens go to a per-chunk array;
//   emit_kernel    one CTA per image: symbol histograms, dynamic Huffman
//                  codes (Moffat-Katajainen lengths limited to 15 bits,
//                  canonical codes, run-length coded code lengths; one
//                  thread), the tokens' bit lengths, a block scan, 32-bit
//                  atomic ORs into the zeroed stream, then zlib/Adler, the
//                  IDAT CRC-32 (per-lane CRCs joined by crc32_combine's GF(2)
//                  shift) and IEND.
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

// Per-image scratch layout (wg_png_scratch_bytes).
struct Layout {
  int64_t nbytes;    // filtered stream bytes: (4W + 1) * H
  int rows_per_chunk, nchunks;
  int64_t f_off, tok_off, tab_off, meta_off, per_image;
};

// LZ77 knobs (A/B on the 1365-tile bench, hillshade / overlay ms and mean
// KB): see DESIGN.md section 6 (tile PNG row).
#ifndef WG_PNG_HBITS
#define WG_PNG_HBITS 11
#endif
#ifndef WG_PNG_LAZY
#define WG_PNG_LAZY 1
#endif
#ifndef WG_PNG_LAZY_MAX
#define WG_PNG_LAZY_MAX 8  // lazy evaluation only after matches shorter than this (zlib's max_lazy)
#endif
#ifndef WG_PNG_RING
#define WG_PNG_RING 16
#endif
#ifndef WG_PNG_QUICK
#define WG_PNG_QUICK 4
#endif
constexpr int kHashBits = WG_PNG_HBITS;
constexpr int kBuckets = 1 << kHashBits;  // per chunk
// each bucket: a ring of the kRing most recent positions with that 3-byte
// hash (+1; 0 = empty) and its head (next slot to write)
constexpr int kRing = WG_PNG_RING;
constexpr int kQuick = WG_PNG_QUICK;  // most recent ring entries tried by the lookahead
constexpr int kImageCands = 6;
constexpr int kCands = kRing + kImageCands;
static_assert(kCands <= 32 && kQuick <= kRing, "one candidate per lane");
constexpr bool kLazy = WG_PNG_LAZY != 0;
constexpr int64_t kTabWords = ((int64_t)kBuckets * (kRing + 1) + 3) / 4 * 4;  // per chunk
constexpr int kWindow = 32768;

__host__ __device__ inline Layout layout_of(int64_t W, int64_t H) {
  Layout l;
  l.nbytes = (4 * W + 1) * H;
  const int64_t row = 4 * W + 1;
  l.rows_per_chunk = (int)(row >= kWindow ? 1 : kWindow / row);
  l.nchunks = (int)((H + l.rows_per_chunk - 1) / l.rows_per_chunk);
  auto up = [](int64_t v) { return (v + 255) / 256 * 256; };
  l.f_off = 0;
  l.tok_off = up(l.nbytes + 8);  // + slack for 4-byte compares
  l.tab_off = l.tok_off + up(l.nbytes * 4);
  l.meta_off = l.tab_off + up((int64_t)l.nchunks * kTabWords * 4);
  l.per_image = l.meta_off + up(8 + (int64_t)l.nchunks * 4);  // adler (u32) + pad + token counts
  return l;
}

struct Batch {
  const uint8_t* level;
  int64_t lw, lh;
  int W, H;
  const int32_t* txy;  // tile coords (units of W/H) or null
  uint8_t* scratch;
  Layout lay;
  uint8_t* out;
  int64_t cap;
  int64_t* lens;
};

__device__ __forceinline__ Img img_of(const Batch& b, int i) {
  return Img{b.level, b.lw, b.lh, b.txy ? (int64_t)b.txy[2 * i] * b.W : 0, b.txy ? (int64_t)b.txy[2 * i + 1] * b.H : 0,
             b.W, b.H};
}

// ---- kernel 1: filtered stream + Adler-32 ----------------------------------
__global__ void __launch_bounds__(kPngThreads) filter_kernel(Batch b) {
  __shared__ unsigned long long s_a, s_w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Img g = img_of(b, blockIdx.x);
  uint8_t* base = b.scratch + (int64_t)blockIdx.x * b.lay.per_image;
  uint8_t* F = base + b.lay.f_off;
  if (threadIdx.x == 0) s_a = s_w = 0;
  __syncthreads();
  unsigned long long sumA = 0, sumW = 0;
  const int64_t row = 4 * (int64_t)g.W + 1;
  for (int r = warp; r < g.H; r += kPngThreads / 32) {
    const int ftype = choose_filter(g, r);
    const int64_t rb = (int64_t)r * row;
    if (lane == 0) {
      F[rb] = (uint8_t)ftype;
      sumA += (unsigned)ftype;
      sumW += (unsigned long long)rb * (unsigned)ftype;
    }
    for (int cbase = 0; cbase < g.W; cbase += kChunkPx) {
      const int c0 = cbase + lane * kLanePx;
      uint32_t f[kLanePx];
      const int n = residuals(g, r, c0, ftype, f);
      for (int k = 0; k < 4 * n; k++) {
        const unsigned v = (f[k >> 2] >> (8 * (k & 3))) & 255u;
        const int64_t pos = rb + 1 + 4 * (int64_t)c0 + k;
        F[pos] = (uint8_t)v;
        sumA += v;
        sumW += (unsigned long long)pos * v;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    sumA += __shfl_xor_sync(0xffffffffu, sumA, o);
    sumW += __shfl_xor_sync(0xffffffffu, sumW, o);
  }
  if (lane == 0) {
    atomicAdd(&s_a, sumA);
    atomicAdd(&s_w, sumW);
  }
  // zero the chunks' bucket tables (positions are stored + 1; 0 = empty)
  uint4* tab = reinterpret_cast<uint4*>(base + b.lay.tab_off);
  const int64_t nt = (int64_t)b.lay.nchunks * kTabWords / 4;
  for (int64_t i = threadIdx.x; i < nt; i += kPngThreads) tab[i] = make_uint4(0, 0, 0, 0);
  for (int k = 0; k < 8; k++)
    if (threadIdx.x == k) F[b.lay.nbytes + k] = 0;  // compare slack
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long N = (unsigned long long)b.lay.nbytes;
    const uint32_t A = (uint32_t)((1 + s_a) % 65521ULL);
    const uint32_t B = (uint32_t)((N + N * s_a - s_w) % 65521ULL);  // N + sum_i (N - i) d_i
    *reinterpret_cast<uint32_t*>(base + b.lay.meta_off) = (B << 16) | A;
  }
}

// ---- kernel 2: LZ77 parse, one warp per chunk ------------------------------
__device__ __forceinline__ uint32_t hash3(const uint8_t* F, int64_t p) {
  const uint32_t v = (uint32_t)F[p] | ((uint32_t)F[p + 1] << 8) | ((uint32_t)F[p + 2] << 16);
  return (v * 2654435761u) >> (32 - kHashBits);
}

// 4 bytes of F starting at byte x (little endian; F is 4-byte aligned and
// padded, so the word after the last is readable)
__device__ __forceinline__ uint32_t load4(const uint8_t* F, int64_t x) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(F) + (x >> 2);
  return __funnelshift_r(__ldg(w), __ldg(w + 1), (unsigned)(x & 3) * 8);
}

// length of the common prefix of F[q..] and F[p..], capped at maxl
__device__ __forceinline__ int match_len(const uint8_t* F, int64_t q, int64_t p, int maxl) {
  int len = 0;
  while (len < maxl) {
    const uint32_t x = load4(F, q + len) ^ load4(F, p + len);
    if (x) {
      len += (__ffs(x) - 1) >> 3;
      break;
    }
    len += 4;
  }
  return len < maxl ? len : maxl;
}

// image-shaped candidate k for position p: distances 1, 4, row, 2 rows,
// row +- 4
__device__ __forceinline__ int64_t image_cand(int64_t p, int k, int64_t S) {
  switch (k) {
    case 0: return p - 1;
    case 1: return p - 4;
    case 2: return p - S;
    case 3: return p - 2 * S;
    case 4: return p - S - 4;
    default: return p - S + 4;
  }
}


__device__ __forceinline__ bool valid_cand(int64_t q, int64_t p) { return q >= 0 && q < p && p - q <= kWindow; }

// The longest match at position pp over all candidates, one per lane: lanes
// 0..kRing-1 the bucket's ring entries, the next kImageCands the image
// distances.  Returns (length << 16) | (32767 - (distance - 1)) of the best
// (ties: the nearer), 0 if none reaches 3 bytes; the same in every lane.
__device__ __forceinline__ unsigned best_match(const uint8_t* F, int64_t pp, int64_t end, int64_t S,
                                               const uint32_t* ring, int64_t nbytes, int lane) {
  const int maxl = (int)(end - pp < 258 ? end - pp : 258);
  unsigned key = 0;
  if (maxl >= 3) {
    int64_t q = -1;
    if (lane < kRing) {
      if (pp + 2 < nbytes) q = (int64_t)ring[(int64_t)hash3(F, pp) * kRing + lane] - 1;
    } else if (lane < kCands) {
      q = image_cand(pp, lane - kRing, S);
    }
    if (valid_cand(q, pp)) {
      const int len = match_len(F, q, pp, maxl);
      if (len >= 3) key = ((unsigned)len << 16) | (unsigned)(32767 - (pp - q - 1));
    }
  }
  for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
  return key;
}

// LZ77 over one chunk with a 32-position lookahead.  Phase 1: lane k checks
// whether the kQuick most recent same-hash positions or the image distances
// of position i + k share its first 3 bytes; the first such lane f ends the
// step (the lanes before it are literals), so incompressible stretches
// advance 32 bytes per step.  Phase 2: the whole warp measures every
// candidate of i + f (all kRing ring entries + image distances) and, lazily,
// of i + f + 1; a strictly longer match one byte later makes i + f a literal
// (zlib's deflate_slow rule).  Every consumed position is then inserted into
// its bucket's ring (same-bucket lanes take consecutive slots in position
// order; deterministic).
__global__ void __launch_bounds__(256) lz_kernel(Batch b, int64_t nwork) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wid >= nwork) return;
  const int lane = threadIdx.x & 31;
  const int img = (int)(wid / b.lay.nchunks), ch = (int)(wid % b.lay.nchunks);
  uint8_t* base = b.scratch + (int64_t)img * b.lay.per_image;
  const uint8_t* F = base + b.lay.f_off;
  uint32_t* tok = reinterpret_cast<uint32_t*>(base + b.lay.tok_off);
  uint32_t* ring = reinterpret_cast<uint32_t*>(base + b.lay.tab_off) + (int64_t)ch * kTabWords;
  uint32_t* heads = ring + (int64_t)kBuckets * kRing;
  uint32_t* counts = reinterpret_cast<uint32_t*>(base + b.lay.meta_off + 8);
  const int64_t S = 4 * (int64_t)b.W + 1;
  const int64_t start = (int64_t)ch * b.lay.rows_per_chunk * S;
  int64_t end = start + (int64_t)b.lay.rows_per_chunk * S;
  if (end > b.lay.nbytes) end = b.lay.nbytes;
  const int64_t nbytes = b.lay.nbytes;
  int64_t ntok = 0;
  uint32_t* out = tok + start;  // this chunk's tokens (at most one per byte)
  int64_t i = start;
  while (i < end) {
    const int64_t p = i + lane;
    bool quick = false;
    if (p + 3 <= end) {
      const uint32_t head = load4(F, p) & 0xFFFFFFu;
      if (p + 2 < nbytes) {
        const uint32_t hb = hash3(F, p);
        const uint32_t h0 = heads[hb];
        for (int k = 1; k <= kQuick && !quick; k++) {
          const int64_t q = (int64_t)ring[(int64_t)hb * kRing + (h0 + kRing - k) % kRing] - 1;
          quick = valid_cand(q, p) && (load4(F, q) & 0xFFFFFFu) == head;
        }
      }
      for (int k = 0; k < kImageCands && !quick; k++) {
        const int64_t q = image_cand(p, k, S);
        quick = valid_cand(q, p) && (load4(F, q) & 0xFFFFFFu) == head;
      }
    }
    const unsigned hit = __ballot_sync(0xffffffffu, quick);
    const int nvalid = (int)min((int64_t)32, end - i);
    const int f = hit ? __ffs(hit) - 1 : nvalid;  // literals before the first match
    if (lane < f) out[ntok + lane] = F[p];
    int64_t adv = f;
    if (hit) {
      const int64_t pf = i + f;
      const unsigned k0 = best_match(F, pf, end, S, ring, nbytes, lane);
      const unsigned k1 =
          (kLazy && (k0 >> 16) < WG_PNG_LAZY_MAX) ? best_match(F, pf + 1, end, S, ring, nbytes, lane) : 0u;
      const bool later = (k1 >> 16) > (k0 >> 16);
      const unsigned kw = later ? k1 : k0;
      const int mlen = (int)(kw >> 16);
      const uint32_t dm1 = 32767u - (kw & 0xFFFFu);  // distance - 1
      if (mlen >= 3) {
        if (later) {
          if (lane == 0) {
            out[ntok + f] = F[pf];
            out[ntok + f + 1] = ((uint32_t)mlen << 16) | dm1;
          }
          ntok += f + 2;
          adv += 1 + mlen;
        } else {
          if (lane == 0) out[ntok + f] = ((uint32_t)mlen << 16) | dm1;
          ntok += f + 1;
          adv += mlen;
        }
      } else {  // the 3-byte hit was at the chunk end: a literal
        if (lane == 0) out[ntok + f] = F[pf];
        ntok += f + 1;
        adv += 1;
      }
    } else {
      ntok += f;
    }
    // insert every consumed position: lanes of one bucket take consecutive
    // ring slots in position order (only the last kRing of a group land)
    for (int64_t b0 = 0; b0 < adv; b0 += 32) {
      const int64_t pi = i + b0 + lane;
      const int nins = adv - b0 < 32 ? (int)(adv - b0) : 32;
      const bool ins = lane < nins && pi + 2 < nbytes;
      const uint32_t hb = ins ? hash3(F, pi) : 0xFFFFFFFFu - lane;
      const unsigned grp = __match_any_sync(0xffffffffu, hb);
      const int leader = __ffs(grp) - 1;
      const int g = __popc(grp), r = __popc(grp & ((1u << lane) - 1u));
      uint32_t h0 = 0;
      if (ins && lane == leader) h0 = heads[hb];
      h0 = __shfl_sync(0xffffffffu, h0, leader);
      if (ins && g - r <= kRing) ring[(int64_t)hb * kRing + (h0 + r) % kRing] = (uint32_t)(pi + 1);
      if (ins && lane == leader) heads[hb] = (h0 + g) % kRing;
      __syncwarp();
    }
    i += adv;
  }
  if (lane == 0) counts[ch] = (uint32_t)ntok;
}

// ---- dynamic Huffman codes (RFC 1951 3.2.7), built by one thread ----------
// Moffat-Katajainen in-place minimum-redundancy lengths: A[0..n) ascending
// frequencies in, code lengths out.
__device__ void min_redundancy(int* A, int n) {
  if (n == 0) return;
  if (n == 1) {
    A[0] = 1;
    return;
  }
  A[0] += A[1];
  int root = 0, leaf = 2, next;
  for (next = 1; next < n - 1; next++) {
    if (leaf >= n || A[root] < A[leaf]) {
      A[next] = A[root];
      A[root++] = next;
    } else {
      A[next] = A[leaf++];
    }
    if (leaf >= n || (root < next && A[root] < A[leaf])) {
      A[next] += A[root];
      A[root++] = next;
    } else {
      A[next] += A[leaf++];
    }
  }
  A[n - 2] = 0;
  for (next = n - 3; next >= 0; next--) A[next] = A[A[next]] + 1;
  int avbl = 1, used = 0, dpth = 0;
  root = n - 2;
  next = n - 1;
  while (avbl > 0) {
    while (root >= 0 && A[root] == dpth) {
      used++;
      root--;
    }
    while (avbl > used) {
      A[next--] = dpth;
      avbl--;
    }
    avbl = 2 * used;
    dpth++;
    used = 0;
  }
}

// Code lengths (<= limit) for freq[0..n); `complete`: the code must be
// complete (lit/len, code-length code); otherwise a single used symbol gets
// length 1 (the distance code's allowed incomplete case).  Scratch: sym, a
// (n ints each).
__device__ void build_lengths(const uint32_t* freq, int n, int limit, bool complete, uint8_t* len, int* sym, int* a) {
  int m = 0;
  for (int i = 0; i < n; i++) {
    len[i] = 0;
    if (freq[i]) sym[m++] = i;
  }
  if (m == 0) return;
  if (m == 1) {
    len[sym[0]] = 1;
    if (complete) len[sym[0] == 0 ? 1 : 0] = 1;  // a dummy second code keeps it complete
    return;
  }
  for (int i = 1; i < m; i++) {  // insertion sort by (freq, symbol) ascending
    const int s = sym[i];
    int j = i - 1;
    while (j >= 0 && (freq[sym[j]] > freq[s] || (freq[sym[j]] == freq[s] && sym[j] > s))) {
      sym[j + 1] = sym[j];
      j--;
    }
    sym[j + 1] = s;
  }
  for (int i = 0; i < m; i++) a[i] = (int)freq[sym[i]];
  min_redundancy(a, m);
  int num[33] = {0};
  for (int i = 0; i < m; i++) num[a[i] > 32 ? 32 : a[i]]++;
  // enforce the limit (miniz's method on the per-length counts)
  for (int i = limit + 1; i <= 32; i++) {
    num[limit] += num[i];
    num[i] = 0;
  }
  uint32_t total = 0;
  for (int i = limit; i > 0; i--) total += (uint32_t)num[i] << (limit - i);
  while (total != (1u << limit)) {
    num[limit]--;
    for (int i = limit - 1; i > 0; i--)
      if (num[i]) {
        num[i]--;
        num[i + 1] += 2;
        break;
      }
    total--;
  }
  // most frequent symbols get the shortest lengths
  int j = m;
  for (int l = 1; l <= limit; l++)
    for (int c = num[l]; c > 0; c--) len[sym[--j]] = (uint8_t)l;
}

// canonical codes (RFC 1951 3.2.2), bit-reversed for LSB-first packing
__device__ void canonical(const uint8_t* len, int n, uint16_t* code) {
  int count[16] = {0};
  for (int i = 0; i < n; i++) count[len[i]]++;
  count[0] = 0;
  int next[16];
  int c = 0;
  for (int bits = 1; bits < 16; bits++) {
    c = (c + count[bits - 1]) << 1;
    next[bits] = c;
  }
  for (int i = 0; i < n; i++)
    if (len[i]) code[i] = (uint16_t)rev((uint32_t)next[len[i]]++, len[i]);
}

__device__ __forceinline__ unsigned len_sym(unsigned L, unsigned& extra, int& ebits) {
  extra = 0;
  ebits = 0;
  if (L == 258) return 285;
  if (L <= 10) return 254 + L;
  const unsigned l = L - 3;
  const int eb = 31 - __clz(l) - 2;
  extra = l & ((1u << eb) - 1);
  ebits = eb;
  return 265 + (eb - 1) * 4 + ((l >> eb) - 4);
}

__device__ __forceinline__ unsigned dist_sym(unsigned d, unsigned& extra, int& ebits) {
  extra = 0;
  ebits = 0;
  if (d <= 4) return d - 1;
  const unsigned l = d - 1;
  const int eb = 31 - __clz(l) - 1;
  extra = l & ((1u << eb) - 1);
  ebits = eb;
  return 2 * (eb + 1) + ((l >> eb) & 1);
}

struct Codes {
  uint16_t lit[286];
  uint8_t litlen[286];
  uint16_t dist[30];
  uint8_t distlen[30];
};

__device__ __forceinline__ int dyn_bits(const Codes& c, uint32_t t) {
  if (t < 256) return c.litlen[t];
  unsigned e;
  int eb, db;
  const unsigned ls = len_sym(t >> 16, e, eb);
  const unsigned ds = dist_sym((t & 0xFFFF) + 1, e, db);
  return c.litlen[ls] + eb + c.distlen[ds] + db;
}

template <bool kWrite>
__device__ __forceinline__ void dyn_put(Bits<kWrite>& o, const Codes& c, uint32_t t) {
  if (t < 256) {
    o.put(c.lit[t], c.litlen[t]);
    return;
  }
  unsigned e;
  int eb;
  const unsigned ls = len_sym(t >> 16, e, eb);
  o.put(c.lit[ls] | (e << c.litlen[ls]), c.litlen[ls] + eb);
  const unsigned ds = dist_sym((t & 0xFFFF) + 1, e, eb);
  o.put(c.dist[ds] | (e << c.distlen[ds]), c.distlen[ds] + eb);
}

__device__ const uint8_t kClOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// The dynamic block: codes built once from the histograms (one thread),
// then the header written or counted from the stored description.
struct DynHeader {
  Codes c;
  uint8_t seq_sym[320], seq_ext[320];
  int ns, hlit, hdist, hclen;
  uint8_t cll[19];
  uint16_t clc[19];
};

__device__ void dyn_build(DynHeader& h, const uint32_t* lf, const uint32_t* df, int* s1, int* s2) {
  Codes& c = h.c;
  build_lengths(lf, 286, 15, true, c.litlen, s1, s2);
  build_lengths(df, 30, 15, false, c.distlen, s1, s2);
  canonical(c.litlen, 286, c.lit);
  canonical(c.distlen, 30, c.dist);
  int hlit = 286;
  while (hlit > 257 && c.litlen[hlit - 1] == 0) hlit--;
  int hdist = 30;
  while (hdist > 1 && c.distlen[hdist - 1] == 0) hdist--;
  // run-length code the lengths (code-length alphabet 0..18)
  uint8_t all[316];
  for (int i = 0; i < hlit; i++) all[i] = c.litlen[i];
  for (int i = 0; i < hdist; i++) all[hlit + i] = c.distlen[i];
  const int n = hlit + hdist;
  int ns = 0;
  uint32_t clf[19] = {0};
  for (int i = 0; i < n;) {
    const uint8_t v = all[i];
    int run = 1;
    while (i + run < n && all[i + run] == v) run++;
    int r = run;
    if (v == 0) {
      while (r >= 11) {
        const int k = r < 138 ? r : 138;
        h.seq_sym[ns] = 18, h.seq_ext[ns++] = (uint8_t)(k - 11), clf[18]++;
        r -= k;
      }
      if (r >= 3) {
        h.seq_sym[ns] = 17, h.seq_ext[ns++] = (uint8_t)(r - 3), clf[17]++;
        r = 0;
      }
      for (; r > 0; r--) h.seq_sym[ns] = 0, h.seq_ext[ns++] = 0, clf[0]++;
    } else {
      h.seq_sym[ns] = v, h.seq_ext[ns++] = 0, clf[v]++;
      r--;
      while (r >= 3) {
        const int k = r < 6 ? r : 6;
        h.seq_sym[ns] = 16, h.seq_ext[ns++] = (uint8_t)(k - 3), clf[16]++;
        r -= k;
      }
      for (; r > 0; r--) h.seq_sym[ns] = v, h.seq_ext[ns++] = 0, clf[v]++;
    }
    i += run;
  }
  build_lengths(clf, 19, 7, true, h.cll, s1, s2);
  canonical(h.cll, 19, h.clc);
  int hclen = 19;
  while (hclen > 4 && h.cll[kClOrder[hclen - 1]] == 0) hclen--;
  h.ns = ns;
  h.hlit = hlit;
  h.hdist = hdist;
  h.hclen = hclen;
}

template <bool kWrite>
__device__ uint64_t dyn_header(Bits<kWrite>& o, const DynHeader& h) {
  const uint64_t p0 = o.pos;
  o.put(0x5u, 3);  // BFINAL = 1, BTYPE = 10 (dynamic)
  o.put((uint32_t)(h.hlit - 257), 5);
  o.put((uint32_t)(h.hdist - 1), 5);
  o.put((uint32_t)(h.hclen - 4), 4);
  for (int i = 0; i < h.hclen; i++) o.put(h.cll[kClOrder[i]], 3);
  for (int i = 0; i < h.ns; i++) {
    const int sy = h.seq_sym[i];
    o.put(h.clc[sy], h.cll[sy]);
    if (sy == 16) o.put(h.seq_ext[i], 2);
    if (sy == 17) o.put(h.seq_ext[i], 3);
    if (sy == 18) o.put(h.seq_ext[i], 7);
  }
  return o.pos - p0;
}

// ---- kernel 3: codes, bits, zlib, checksums, chunks -----------------------
__global__ void __launch_bounds__(kPngThreads) emit_kernel(Batch b) {
  __shared__ uint32_t s_table[256];
  __shared__ unsigned long long s_scan[kPngThreads];
  __shared__ uint32_t s_lf[286], s_df[30];
  __shared__ DynHeader s_dyn;
  __shared__ int s_tmp1[288], s_tmp2[288];
  __shared__ uint64_t s_hdr_bits;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* base = b.scratch + (int64_t)blockIdx.x * b.lay.per_image;
  const uint32_t* tok = reinterpret_cast<const uint32_t*>(base + b.lay.tok_off);
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(base + b.lay.meta_off + 8);
  uint8_t* img = b.out + (int64_t)blockIdx.x * b.cap;
  const int64_t S = 4 * (int64_t)b.W + 1;
  const int nch = b.lay.nchunks;
  for (int i = threadIdx.x; i < 256; i += kPngThreads) s_table[i] = crc_table_entry((uint32_t)i);
  for (int i = threadIdx.x; i < 286; i += kPngThreads) s_lf[i] = 0;
  if (threadIdx.x < 30) s_df[threadIdx.x] = 0;
  __syncthreads();
  // histograms
  for (int c = 0; c < nch; c++) {
    const uint32_t* t = tok + (int64_t)c * b.lay.rows_per_chunk * S;
    const int64_t n = counts[c];
    for (int64_t k = threadIdx.x; k < n; k += kPngThreads) {
      const uint32_t v = t[k];
      if (v < 256) {
        atomicAdd(&s_lf[v], 1u);
      } else {
        unsigned e;
        int eb;
        atomicAdd(&s_lf[len_sym(v >> 16, e, eb)], 1u);
        atomicAdd(&s_df[dist_sym((v & 0xFFFF) + 1, e, eb)], 1u);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s_lf[256] = 1;  // end of block
    dyn_build(s_dyn, s_lf, s_df, s_tmp1, s_tmp2);
    Bits<false> cnt{nullptr, 0};
    s_hdr_bits = dyn_header(cnt, s_dyn);
  }
  __syncthreads();
  const Codes& cd = s_dyn.c;
  // pass 1: total bits
  unsigned long long mine = 0;
  for (int c = 0; c < nch; c++) {
    const uint32_t* t = tok + (int64_t)c * b.lay.rows_per_chunk * S;
    const int64_t n = counts[c];
    for (int64_t k = threadIdx.x; k < n; k += kPngThreads) mine += (unsigned long long)dyn_bits(cd, t[k]);
  }
  s_scan[threadIdx.x] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int k = 0; k < kPngThreads; k++) tot += s_scan[k];
    s_scan[0] = tot;
  }
  __syncthreads();
  const uint64_t total_bits = s_hdr_bits + s_scan[0] + cd.litlen[256];
  const int64_t dbytes = (int64_t)((total_bits + 7) / 8);
  const int64_t zlen = 2 + dbytes + 4;
  const int64_t file_len = kPrefix + zlen + 4 + 12;
  __syncthreads();
  if (file_len > b.cap) {  // dynamic codes lost to the worst-case bound: cannot happen in practice
    if (threadIdx.x == 0) b.lens[blockIdx.x] = -1;
    return;
  }
  uint32_t* words = reinterpret_cast<uint32_t*>(img);
  const int64_t w_lo = (kPrefix + 2) / 4, w_hi = (kPrefix + 2 + dbytes + 3) / 4;
  for (int64_t w = w_lo + threadIdx.x; w < w_hi; w += kPngThreads) words[w] = 0u;
  __syncthreads();
  const uint64_t bit_start = (uint64_t)(kPrefix + 2) * 8;
  if (threadIdx.x == 0) {
    const uint8_t sig[8] = {0x89, 'P', 'N', 'G', 0x0D, 0x0A, 0x1A, 0x0A};
    for (int i = 0; i < 8; i++) img[i] = sig[i];
    put_be32(img + 8, 13);
    img[12] = 'I', img[13] = 'H', img[14] = 'D', img[15] = 'R';
    put_be32(img + 16, (uint32_t)b.W);
    put_be32(img + 20, (uint32_t)b.H);
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
  if (threadIdx.x == 0) {
    Bits<true> o{words, bit_start};
    dyn_header(o, s_dyn);
    Bits<true> e{words, bit_start + total_bits - cd.litlen[256]};
    e.put(cd.lit[256], cd.litlen[256]);  // end of block
  }
  // pass 2: per chunk, block-scan the token bits and write them
  uint64_t bit = bit_start + s_hdr_bits;
  for (int c = 0; c < nch; c++) {
    const uint32_t* t = tok + (int64_t)c * b.lay.rows_per_chunk * S;
    const int64_t n = counts[c];
    const int64_t per = (n + kPngThreads - 1) / kPngThreads;
    const int64_t k0 = threadIdx.x * per < n ? threadIdx.x * per : n;
    const int64_t k1 = k0 + per < n ? k0 + per : n;
    unsigned long long m = 0;
    for (int64_t k = k0; k < k1; k++) m += (unsigned long long)dyn_bits(cd, t[k]);
    __syncthreads();
    s_scan[threadIdx.x] = m;
    __syncthreads();
    for (int o = 1; o < kPngThreads; o <<= 1) {
      const unsigned long long y = threadIdx.x >= (unsigned)o ? s_scan[threadIdx.x - o] : 0;
      __syncthreads();
      s_scan[threadIdx.x] += y;
      __syncthreads();
    }
    Bits<true> o{words, bit + s_scan[threadIdx.x] - m};
    for (int64_t k = k0; k < k1; k++) dyn_put(o, cd, t[k]);
    bit += s_scan[kPngThreads - 1];
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) put_be32(img + kPrefix + 2 + dbytes, *reinterpret_cast<const uint32_t*>(base + b.lay.meta_off));
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
      b.lens[blockIdx.x] = file_len;
    }
  }
}

int launch_png(Batch b, int64_t n, cudaStream_t st) {
  filter_kernel<<<(unsigned)n, kPngThreads, 0, st>>>(b);
  WG_LAUNCH_CHECK("filter_kernel");
  const int64_t nwork = n * b.lay.nchunks;
  lz_kernel<<<(unsigned)((nwork * 32 + 255) / 256), 256, 0, st>>>(b, nwork);
  WG_LAUNCH_CHECK("lz_kernel");
  emit_kernel<<<(unsigned)n, kPngThreads, 0, st>>>(b);
  WG_LAUNCH_CHECK("emit_kernel");
  return WG_OK;
}

}  // namespace

extern "C" {

int64_t wg_png_capacity(int64_t width, int64_t height) {
  if (width < 1 || height < 1 || width > 0x7fffffff || height > 0x7fffffff) return -1;
  const int64_t raw = (4 * width + 1) * height;
  // fixed Huffman needs <= 9 bits per byte (a match never costs more than
  // its literals); the dynamic code is optimal up to the length-limit
  // adjustment, plus its header: a 1/64 + 4 KiB margin
  const int64_t deflate = (raw * 9 + 3 + 7 + 7) / 8 + raw / 64 + 4096;
  return ((kPrefix + 2 + deflate + 4 + 4 + 12) + 255) / 256 * 256;
}

size_t wg_png_scratch_bytes(int64_t width, int64_t height, int64_t nimages) {
  if (width < 1 || height < 1 || nimages < 0) return 0;
  return (size_t)(layout_of(width, height).per_image * nimages);
}

int wg_png_tiles(const uint8_t* level, int64_t width, int64_t height, int64_t tile_px, const int32_t* txy,
                 int64_t ntiles, uint8_t* out, int64_t cap, int64_t* lens, void* scratch, void* stream) {
  if (ntiles <= 0) return WG_OK;
  const int64_t need = wg_png_capacity(tile_px, tile_px);
  if (need < 0 || tile_px > 65535) return wg::set_error(WG_EARG, "bad tile_px %lld", (long long)tile_px);
  if (cap < need || cap % 4) return wg::set_error(WG_EARG, "per-tile capacity %lld < %lld", (long long)cap, (long long)need);
  if (!level || !txy || !out || !lens || !scratch || width < 1 || height < 1) return wg::set_error(WG_EARG, "bad arguments");
  if ((((uintptr_t)level) & 3) || (((uintptr_t)out) & 3) || (((uintptr_t)scratch) & 255))
    return wg::set_error(WG_EARG, "misaligned buffer");
  if (ntiles > 0x7fffffff) return wg::set_error(WG_ELIMIT, "too many tiles");
  Batch b{level, width, height, (int)tile_px, (int)tile_px, txy, (uint8_t*)scratch, layout_of(tile_px, tile_px),
          out, cap, lens};
  if (b.lay.nchunks > 1024) return wg::set_error(WG_ELIMIT, "image too tall");
  return launch_png(b, ntiles, wg::as_stream(stream));
}

int wg_png_encode(const uint8_t* pixels, int64_t width, int64_t height, uint8_t* out, int64_t cap, int64_t* len,
                  void* scratch, void* stream) {
  const int64_t need = wg_png_capacity(width, height);
  if (need < 0 || width > 65535 || height > 65535)
    return wg::set_error(WG_EARG, "bad image size %lldx%lld", (long long)width, (long long)height);
  if (cap < need || cap % 4) return wg::set_error(WG_EARG, "capacity %lld < %lld", (long long)cap, (long long)need);
  if (!pixels || !out || !len || !scratch) return wg::set_error(WG_EARG, "null buffer");
  if ((((uintptr_t)pixels) & 3) || (((uintptr_t)out) & 3) || (((uintptr_t)scratch) & 255))
    return wg::set_error(WG_EARG, "misaligned buffer");
  Batch b{pixels, width, height, (int)width, (int)height, nullptr, (uint8_t*)scratch, layout_of(width, height), out,
          cap, len};
  return launch_png(b, 1, wg::as_stream(stream));
}

}  // extern "C"

// Raster-pass kernels of the terrain prefix and the release / snow nodes:
//   K1  fetch_tiles / stitch_tiles copies   (tiles.py:115-136, 153-218)
//   a5  DemGrid scan: nodata + finiteness     (grid.py:80-98, 129-130)
//   K2  surface_normals (+ fused steepness)   (terrain.py:69-102)
//   K3  steepness                             (terrain.py:99-102)
//   K4  release_points mask + ordinal list    (simulate.py:207-225, 465)
//   K9  snow alpha texture                    (simulate.py:520-560)
//   K6  runout invariants + stats             (simulate.py:159-190, 507-514)
//   synthetic DEM combine (bench/test input)
// All are HBM-streaming passes: grid-stride loops over
// sm_count x resident CTAs, IEEE f64 through _rn intrinsics where the
// reference's bits must be reproduced.
#include "wg_internal.cuh"
#include "wg_fp64.h"

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kBlock = 256;

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------- grid scan
__global__ void grid_scan_kernel(const double* __restrict__ e, int64_t n, double nodata,
                                 unsigned long long* counts) {
  unsigned long long nd = 0, bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = __ldg(e + i);
    if (v == nodata) nd++;
    else if (!isfinite(v)) bad++;
  }
  nd = warp_sum(nd);
  bad = warp_sum(bad);
  if ((threadIdx.x & 31) == 0) {
    if (nd) atomicAdd(counts, nd);
    if (bad) atomicAdd(counts + 1, bad);
  }
}

// ---------------------------------------------------------------- 2D copy
__global__ void copy2d_kernel(const double* __restrict__ src, int64_t src_ld, double* __restrict__ dst,
                              int64_t dst_ld, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / cols, c = t - r * cols;
    dst[r * dst_ld + c] = __ldg(src + r * src_ld + c);
  }
}

// ---------------------------------------------------------------- normals
// degrees(arccos(clip(nz, -1, 1))); np.degrees multiplies by 180/pi.
__device__ __forceinline__ double slope_of(double nz) {
  const double c = wg_min(wg_max(nz, -1.0), 1.0);
  return WG_MUL(acos(c), 57.29577951308232);
}

// One thread per cell; neighbours come through L1/L2 (each DEM row is read
// by three consecutive row passes of the grid-stride loop, which the 126 MB L2
// keeps resident), so HBM traffic stays at the 8 B in + 24 B (+8 B) out floor.
__global__ void normals_kernel(const double* __restrict__ e, int64_t nrows, int64_t ncols, double cs, double two_cs,
                               double* __restrict__ nrm, double* __restrict__ slope) {
  const int64_t total = nrows * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / ncols, j = t - i * ncols;
    const double* row = e + i * ncols;
    double dzdx, dzdy;
    if (j == 0) dzdx = WG_DIV(WG_SUB(__ldg(row + 1), __ldg(row)), cs);
    else if (j == ncols - 1) dzdx = WG_DIV(WG_SUB(__ldg(row + j), __ldg(row + j - 1)), cs);
    else dzdx = WG_DIV(WG_SUB(__ldg(row + j + 1), __ldg(row + j - 1)), two_cs);
    if (i == 0) dzdy = WG_DIV(WG_SUB(__ldg(e + j), __ldg(e + ncols + j)), cs);
    else if (i == nrows - 1) dzdy = WG_DIV(WG_SUB(__ldg(row - ncols + j), __ldg(row + j)), cs);
    else dzdy = WG_DIV(WG_SUB(__ldg(row - ncols + j), __ldg(row + ncols + j)), two_cs);
    const double nx = wg_neg(dzdx), ny = wg_neg(dzdy);
    const double len = WG_SQRT(WG_ADD(WG_ADD(WG_MUL(nx, nx), WG_MUL(ny, ny)), 1.0));
    const double nz = WG_DIV(1.0, len);
    double* o = nrm + 3 * t;
    o[0] = WG_DIV(nx, len);
    o[1] = WG_DIV(ny, len);
    o[2] = nz;
    if (slope != nullptr) slope[t] = slope_of(nz);
  }
}

__global__ void steepness_kernel(const double* __restrict__ nrm, int64_t n, double* __restrict__ slope) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    slope[t] = slope_of(__ldg(nrm + 3 * t + 2));
}

// ---------------------------------------------------------------- hillshade
// shade = clip(n0*lx + n1*ly + n2*lz, 0, 1); floor(shade*255 + 0.5) (terrain.py:297-299)
__global__ void hillshade_kernel(const double* __restrict__ nrm, int64_t n, double lx, double ly, double lz,
                                 uint8_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double* v = nrm + 3 * t;
    const double dot = WG_ADD(WG_ADD(WG_MUL(__ldg(v), lx), WG_MUL(__ldg(v + 1), ly)), WG_MUL(__ldg(v + 2), lz));
    const double sh = wg_min(wg_max(dot, 0.0), 1.0);
    out[t] = (uint8_t)(int)floor(WG_ADD(WG_MUL(sh, 255.0), 0.5));
  }
}

// ---------------------------------------------------------------- release mask
__global__ void release_mask_kernel(const double* __restrict__ s, int64_t nrows, int64_t ncols, double lo, double hi,
                                    int64_t stride, uint8_t* __restrict__ mask) {
  const int64_t total = nrows * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / ncols, j = t - i * ncols;
    const double v = __ldg(s + t);
    mask[t] = (uint8_t)((v >= lo) & (v <= hi) & (i % stride == 0) & (j % stride == 0));
  }
}

// ---------------------------------------------------------------- compaction
// Three passes (count per tile, scan of tile counts, scatter) produce the
// row-major list of set cells -- np.flatnonzero order, which fixes the
// release ordinal k of every cell (simulate.py:465-480).
constexpr int kTile = kBlock * 16;  // cells per tile: 16 per thread

__device__ __forceinline__ int block_exclusive_scan(int v, int* total, int* smem /*>= 32*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int w = lane < (blockDim.x >> 5) ? smem[lane] : 0;
    int winc = w;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(kFull, winc, o);
      if (lane >= o) winc += y;
    }
    smem[lane] = winc - w;
    if (lane == 31) smem[32] = winc;
  }
  __syncthreads();
  int r = smem[wid] + inc - v;
  *total = smem[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ int count16(const uint8_t* __restrict__ m, int64_t base, int64_t n) {
  int c = 0;
  if (base + 16 <= n && (((uintptr_t)(m + base)) & 15) == 0) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(m + base));
    c = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);  // mask bytes are 0/1
  } else {
    for (int q = 0; q < 16; q++)
      if (base + q < n) c += m[base + q] != 0;
  }
  return c;
}

__global__ void compact_count_kernel(const uint8_t* __restrict__ m, int64_t n, int* __restrict__ tile_counts) {
  __shared__ int smem[33];
  const int64_t base = (int64_t)blockIdx.x * kTile + threadIdx.x * 16;
  int c = base < n ? count16(m, base, n) : 0;
  int total;
  block_exclusive_scan(c, &total, smem);
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = total;
}

// single-CTA exclusive scan over the tile counts (one per 4096 cells)
__global__ void compact_scan_kernel(const int* __restrict__ tile_counts, int64_t ntiles, int64_t* __restrict__ offs,
                                    int64_t* __restrict__ count) {
  __shared__ int smem[33];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < ntiles; b += blockDim.x) {
    const int64_t t = b + threadIdx.x;
    const int v = t < ntiles ? tile_counts[t] : 0;
    int total;
    const int ex = block_exclusive_scan(v, &total, smem);
    if (t < ntiles) offs[t] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = carry;
}

__global__ void compact_scatter_kernel(const uint8_t* __restrict__ m, int64_t n, const int64_t* __restrict__ offs,
                                       int64_t* __restrict__ cells) {
  __shared__ int smem[33];
  const int64_t base = (int64_t)blockIdx.x * kTile + threadIdx.x * 16;
  uint8_t v[16];
  int c = 0;
  for (int q = 0; q < 16; q++) {
    v[q] = (base + q < n) ? m[base + q] : 0;
    c += v[q] != 0;
  }
  int total;
  int pos = block_exclusive_scan(c, &total, smem);
  int64_t o = offs[blockIdx.x] + pos;
  for (int q = 0; q < 16; q++)
    if (v[q]) cells[o++] = base + q;
}

// ---------------------------------------------------------------- snow
__global__ void snow_kernel(const double* __restrict__ z, const double* __restrict__ s, int64_t n, double base,
                            double alt_div, double top, double sl_div, int has_nodata, double nodata,
                            uchar4* __restrict__ px) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double zv = __ldg(z + t);
    const double a_alt = wg_min(wg_max(WG_DIV(WG_SUB(zv, base), alt_div), 0.0), 1.0);
    const double a_sl = wg_min(wg_max(WG_DIV(WG_SUB(top, __ldg(s + t)), sl_div), 0.0), 1.0);
    const double a = floor(WG_ADD(WG_MUL(255.0, WG_MUL(a_alt, a_sl)), 0.5));
    unsigned char alpha = (unsigned char)(int)a;
    if (has_nodata && zv == nodata) alpha = 0;
    px[t] = make_uchar4(255, 255, 255, alpha);
  }
}

// ---------------------------------------------------------------- runout stats
__global__ void runout_stats_kernel(const long long* __restrict__ hits, const double* __restrict__ z, int64_t n,
                                    unsigned long long* out) {
  unsigned long long sum = 0, nnz = 0, zmax = 0, bad = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const long long h = __ldg(hits + t);
    const double zv = __ldg(z + t);
    sum += (unsigned long long)h;
    nnz += h != 0;
    const bool ok = isfinite(zv) && zv >= 0.0 && h >= 0 && !(zv > 0.0 && h == 0);
    bad += !ok;
    const unsigned long long zb = wg_bits(zv);
    if (ok && zb > zmax) zmax = zb;
  }
  sum = warp_sum(sum);
  nnz = warp_sum(nnz);
  bad = warp_sum(bad);
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(kFull, zmax, o);
    zmax = y > zmax ? y : zmax;
  }
  if ((threadIdx.x & 31) == 0) {
    if (sum) atomicAdd(out, sum);
    if (nnz) atomicAdd(out + 1, nnz);
    if (zmax) atomicMax(out + 2, zmax);
    if (bad) atomicAdd(out + 3, bad);
  }
}

// ---------------------------------------------------------------- synthetic DEM
__global__ void synth_kernel(const double* __restrict__ rowf, const double* __restrict__ colf,
                             const double* __restrict__ lin, int noct, int64_t nrows, int64_t ncols,
                             double* __restrict__ e) {
  const int64_t total = nrows * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ncols, c = t - r * ncols;
    double z = __ldg(lin + c);
    for (int o = 0; o < noct; o++) z = WG_ADD(z, WG_MUL(__ldg(rowf + o * nrows + r), __ldg(colf + o * ncols + c)));
    e[t] = z;
  }
}

__global__ void sub_scalar_kernel(double* __restrict__ e, int64_t n, double v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    e[t] = WG_SUB(e[t], v);
}

}  // namespace

extern "C" {

int wg_grid_scan(const double* elev, int64_t n, double nodata, uint64_t* counts, void* stream) {
  if (n <= 0) return WG_OK;
  if (!elev || !counts) return wg::set_error(WG_EARG, "null buffer");
  grid_scan_kernel<<<wg::stream_grid(n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      elev, n, nodata, reinterpret_cast<unsigned long long*>(counts));
  WG_LAUNCH_CHECK("grid_scan_kernel");
  return WG_OK;
}

int wg_copy2d_f64(const double* src, int64_t src_ld, double* dst, int64_t dst_ld, int64_t rows, int64_t cols,
                  void* stream) {
  if (rows <= 0 || cols <= 0) return WG_OK;
  if (!src || !dst || src_ld < cols || dst_ld < cols) return wg::set_error(WG_EARG, "bad copy2d arguments");
  copy2d_kernel<<<wg::stream_grid(rows * cols, kBlock), kBlock, 0, wg::as_stream(stream)>>>(src, src_ld, dst, dst_ld,
                                                                                             rows, cols);
  WG_LAUNCH_CHECK("copy2d_kernel");
  return WG_OK;
}

int wg_normals(const double* elev, int64_t nrows, int64_t ncols, double cs, double two_cs, double* normals,
               double* slope, void* stream) {
  if (nrows < 2 || ncols < 2) return wg::set_error(WG_EARG, "grid must be at least 2x2");
  if (!elev || !normals) return wg::set_error(WG_EARG, "null buffer");
  normals_kernel<<<wg::stream_grid(nrows * ncols, kBlock), kBlock, 0, wg::as_stream(stream)>>>(elev, nrows, ncols, cs,
                                                                                                two_cs, normals, slope);
  WG_LAUNCH_CHECK("normals_kernel");
  return WG_OK;
}

int wg_steepness(const double* normals, int64_t n, double* slope, void* stream) {
  if (n <= 0) return WG_OK;
  if (!normals || !slope) return wg::set_error(WG_EARG, "null buffer");
  steepness_kernel<<<wg::stream_grid(n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(normals, n, slope);
  WG_LAUNCH_CHECK("steepness_kernel");
  return WG_OK;
}

int wg_hillshade(const double* normals, int64_t n, double lx, double ly, double lz, uint8_t* out, void* stream) {
  if (n <= 0) return WG_OK;
  if (!normals || !out) return wg::set_error(WG_EARG, "null buffer");
  hillshade_kernel<<<wg::stream_grid(n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(normals, n, lx, ly, lz, out);
  WG_LAUNCH_CHECK("hillshade_kernel");
  return WG_OK;
}

int wg_release_mask(const double* slope, int64_t nrows, int64_t ncols, double lo, double hi, int64_t stride,
                    uint8_t* mask, void* stream) {
  if (stride < 1) return wg::set_error(WG_EARG, "stride must be >= 1, got %lld", (long long)stride);
  if (nrows * ncols <= 0) return WG_OK;
  if (!slope || !mask) return wg::set_error(WG_EARG, "null buffer");
  release_mask_kernel<<<wg::stream_grid(nrows * ncols, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      slope, nrows, ncols, lo, hi, stride, mask);
  WG_LAUNCH_CHECK("release_mask_kernel");
  return WG_OK;
}

size_t wg_compact_scratch_bytes(int64_t n) {
  const int64_t ntiles = (n + kTile - 1) / kTile;
  return (size_t)ntiles * (sizeof(int) + sizeof(int64_t)) + 256;
}

int wg_mask_compact(const uint8_t* mask, int64_t n, int64_t* cells, int64_t* count, void* scratch, void* stream) {
  cudaStream_t st = wg::as_stream(stream);
  if (!count) return wg::set_error(WG_EARG, "null count");
  if (n <= 0) {
    WG_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return WG_OK;
  }
  if (!mask || !cells || !scratch) return wg::set_error(WG_EARG, "null buffer");
  const int64_t ntiles = (n + kTile - 1) / kTile;
  if (ntiles > 0x7fffffff) return wg::set_error(WG_EARG, "mask too large");
  int64_t* offs = reinterpret_cast<int64_t*>(scratch);
  int* tile_counts = reinterpret_cast<int*>(offs + ntiles);
  compact_count_kernel<<<(unsigned)ntiles, kBlock, 0, st>>>(mask, n, tile_counts);
  WG_LAUNCH_CHECK("compact_count_kernel");
  compact_scan_kernel<<<1, 1024, 0, st>>>(tile_counts, ntiles, offs, count);
  WG_LAUNCH_CHECK("compact_scan_kernel");
  compact_scatter_kernel<<<(unsigned)ntiles, kBlock, 0, st>>>(mask, n, offs, cells);
  WG_LAUNCH_CHECK("compact_scatter_kernel");
  return WG_OK;
}

int wg_snow(const double* elev, const double* slope, int64_t n, double base, double alt_div, double top,
            double sl_div, int has_nodata, double nodata, uint8_t* pixels, void* stream) {
  if (n <= 0) return WG_OK;
  if (!elev || !slope || !pixels) return wg::set_error(WG_EARG, "null buffer");
  snow_kernel<<<wg::stream_grid(n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      elev, slope, n, base, alt_div, top, sl_div, has_nodata, nodata, reinterpret_cast<uchar4*>(pixels));
  WG_LAUNCH_CHECK("snow_kernel");
  return WG_OK;
}

int wg_runout_stats(const int64_t* hits, const double* zmax, int64_t n, uint64_t* out, void* stream) {
  if (n <= 0) return WG_OK;
  if (!hits || !zmax || !out) return wg::set_error(WG_EARG, "null buffer");
  runout_stats_kernel<<<wg::stream_grid(n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      reinterpret_cast<const long long*>(hits), zmax, n, reinterpret_cast<unsigned long long*>(out));
  WG_LAUNCH_CHECK("runout_stats_kernel");
  return WG_OK;
}

int wg_synth_combine(const double* rowf, const double* colf, const double* lin, int noct, int64_t nrows,
                     int64_t ncols, double* elev, void* stream) {
  if (nrows * ncols <= 0) return WG_OK;
  synth_kernel<<<wg::stream_grid(nrows * ncols, kBlock), kBlock, 0, wg::as_stream(stream)>>>(rowf, colf, lin, noct,
                                                                                              nrows, ncols, elev);
  WG_LAUNCH_CHECK("synth_kernel");
  return WG_OK;
}

int wg_sub_scalar(double* elev, int64_t n, double v, void* stream) {
  if (n <= 0) return WG_OK;
  sub_scalar_kernel<<<wg::stream_grid(n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(elev, n, v);
  WG_LAUNCH_CHECK("sub_scalar_kernel");
  return WG_OK;
}

}  // extern "C"

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
#include "wg_div.cuh"
#include "wg_fp64.h"
#include "wg_acos.h"

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
// degrees(arccos(clip(nz, -1, 1))) (terrain.py:101-102): numpy's arccos bit
// for bit (wg_acos.h), np.degrees multiplies by 180/pi.
__device__ __forceinline__ double slope_of(double nz) {
  const double c = wg_min(wg_max(nz, -1.0), 1.0);
  return WG_MUL(wg_acos(c), 57.29577951308232);
}

// Release-mask guard band: lattice cells whose slope
// lies within kGuardDeg of a band edge are counted, so a caller can see when
// a threshold decision rests on the last bits of the slope.  The mask kernels
// accumulate counts[0] = set cells (ReleaseMask.count without another pass)
// and counts[1] = borderline cells.
constexpr double kGuardDeg = 1e-9;
__device__ __forceinline__ unsigned borderline(double x, double lo, double hi) {
  return (unsigned)((fabs(x - lo) < kGuardDeg) | (fabs(x - hi) < kGuardDeg));
}

__device__ __forceinline__ void add_counts(unsigned long long* counts, unsigned set, unsigned near) {
  set = __reduce_add_sync(0xffffffffu, set);
  near = __reduce_add_sync(0xffffffffu, near);
  if ((threadIdx.x & 31) == 0) {
    if (set) atomicAdd(counts, (unsigned long long)set);
    if (near) atomicAdd(counts + 1, (unsigned long long)near);
  }
}

// The unit normal of cell (i, j) from its own height and its four
// neighbours' (terrain.py:69-96): central differences inside, one-sided on
// the borders (terrain.py:79-88; neighbours beyond a border are not read),
// five divisions through shared reciprocals with one guard for all of them
// -- the rare guard miss recomputes the cell with __ddiv_rn.  Shared by the
// normals pass and the lattice mask so both give the same bits.
// kInterior: the caller knows the cell is not on a border (a warp-uniform
// test in the normals pass), so the border selects drop out.
template <bool kInterior = false>
__device__ __forceinline__ void cell_normal(double cur, double west, double east, double up, double dn, int i, int jc,
                                            int nrows, int ncols, double cs, double two_cs, double rcs, double r2cs,
                                            bool cs_ok, double& n0, double& n1, double& nz) {
  const bool xb = !kInterior && ((jc == 0) | (jc == ncols - 1));
  const bool yb = !kInterior && ((i == 0) | (i == nrows - 1));
  const double xa = kInterior ? WG_SUB(east, west)
                              : WG_SUB(jc == 0 ? east : (jc == ncols - 1 ? cur : east),
                                       jc == 0 ? cur : (jc == ncols - 1 ? west : west));
  const double ya = kInterior ? WG_SUB(up, dn) : WG_SUB(i == 0 ? cur : up, i == 0 ? dn : (i == nrows - 1 ? cur : dn));
  const double xd = xb ? cs : two_cs, xr = xb ? rcs : r2cs;
  const double yd = yb ? cs : two_cs, yr = yb ? rcs : r2cs;
  bool ok = cs_ok;
  double dzdx = div_fast(xa, xd, xr, ok), dzdy = div_fast(ya, yd, yr, ok);
  double nx = -dzdx, ny = -dzdy;
  double len = WG_SQRT(WG_ADD(WG_ADD(WG_MUL(nx, nx), WG_MUL(ny, ny)), 1.0));
  const double rl = rcp_refined(len);
  ok = ok && b_ok(len);
  n0 = div_fast(nx, len, rl, ok);
  n1 = div_fast(ny, len, rl, ok);
  nz = div_fast(1.0, len, rl, ok);
  if (!ok) {
    dzdx = __ddiv_rn(xa, xd);
    dzdy = __ddiv_rn(ya, yd);
    nx = -dzdx;
    ny = -dzdy;
    len = WG_SQRT(WG_ADD(WG_ADD(WG_MUL(nx, nx), WG_MUL(ny, ny)), 1.0));
    n0 = __ddiv_rn(nx, len);
    n1 = __ddiv_rn(ny, len);
    nz = __ddiv_rn(1.0, len);
  }
}

// 2.5-D stencil: a thread owns one column of a band of kNormBand rows and
// walks down it with a rolling (north, centre, south) register window, so
// every DEM value is loaded once per band (+2 halo rows); east/west
// neighbours come from warp shuffles (edge lanes load their halo).  The five
// divisions per cell use two kernel-wide cellsize reciprocals and one shared
// reciprocal of |n| (wg_div.cuh, __ddiv_rn-exact).  Normals are staged per
// warp in shared memory and written as 16-byte vectors (768 contiguous bytes
// per warp-row).  HBM floor: 8 B in + 24 B (+8 B slope) out per cell.
constexpr int kNormBand = 64;
constexpr int kNormThreads = 256;

#ifndef WG_NORM_MINB
#define WG_NORM_MINB 4  // 61 registers, 4 blocks/SM (A/B: 3.23 -> 2.92 ms with the prefetch)
#endif
__global__ void __launch_bounds__(kNormThreads, WG_NORM_MINB) normals_kernel(const double* __restrict__ e, int nrows, int ncols,
                                                               double cs, double two_cs, double* __restrict__ nrm,
                                                               double* __restrict__ slope) {
  __shared__ __align__(16) double stage[kNormThreads / 32][96];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j = blockIdx.x * kNormThreads + threadIdx.x;
  const int jw0 = j - lane;  // first column of this warp
  if (jw0 >= ncols) return;  // whole warp outside (warp-uniform)
  const bool live = j < ncols;
  const int jc = live ? j : ncols - 1;
  const int i0 = blockIdx.y * kNormBand, i1 = min(i0 + kNormBand, nrows);
  const double rcs = rcp_refined(cs), r2cs = rcp_refined(two_cs);
  const bool cs_fast = b_ok(cs), c2_fast = b_ok(two_cs);
  const double* col = e + jc;
  const bool interior_cols = jw0 > 0 && jw0 + 32 < ncols;  // no lane of the warp on the west / east border
  double up = i0 > 0 ? __ldg(col + (size_t)(i0 - 1) * ncols) : 0.0;
  double cur = __ldg(col + (size_t)i0 * ncols);
  // the row below is loaded one iteration ahead, so its latency overlaps a
  // row of arithmetic
  double dn = (i0 + 1 < nrows) ? __ldg(col + (size_t)(i0 + 1) * ncols) : 0.0;
  for (int i = i0; i < i1; i++) {
    const double dn2 = (i + 2 < nrows) ? __ldg(col + (size_t)(i + 2) * ncols) : 0.0;
    // east / west neighbours of row i
    double west = __shfl_up_sync(0xffffffffu, cur, 1);
    double east = __shfl_down_sync(0xffffffffu, cur, 1);
    const double* row = e + (size_t)i * ncols;
    if (lane == 0 && jc > 0) west = __ldg(row + jc - 1);
    if ((lane == 31 || j + 1 >= ncols) && jc + 1 < ncols) east = __ldg(row + jc + 1);
    double n0, n1, nz;
    if (interior_cols && i > 0 && i < nrows - 1)  // warp-uniform
      cell_normal<true>(cur, west, east, up, dn, i, jc, nrows, ncols, cs, two_cs, rcs, r2cs, c2_fast, n0, n1, nz);
    else
      cell_normal(cur, west, east, up, dn, i, jc, nrows, ncols, cs, two_cs, rcs, r2cs, cs_fast && c2_fast, n0, n1, nz);
    const size_t cell = (size_t)i * ncols + j;
    if (slope != nullptr && live) slope[cell] = slope_of(nz);
    if (nrm != nullptr) {
      // stage the warp's 32 x 3 doubles, then 16-byte stores when aligned
      const size_t base = (size_t)i * ncols + jw0;  // first cell of the warp-row
      const int nlive = min(32, ncols - jw0);
      double* st = stage[wid];
      st[3 * lane] = n0;
      st[3 * lane + 1] = n1;
      st[3 * lane + 2] = nz;
      __syncwarp();
      double* out = nrm + 3 * base;
      if ((((uintptr_t)out) & 15) == 0 && nlive == 32) {
        double2* o2 = reinterpret_cast<double2*>(out);
        const double2* s2 = reinterpret_cast<const double2*>(st);
        o2[lane] = s2[lane];
        if (lane < 16) o2[32 + lane] = s2[32 + lane];
      } else {
        for (int q = lane; q < 3 * nlive; q += 32) out[q] = st[q];
      }
      __syncwarp();
    }
    up = cur;
    cur = dn;
    dn = dn2;
  }
}

__global__ void acos_eval_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ a,
                                 double* __restrict__ d) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double v = __ldg(x + t);
    if (a != nullptr) a[t] = wg_acos(v);
    if (d != nullptr) d[t] = slope_of(v);
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

// The service's hillshade base layer (service.py:527-538): the same shade as
// an opaque gray RGBA texel, texture_from_gray fused in (one 4-byte store).
__global__ void hillshade_rgba_kernel(const double* __restrict__ nrm, int64_t n, double lx, double ly, double lz,
                                      uint32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double* v = nrm + 3 * t;
    const double dot = WG_ADD(WG_ADD(WG_MUL(__ldg(v), lx), WG_MUL(__ldg(v + 1), ly)), WG_MUL(__ldg(v + 2), lz));
    const double sh = wg_min(wg_max(dot, 0.0), 1.0);
    const uint32_t g = (uint32_t)(int)floor(WG_ADD(WG_MUL(sh, 255.0), 0.5));
    out[t] = g | (g << 8) | (g << 16) | 0xFF000000u;
  }
}

// ---------------------------------------------------------------- release mask
// Each thread writes 16 mask bytes of one row (one 16-B store when aligned);
// the slope is read only at stride-lattice cells, the only cells the mask can
// set (simulate.py:222-225), so for stride > 1 the pass is write-bound.
__global__ void release_mask_kernel(const double* __restrict__ s, int nrows, int ncols, double lo, double hi,
                                    int stride, uint8_t* __restrict__ mask, unsigned long long* __restrict__ counts) {
  const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 16;
  unsigned set = 0, near = 0;
  for (int i = blockIdx.y; c0 < ncols && i < nrows; i += gridDim.y) {
    const size_t rowoff = (size_t)i * ncols;
    unsigned char v[16];
    const bool lat_row = (i % stride) == 0;
    int c = c0 % stride == 0 ? c0 : c0 + (stride - c0 % stride);
#pragma unroll
    for (int q = 0; q < 16; q++) v[q] = 0;
    if (lat_row) {
      for (; c < c0 + 16 && c < ncols; c += stride) {
        const double x = __ldg(s + rowoff + c);
        v[c - c0] = (unsigned char)((x >= lo) & (x <= hi));
        set += v[c - c0];
        near += borderline(x, lo, hi);
      }
    }
    uint8_t* out = mask + rowoff + c0;
    if (c0 + 16 <= ncols && (((uintptr_t)out) & 15) == 0) {
      uint4 w;
      w.x = v[0] | (v[1] << 8) | (v[2] << 16) | ((unsigned)v[3] << 24);
      w.y = v[4] | (v[5] << 8) | (v[6] << 16) | ((unsigned)v[7] << 24);
      w.z = v[8] | (v[9] << 8) | (v[10] << 16) | ((unsigned)v[11] << 24);
      w.w = v[12] | (v[13] << 8) | (v[14] << 16) | ((unsigned)v[15] << 24);
      *reinterpret_cast<uint4*>(out) = w;
    } else {
      for (int q = 0; q < 16 && c0 + q < ncols; q++) out[q] = v[q];
    }
  }
  if (counts != nullptr) add_counts(counts, set, near);
}

// Release mask straight from the DEM for grids whose slope field is not
// otherwise needed (C5): the slope is computed only at stride-lattice cells
// of rows [row0, row1) (the only cells the mask can set), with the normals
// pass's own per-cell arithmetic, so the mask equals
// detect_release_points(steepness_deg(compute_normals(grid))) bit for bit.
// Other mask bytes are zeroed by the caller.
__global__ void lattice_mask_kernel(const double* __restrict__ e, int nrows, int ncols, double cs, double two_cs,
                                    double lo, double hi, int stride, int row0, int row1, uint8_t* __restrict__ mask,
                                    unsigned long long* __restrict__ counts) {
  const int64_t lr = (row1 - row0 + stride - 1) / stride, lc = (ncols + stride - 1) / stride;
  const double rcs = rcp_refined(cs), r2cs = rcp_refined(two_cs);
  const bool cs_ok = b_ok(cs) && b_ok(two_cs);
  unsigned set = 0, near = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < lr * lc; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = row0 + (int)(t / lc) * stride, j = (int)(t % lc) * stride;
    const double* c = e + (size_t)i * ncols + j;
    const double cur = __ldg(c);
    const double west = j > 0 ? __ldg(c - 1) : 0.0, east = j + 1 < ncols ? __ldg(c + 1) : 0.0;
    const double up = i > 0 ? __ldg(c - ncols) : 0.0, dn = i + 1 < nrows ? __ldg(c + ncols) : 0.0;
    double n0, n1, nz;
    cell_normal(cur, west, east, up, dn, i, j, nrows, ncols, cs, two_cs, rcs, r2cs, cs_ok, n0, n1, nz);
    const double x = slope_of(nz);
    const unsigned in = (unsigned)((x >= lo) & (x <= hi));
    mask[(size_t)(i - row0) * ncols + j] = (uint8_t)in;
    set += in;
    near += borderline(x, lo, hi);
  }
  if (counts != nullptr) add_counts(counts, set, near);
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
  grid_scan_kernel<<<wg::resident_grid(grid_scan_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      elev, n, nodata, reinterpret_cast<unsigned long long*>(counts));
  WG_LAUNCH_CHECK("grid_scan_kernel");
  return WG_OK;
}

int wg_copy2d_f64(const double* src, int64_t src_ld, double* dst, int64_t dst_ld, int64_t rows, int64_t cols,
                  void* stream) {
  if (rows <= 0 || cols <= 0) return WG_OK;
  if (!src || !dst || src_ld < cols || dst_ld < cols) return wg::set_error(WG_EARG, "bad copy2d arguments");
  copy2d_kernel<<<wg::resident_grid(copy2d_kernel, rows * cols, kBlock), kBlock, 0, wg::as_stream(stream)>>>(src, src_ld, dst, dst_ld,
                                                                                             rows, cols);
  WG_LAUNCH_CHECK("copy2d_kernel");
  return WG_OK;
}

int wg_normals(const double* elev, int64_t nrows, int64_t ncols, double cs, double two_cs, double* normals,
               double* slope, void* stream) {
  if (nrows < 2 || ncols < 2) return wg::set_error(WG_EARG, "grid must be at least 2x2");
  if (!elev || (!normals && !slope)) return wg::set_error(WG_EARG, "null buffer");
  if (nrows > 0x7fffffff || ncols > 0x7fffffff) return wg::set_error(WG_EARG, "grid too large");
  const dim3 grid((unsigned)((ncols + kNormThreads - 1) / kNormThreads), (unsigned)((nrows + kNormBand - 1) / kNormBand));
  normals_kernel<<<grid, kNormThreads, 0, wg::as_stream(stream)>>>(elev, (int)nrows, (int)ncols, cs, two_cs, normals,
                                                                   slope);
  WG_LAUNCH_CHECK("normals_kernel");
  return WG_OK;
}

int wg_steepness(const double* normals, int64_t n, double* slope, void* stream) {
  if (n <= 0) return WG_OK;
  if (!normals || !slope) return wg::set_error(WG_EARG, "null buffer");
  steepness_kernel<<<wg::resident_grid(steepness_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(normals, n, slope);
  WG_LAUNCH_CHECK("steepness_kernel");
  return WG_OK;
}

int wg_acos_eval(const double* x, int64_t n, double* a, double* d, void* stream) {
  if (n <= 0) return WG_OK;
  if (!x || (!a && !d)) return wg::set_error(WG_EARG, "null buffer");
  acos_eval_kernel<<<wg::resident_grid(acos_eval_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(x, n, a, d);
  WG_LAUNCH_CHECK("acos_eval_kernel");
  return WG_OK;
}

int wg_hillshade(const double* normals, int64_t n, double lx, double ly, double lz, uint8_t* out, void* stream) {
  if (n <= 0) return WG_OK;
  if (!normals || !out) return wg::set_error(WG_EARG, "null buffer");
  hillshade_kernel<<<wg::resident_grid(hillshade_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(normals, n, lx, ly, lz, out);
  WG_LAUNCH_CHECK("hillshade_kernel");
  return WG_OK;
}

int wg_hillshade_rgba(const double* normals, int64_t n, double lx, double ly, double lz, uint8_t* out, void* stream) {
  if (n <= 0) return WG_OK;
  if (!normals || !out) return wg::set_error(WG_EARG, "null buffer");
  if (((uintptr_t)out) & 3) return wg::set_error(WG_EARG, "out must be 4-byte aligned");
  hillshade_rgba_kernel<<<wg::resident_grid(hillshade_rgba_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      normals, n, lx, ly, lz, reinterpret_cast<uint32_t*>(out));
  WG_LAUNCH_CHECK("hillshade_rgba_kernel");
  return WG_OK;
}

int wg_release_mask(const double* slope, int64_t nrows, int64_t ncols, double lo, double hi, int64_t stride,
                    uint8_t* mask, uint64_t* counts, void* stream) {
  if (stride < 1) return wg::set_error(WG_EARG, "stride must be >= 1, got %lld", (long long)stride);
  if (nrows * ncols <= 0) return WG_OK;
  if (!slope || !mask) return wg::set_error(WG_EARG, "null buffer");
  if (nrows > 0x7fffffff || ncols > 0x7fffffff) return wg::set_error(WG_EARG, "grid too large");
  const int st = stride > ncols + nrows ? (int)(ncols + nrows) : (int)stride;  // larger strides: same lattice
  const dim3 grid((unsigned)((ncols + 16 * kBlock - 1) / (16 * kBlock)), (unsigned)(nrows < 8192 ? nrows : 8192));
  release_mask_kernel<<<grid, kBlock, 0, wg::as_stream(stream)>>>(slope, (int)nrows, (int)ncols, lo, hi, st, mask,
                                                                  reinterpret_cast<unsigned long long*>(counts));
  WG_LAUNCH_CHECK("release_mask_kernel");
  return WG_OK;
}

int wg_lattice_release_mask(const double* elev, int64_t nrows, int64_t ncols, double cs, double two_cs, double lo,
                            double hi, int64_t stride, int64_t row0, int64_t row1, uint8_t* mask, uint64_t* counts,
                            void* stream) {
  if (stride < 1) return wg::set_error(WG_EARG, "stride must be >= 1, got %lld", (long long)stride);
  if (nrows < 2 || ncols < 2) return wg::set_error(WG_EARG, "grid must be at least 2x2");
  if (row0 < 0 || row1 < row0 || row1 > nrows) return wg::set_error(WG_EARG, "bad row range");
  if (nrows > 0x7fffffff || ncols > 0x7fffffff) return wg::set_error(WG_EARG, "grid too large");
  if (row1 == row0) return WG_OK;
  if (!elev || !mask) return wg::set_error(WG_EARG, "null buffer");
  cudaStream_t st = wg::as_stream(stream);
  WG_CUDA_TRY(cudaMemsetAsync(mask, 0, (size_t)(row1 - row0) * (size_t)ncols, st));
  const int64_t s = stride > nrows + ncols ? nrows + ncols : stride;  // larger strides: same lattice
  const int64_t cells = ((row1 - row0 + s - 1) / s) * ((ncols + s - 1) / s);
  lattice_mask_kernel<<<wg::resident_grid(lattice_mask_kernel, cells, kBlock), kBlock, 0, st>>>(
      elev, (int)nrows, (int)ncols, cs, two_cs, lo, hi, (int)s, (int)row0, (int)row1, mask,
      reinterpret_cast<unsigned long long*>(counts));
  WG_LAUNCH_CHECK("lattice_mask_kernel");
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
  snow_kernel<<<wg::resident_grid(snow_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      elev, slope, n, base, alt_div, top, sl_div, has_nodata, nodata, reinterpret_cast<uchar4*>(pixels));
  WG_LAUNCH_CHECK("snow_kernel");
  return WG_OK;
}

int wg_runout_stats(const int64_t* hits, const double* zmax, int64_t n, uint64_t* out, void* stream) {
  if (n <= 0) return WG_OK;
  if (!hits || !zmax || !out) return wg::set_error(WG_EARG, "null buffer");
  runout_stats_kernel<<<wg::resident_grid(runout_stats_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(
      reinterpret_cast<const long long*>(hits), zmax, n, reinterpret_cast<unsigned long long*>(out));
  WG_LAUNCH_CHECK("runout_stats_kernel");
  return WG_OK;
}

int wg_synth_combine(const double* rowf, const double* colf, const double* lin, int noct, int64_t nrows,
                     int64_t ncols, double* elev, void* stream) {
  if (nrows * ncols <= 0) return WG_OK;
  synth_kernel<<<wg::resident_grid(synth_kernel, nrows * ncols, kBlock), kBlock, 0, wg::as_stream(stream)>>>(rowf, colf, lin, noct,
                                                                                              nrows, ncols, elev);
  WG_LAUNCH_CHECK("synth_kernel");
  return WG_OK;
}

int wg_sub_scalar(double* elev, int64_t n, double v, void* stream) {
  if (n <= 0) return WG_OK;
  sub_scalar_kernel<<<wg::resident_grid(sub_scalar_kernel, n, kBlock), kBlock, 0, wg::as_stream(stream)>>>(elev, n, v);
  WG_LAUNCH_CHECK("sub_scalar_kernel");
  return WG_OK;
}

}  // extern "C"

// Tile-sparse merge of the multi-GPU runout rasters (the
// reference's merge is the per-chunk partial sum / max, simulate.py:489-503).
//
// Each rank simulates the particles of its release-row bands into private
// int64 hit / f64 drop rasters and a touched-tile map (traj.cu).  A band's
// rows belong to one rank; the particles of a band mostly stay near it, so a
// rank touches a few foreign tiles along its band edges.  Those are the only
// data exchanged: packed here into 2*T*T-word blocks (T*T hits, then T*T
// drop bit patterns; cells outside the grid zero), sent to their owners with
// an NCCL all-to-all, and added / max-ed into the owner's rasters here.  Sum
// and max are exact and commutative, so the owners' bands are bit-identical
// to a single-GPU run.  Tiles are (2^tile_log2)^2 cells, row-major over the
// grid: tile t covers rows (t / tiles_x) * T .. +T, columns (t % tiles_x) * T.
#include "wg_internal.cuh"

namespace {

constexpr int kBlock = 256;

__global__ void sorted_offsets_kernel(const int64_t* __restrict__ ids, int64_t n, const int64_t* __restrict__ bounds,
                                      int64_t nb, int64_t* __restrict__ out) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int64_t v = bounds[b];
  int64_t lo = 0, hi = n;  // first index with ids[i] >= v
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (ids[m] < v) lo = m + 1;
    else hi = m;
  }
  out[b] = lo;
}

struct TileGeom {
  int64_t nrows, ncols, tiles_x;
  int sh;
};

__device__ __forceinline__ void tile_origin(const TileGeom& g, int64_t id, int64_t& r0, int64_t& c0) {
  const int64_t ty = id / g.tiles_x;
  r0 = ty << g.sh;
  c0 = (id - ty * g.tiles_x) << g.sh;
}

// one CTA per output tile; segs = (src_off, dst_off, count) triples with
// ascending, contiguous dst_off
__global__ void pack_kernel(const unsigned long long* __restrict__ hits, const unsigned long long* __restrict__ zbits,
                            TileGeom g, const int64_t* __restrict__ ids, const int64_t* __restrict__ segs, int nseg,
                            int64_t nout, int64_t* __restrict__ out_ids, unsigned long long* __restrict__ out) {
  const int T = 1 << g.sh;
  const int64_t cells = (int64_t)T * T;
  for (int64_t o = blockIdx.x; o < nout; o += gridDim.x) {
    int a = 0, b = nseg - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (segs[3 * m + 1] <= o) a = m;
      else b = m - 1;
    }
    const int64_t id = ids[segs[3 * a] + (o - segs[3 * a + 1])];
    if (threadIdx.x == 0) out_ids[o] = id;
    int64_t r0, c0;
    tile_origin(g, id, r0, c0);
    unsigned long long* dst = out + o * 2 * cells;
    for (int64_t q = threadIdx.x; q < cells; q += blockDim.x) {
      const int64_t r = r0 + (q >> g.sh), c = c0 + (q & (T - 1));
      unsigned long long h = 0, z = 0;
      if (r < g.nrows && c < g.ncols) {
        const int64_t cell = r * g.ncols + c;
        h = hits[cell];
        z = zbits[cell];
      }
      dst[q] = h;
      dst[cells + q] = z;
    }
  }
}

// received blocks may target one tile from several ranks: atomics
__global__ void accumulate_kernel(unsigned long long* __restrict__ hits, unsigned long long* __restrict__ zbits,
                                  TileGeom g, const int64_t* __restrict__ ids, int64_t n,
                                  const unsigned long long* __restrict__ in) {
  const int T = 1 << g.sh;
  const int64_t cells = (int64_t)T * T;
  for (int64_t o = blockIdx.x; o < n; o += gridDim.x) {
    int64_t r0, c0;
    tile_origin(g, ids[o], r0, c0);
    const unsigned long long* src = in + o * 2 * cells;
    for (int64_t q = threadIdx.x; q < cells; q += blockDim.x) {
      const int64_t r = r0 + (q >> g.sh), c = c0 + (q & (T - 1));
      if (r >= g.nrows || c >= g.ncols) continue;
      const int64_t cell = r * g.ncols + c;
      const unsigned long long h = src[q], z = src[cells + q];
      // reductions with unused results as PTX red (REDG: cheaper than an
      // atomic to RZ in the trajectory kernel); drops are >= +0.0, so bit
      // order is value order
      if (h) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(hits + cell), "l"(h) : "memory");
      if (z) asm volatile("red.global.max.u64 [%0], %1;" ::"l"(zbits + cell), "l"(z) : "memory");
    }
  }
}

__global__ void zero_kernel(unsigned long long* __restrict__ hits, unsigned long long* __restrict__ zbits, TileGeom g,
                            const int64_t* __restrict__ ids, int64_t n) {
  const int T = 1 << g.sh;
  const int64_t cells = (int64_t)T * T;
  for (int64_t o = blockIdx.x; o < n; o += gridDim.x) {
    int64_t r0, c0;
    tile_origin(g, ids[o], r0, c0);
    for (int64_t q = threadIdx.x; q < cells; q += blockDim.x) {
      const int64_t r = r0 + (q >> g.sh), c = c0 + (q & (T - 1));
      if (r >= g.nrows || c >= g.ncols) continue;
      hits[r * g.ncols + c] = 0;
      zbits[r * g.ncols + c] = 0;
    }
  }
}

int geom_of(int64_t nrows, int64_t ncols, int tile_log2, TileGeom& g) {
  if (nrows < 1 || ncols < 1) return wg::set_error(WG_EARG, "empty grid");
  if (tile_log2 < 1 || tile_log2 > 12) return wg::set_error(WG_EARG, "tile_log2 must be in [1, 12]");
  g.nrows = nrows;
  g.ncols = ncols;
  g.sh = tile_log2;
  g.tiles_x = (ncols + (1LL << tile_log2) - 1) >> tile_log2;
  return WG_OK;
}

int tile_grid(int64_t n) {
  const int64_t cap = (int64_t)wg::sm_count() * 8;
  return (int)(n < cap ? (n > 0 ? n : 1) : cap);
}

}  // namespace

extern "C" {

int wg_sorted_offsets(const int64_t* ids, int64_t n, const int64_t* bounds, int64_t nb, int64_t* out, void* stream) {
  if (nb <= 0) return WG_OK;
  if (!bounds || !out || (n > 0 && !ids)) return wg::set_error(WG_EARG, "null buffer");
  sorted_offsets_kernel<<<(unsigned)((nb + kBlock - 1) / kBlock), kBlock, 0, wg::as_stream(stream)>>>(ids, n, bounds,
                                                                                                      nb, out);
  WG_LAUNCH_CHECK("sorted_offsets_kernel");
  return WG_OK;
}

int wg_tiles_pack(const int64_t* hits, const double* zmax, int64_t nrows, int64_t ncols, int tile_log2,
                  const int64_t* ids, const int64_t* segs, int64_t nseg, int64_t nout, int64_t* out_ids,
                  int64_t* out_data, void* stream) {
  TileGeom g;
  int rc = geom_of(nrows, ncols, tile_log2, g);
  if (rc) return rc;
  if (nout <= 0) return WG_OK;
  if (nseg < 1 || nseg > 0x7fffffff) return wg::set_error(WG_EARG, "bad segment count");
  if (!hits || !zmax || !ids || !segs || !out_ids || !out_data) return wg::set_error(WG_EARG, "null buffer");
  pack_kernel<<<tile_grid(nout), kBlock, 0, wg::as_stream(stream)>>>(
      reinterpret_cast<const unsigned long long*>(hits), reinterpret_cast<const unsigned long long*>(zmax), g, ids,
      segs, (int)nseg, nout, out_ids, reinterpret_cast<unsigned long long*>(out_data));
  WG_LAUNCH_CHECK("pack_kernel");
  return WG_OK;
}

int wg_tiles_accumulate(int64_t* hits, double* zmax, int64_t nrows, int64_t ncols, int tile_log2, const int64_t* ids,
                        int64_t n, const int64_t* data, void* stream) {
  TileGeom g;
  int rc = geom_of(nrows, ncols, tile_log2, g);
  if (rc) return rc;
  if (n <= 0) return WG_OK;
  if (!hits || !zmax || !ids || !data) return wg::set_error(WG_EARG, "null buffer");
  accumulate_kernel<<<tile_grid(n), kBlock, 0, wg::as_stream(stream)>>>(
      reinterpret_cast<unsigned long long*>(hits), reinterpret_cast<unsigned long long*>(zmax), g, ids, n,
      reinterpret_cast<const unsigned long long*>(data));
  WG_LAUNCH_CHECK("accumulate_kernel");
  return WG_OK;
}

int wg_tiles_zero(int64_t* hits, double* zmax, int64_t nrows, int64_t ncols, int tile_log2, const int64_t* ids,
                  int64_t n, void* stream) {
  TileGeom g;
  int rc = geom_of(nrows, ncols, tile_log2, g);
  if (rc) return rc;
  if (n <= 0) return WG_OK;
  if (!hits || !zmax || !ids) return wg::set_error(WG_EARG, "null buffer");
  zero_kernel<<<tile_grid(n), kBlock, 0, wg::as_stream(stream)>>>(reinterpret_cast<unsigned long long*>(hits),
                                                                  reinterpret_cast<unsigned long long*>(zmax), g, ids,
                                                                  n);
  WG_LAUNCH_CHECK("zero_kernel");
  return WG_OK;
}

}  // extern "C"

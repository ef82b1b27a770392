/* TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.
 *
 * Scalar C restatement of the reference particle engine
 * (/root/reference/pkg/src/demflow/simulate.py), used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * leg.  Nothing in paper_2506_23364_b200/ may link or call it.
 *
 * Followed line by line:
 *   rng.py:38-43      mix64 (SplitMix64 finaliser)
 *   rng.py:46-56      derive_key(seed, k, p)
 *   rng.py:59-67      draw_bits / unit_from_bits
 *   simulate.py:231-259 _bilinear_batch  (height + downslope gradient)
 *   simulate.py:262-267 _cells_of
 *   simulate.py:270-412 _simulate_batch  (one particle at a time: the batch
 *                        is lockstep but particles never interact, and every
 *                        draw is addressed by (key, step) -- simulate.py:12-16)
 *   simulate.py:441-504 run_avalanche    (particle i = k*P + p, k = release
 *                        ordinal in row-major order, start = cell centre)
 * Jitter trig calls the host's glibc sin/cos exactly as np.sin/np.cos do
 * (simulate.py:359-360), so on a glibc-2.39 FMA host this oracle is
 * bit-identical to the reference by construction; tests/ pin it against the
 * reference's shipped goldens (pkg/demos/out) and fixtures generated from the
 * reference itself (tests/golden/make_golden.py).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fno-builtin, no
 * -ffast-math: every + - * / sqrt is a separately rounded IEEE op as in numpy).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL
#define FLAT_GRADIENT_THRESHOLD 1e-6 /* terrain.py:19 */
#define FLAT_DIR_EPS 1e-9            /* simulate.py:42 */

static uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * MIX1;
  x = (x ^ (x >> 27)) * MIX2;
  return x ^ (x >> 31);
}

uint64_t orc_derive_key(uint64_t seed, uint64_t k, uint64_t p) {
  uint64_t h = 0;
  h = mix64((h + GOLDEN) ^ seed);
  h = mix64((h + GOLDEN) ^ k);
  h = mix64((h + GOLDEN) ^ p);
  return h;
}

double orc_draw_unit(uint64_t key, uint64_t counter) {
  uint64_t bits = mix64(key + (counter + 1) * GOLDEN);
  return (double)(bits >> 11) * 0x1.0p-53;
}

typedef struct {
  const double* e;
  int64_t nrows, ncols;
  double ox, oy, cs, xmax, ymax;
  double tana, p, omp, rscale, rh;
  int64_t max_steps;
} world_t;

/* simulate.py:231-259 */
static void bilinear(const world_t* w, double x, double y, double* z, double* gx, double* gy) {
  double u = (x - w->ox) / w->cs - 0.5;
  double v = (y - w->oy) / w->cs - 0.5;
  double cmax = (double)w->ncols - 1.0, rmax = (double)w->nrows - 1.0;
  u = u > 0.0 ? u : 0.0; /* np.maximum(u, 0.0) */
  u = u < cmax ? u : cmax;
  v = v > 0.0 ? v : 0.0;
  v = v < rmax ? v : rmax;
  double j0f = floor(u), s0f = floor(v);
  if (j0f > (double)w->ncols - 2.0) j0f = (double)w->ncols - 2.0;
  if (s0f > (double)w->nrows - 2.0) s0f = (double)w->nrows - 2.0;
  double wu = u - j0f, wv = v - s0f;
  int64_t j0 = (int64_t)j0f, s0 = (int64_t)s0f;
  int64_t i1 = (w->nrows - 1) - s0, i0 = i1 - 1;
  double z00 = w->e[i1 * w->ncols + j0], z10 = w->e[i1 * w->ncols + j0 + 1];
  double z01 = w->e[i0 * w->ncols + j0], z11 = w->e[i0 * w->ncols + j0 + 1];
  double gx_s = z10 - z00, gx_n = z11 - z01, gy_w = z01 - z00, gy_e = z11 - z10;
  double zs = z00 + gx_s * wu, zn = z01 + gx_n * wu;
  *z = zs + (zn - zs) * wv;
  double dzdx = (gx_s + (gx_n - gx_s) * wv) / w->cs;
  double dzdy = (gy_w + (gy_e - gy_w) * wu) / w->cs;
  *gx = -dzdx;
  *gy = -dzdy;
}

/* simulate.py:262-267 */
static int64_t cell_of(const world_t* w, double x, double y) {
  double cf = floor((x - w->ox) / w->cs), sf = floor((y - w->oy) / w->cs);
  int64_t col = (int64_t)cf, s = (int64_t)sf;
  if (col < 0) col = 0;
  if (col > w->ncols - 1) col = w->ncols - 1;
  if (s < 0) s = 0;
  if (s > w->nrows - 1) s = w->nrows - 1;
  return ((w->nrows - 1) - s) * w->ncols + col;
}

typedef struct {
  int64_t* hits;
  double* zmax;
  double* path; /* optional (cap x 2) */
  int64_t path_cap, path_len;
  int shared; /* rasters shared between threads -> atomics */
} sink_t;

static void hit(sink_t* sk, int64_t cell, double delta, int with_z) {
  if (!sk->hits) return;
  if (sk->shared) {
    __atomic_fetch_add(&sk->hits[cell], 1, __ATOMIC_RELAXED);
    if (with_z) {
      uint64_t* zb = (uint64_t*)&sk->zmax[cell];
      uint64_t nb;
      memcpy(&nb, &delta, 8);
      uint64_t cur = __atomic_load_n(zb, __ATOMIC_RELAXED);
      /* non-negative doubles order like their bit patterns */
      while (nb > cur && !__atomic_compare_exchange_n(zb, &cur, nb, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
      }
    }
  } else {
    sk->hits[cell] += 1;
    if (with_z && delta > sk->zmax[cell]) sk->zmax[cell] = delta;
  }
}

static void rec(sink_t* sk, double x, double y) {
  if (!sk->path) return;
  if (sk->path_len < sk->path_cap) {
    sk->path[2 * sk->path_len] = x;
    sk->path[2 * sk->path_len + 1] = y;
  }
  sk->path_len++;
}

/* One particle of simulate.py:270-412.  Returns the stop reason code
 * (0 RUNOUT_ANGLE, 1 DOMAIN_EXIT, 2 FLAT, 3 MAX_STEPS; simulate.py:62-67). */
static int particle(const world_t* w, double sx, double sy, uint64_t key, sink_t* sk, int64_t* steps_out,
                    double* end_xy) {
  double x = sx, y = sy, z, gx, gy;
  bilinear(w, x, y, &z, &gx, &gy);
  const double zrel = z, relx = x, rely = y;
  double dpx = 0.0, dpy = 0.0;
  int64_t steps = 0;
  int reason;
  rec(sk, x, y);
  hit(sk, cell_of(w, x, y), 0.0, 0); /* simulate.py:315-317: start visit, no z update */
  for (;;) {
    double ddx = x - relx, ddy = y - rely;
    double hdist = sqrt(ddx * ddx + ddy * ddy);
    if (steps >= 1 && (zrel - z) < w->tana * hdist) { reason = 0; break; }
    if (steps >= w->max_steps) { reason = 3; break; }
    double zd, ggx, ggy;
    bilinear(w, x, y, &zd, &ggx, &ggy);
    double gmag = sqrt(ggx * ggx + ggy * ggy);
    double ux = 0.0, uy = 0.0;
    if (gmag >= FLAT_GRADIENT_THRESHOLD) { ux = ggx / gmag; uy = ggy / gmag; }
    double bx, by;
    if (steps == 0) { bx = ux; by = uy; }
    else { bx = w->p * dpx + w->omp * ux; by = w->p * dpy + w->omp * uy; }
    double bmag = sqrt(bx * bx + by * by);
    if (bmag < FLAT_DIR_EPS) { reason = 2; break; }
    double dx = bx / bmag, dy = by / bmag;
    if (w->rscale != 0.0) {
      double u01 = orc_draw_unit(key, (uint64_t)steps);
      double theta = (2.0 * u01 - 1.0) * w->rh;
      double ct = cos(theta), st = sin(theta);
      double ndx = dx * ct - dy * st, ndy = dx * st + dy * ct;
      dx = ndx;
      dy = ndy;
    }
    double nx = x + w->cs * dx, ny = y + w->cs * dy;
    int outside = (nx < w->ox) || (nx > w->xmax) || (ny < w->oy) || (ny > w->ymax);
    double fx = nx, fy = ny;
    if (outside) {
      double tx = 1.0, ty = 1.0;
      if (nx < w->ox) tx = (w->ox - x) / (nx - x);
      else if (nx > w->xmax) tx = (w->xmax - x) / (nx - x);
      if (ny < w->oy) ty = (w->oy - y) / (ny - y);
      else if (ny > w->ymax) ty = (w->ymax - y) / (ny - y);
      double tc = ty < tx ? ty : tx; /* np.minimum */
      fx = x + (nx - x) * tc;
      fy = y + (ny - y) * tc;
    }
    double znew, g2x, g2y;
    bilinear(w, fx, fy, &znew, &g2x, &g2y);
    double delta = z - znew;
    delta = delta > 0.0 ? delta : 0.0; /* np.maximum(0.0, .) (ties keep +0.0) */
    hit(sk, cell_of(w, fx, fy), delta, 1);
    rec(sk, fx, fy);
    x = fx; y = fy; z = znew; dpx = dx; dpy = dy; steps++;
    if (outside) { reason = 1; break; }
  }
  if (steps_out) *steps_out = steps;
  if (end_xy) { end_xy[0] = x; end_xy[1] = y; }
  return reason;
}

static void init_world(world_t* w, const double* e, int64_t nrows, int64_t ncols, double ox, double oy, double cs,
                       double xmax, double ymax, double tana, double p, double omp, double rscale, double rh,
                       int64_t max_steps) {
  w->e = e; w->nrows = nrows; w->ncols = ncols; w->ox = ox; w->oy = oy; w->cs = cs;
  w->xmax = xmax; w->ymax = ymax; w->tana = tana; w->p = p; w->omp = omp; w->rscale = rscale;
  w->rh = rh; w->max_steps = max_steps;
}

/* simulate_particle (simulate.py:415-438).  Returns reason; path has
 * min(len, cap) rows written, *path_len = full length. */
int orc_simulate_particle(const double* e, int64_t nrows, int64_t ncols, double ox, double oy, double cs,
                          double xmax, double ymax, double tana, double p, double omp, double rscale, double rh,
                          int64_t max_steps, double sx, double sy, uint64_t key, double* path, int64_t cap,
                          int64_t* path_len) {
  world_t w;
  init_world(&w, e, nrows, ncols, ox, oy, cs, xmax, ymax, tana, p, omp, rscale, rh, max_steps);
  sink_t sk = {0};
  sk.path = path;
  sk.path_cap = cap;
  int r = particle(&w, sx, sy, key, &sk, NULL, NULL);
  *path_len = sk.path_len;
  return r;
}

typedef struct {
  const world_t* w;
  const int64_t* cells; /* flat release-cell indices, row-major order */
  int64_t per_cell;
  uint64_t seed;
  int64_t lo, hi, chunk;
  int64_t* next; /* shared chunk cursor */
  int64_t* hits;
  double* zmax;
  /* optional per-particle records, indexed i - lo0 */
  int64_t lo0;
  int8_t* reasons;
  int64_t* steps;
  double* ends;
  int shared;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  sink_t sk = {0};
  sk.hits = j->hits;
  sk.zmax = j->zmax;
  sk.shared = j->shared;
  for (;;) {
    int64_t c = __atomic_fetch_add(j->next, j->chunk, __ATOMIC_RELAXED);
    if (c >= j->hi) break;
    int64_t e = c + j->chunk < j->hi ? c + j->chunk : j->hi;
    for (int64_t i = c; i < e; i++) {
      int64_t k = i / j->per_cell, pp = i % j->per_cell;
      int64_t flat = j->cells[k];
      int64_t row = flat / j->w->ncols, col = flat % j->w->ncols;
      double cx = j->w->ox + ((double)col + 0.5) * j->w->cs; /* simulate.py:474-475 */
      double cy = j->w->oy + ((double)(j->w->nrows - 1 - row) + 0.5) * j->w->cs;
      uint64_t key = orc_derive_key(j->seed, (uint64_t)k, (uint64_t)pp);
      int64_t st;
      double end[2];
      int r = particle(j->w, cx, cy, key, &sk, &st, end);
      if (j->reasons) j->reasons[i - j->lo0] = (int8_t)r;
      if (j->steps) j->steps[i - j->lo0] = st;
      if (j->ends) { j->ends[2 * (i - j->lo0)] = end[0]; j->ends[2 * (i - j->lo0) + 1] = end[1]; }
    }
  }
  return NULL;
}

/* run_avalanche over particle range [lo, hi) of the global index
 * i = k * per_cell + p, accumulating into hits / zmax (caller zero-inits). */
int orc_run_particles(const double* e, int64_t nrows, int64_t ncols, double ox, double oy, double cs, double xmax,
                      double ymax, double tana, double p, double omp, double rscale, double rh, int64_t max_steps,
                      const int64_t* cells, int64_t per_cell, uint64_t seed, int64_t lo, int64_t hi, int64_t* hits,
                      double* zmax, int8_t* reasons, int64_t* steps, double* ends, int threads) {
  world_t w;
  init_world(&w, e, nrows, ncols, ox, oy, cs, xmax, ymax, tana, p, omp, rscale, rh, max_steps);
  if (threads < 1) threads = 1;
  int64_t next = lo;
  job_t base = {&w, cells, per_cell, seed, lo, hi, 64, &next, hits, zmax, lo, reasons, steps, ends, threads > 1};
  if (threads == 1) {
    worker(&base);
    return 0;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, worker, &base);
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  free(th);
  return 0;
}

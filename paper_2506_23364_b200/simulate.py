"""Monte-Carlo gravitational mass flow and snow-cover shading
(mirrors demflow/simulate.py).

The particle engine is the sm_100a kernel in csrc/traj.cu; this module keeps
the reference's types, parameter validation, error behaviour and host-side
scalar derivations (simulate.py:292-298), which are computed here with Python
floats exactly as the reference does and handed to the kernel verbatim.

Multi-GPU (opt-in): ``run_avalanche(..., group=pg)`` shards the particles
by release-row bands over the ranks of the process group and merges the
private rasters tile-sparsely (shard.py); every rank then holds the
bitwise-identical raster a single GPU (and the reference) produces.  Without
``group`` the call is local, as the reference's is.
"""

from __future__ import annotations

import ctypes
import math
import weakref
from dataclasses import dataclass, replace
from enum import Enum

import numpy as np
import torch

from . import _device, _lib, rng
from ._resident import Resident
from .grid import DemGrid
from .overlay import OverlayTexture
from .terrain import NormalField, SlopeField, steepness_deg

_FLAT_DIR_EPS = 1e-9
FLAT_GRADIENT_THRESHOLD = 1e-6  # terrain.py:19 (re-exported by the reference's simulate)
_HALF_PI = math.pi / 2.0


class SimulationError(ValueError):
    pass


class ParamError(ValueError):
    pass


class StopReason(str, Enum):
    RUNOUT_ANGLE = "RUNOUT_ANGLE"
    DOMAIN_EXIT = "DOMAIN_EXIT"
    FLAT = "FLAT"
    MAX_STEPS = "MAX_STEPS"


_REASON_BY_CODE = (
    StopReason.RUNOUT_ANGLE,
    StopReason.DOMAIN_EXIT,
    StopReason.FLAT,
    StopReason.MAX_STEPS,
)


@dataclass(frozen=True)
class AvalancheParams:
    """Knobs of the mass-flow model (simulate.py:70-105)."""

    persistence: float = 0.9
    randomness: float = 0.16
    runout_angle_deg: float = 25.0
    particles_per_release_cell: int = 2048
    seed: int = 0
    max_steps: int | None = None

    def __post_init__(self):
        if not (0.0 <= self.persistence <= 1.0):
            raise ParamError(f"persistence must be in [0, 1], got {self.persistence}")
        if not (0.0 <= self.randomness <= 1.0):
            raise ParamError(f"randomness must be in [0, 1], got {self.randomness}")
        if not (0.0 < self.runout_angle_deg < 90.0):
            raise ParamError(f"runout_angle_deg must be in (0, 90), got {self.runout_angle_deg}")
        if self.particles_per_release_cell < 1:
            raise ParamError(
                f"particles_per_release_cell must be >= 1, got {self.particles_per_release_cell}"
            )
        if self.max_steps is not None and self.max_steps < 1:
            raise ParamError(f"max_steps must be >= 1, got {self.max_steps}")


@dataclass(frozen=True)
class SnowParams:
    """Snow shading: altitude ramp times steepness ramp (simulate.py:108-132)."""

    snow_line_m: float
    altitude_blend_m: float = 200.0
    max_steepness_deg: float = 50.0
    steepness_blend_deg: float = 10.0

    def __post_init__(self):
        if self.altitude_blend_m < 0:
            raise ParamError(f"altitude_blend_m must be >= 0, got {self.altitude_blend_m}")
        if self.steepness_blend_deg < 0:
            raise ParamError(f"steepness_blend_deg must be >= 0, got {self.steepness_blend_deg}")
        if not (0.0 <= self.max_steepness_deg <= 90.0):
            raise ParamError(f"max_steepness_deg must be in [0, 90], got {self.max_steepness_deg}")


class ReleaseMask(Resident):
    """Boolean raster marking particle release cells (simulate.py:135-156).

    Masks produced by the steepness band (detect_release_points,
    release_mask_from_dem) carry the producing kernel's device counters: the
    set-cell count and ``borderline``, the lattice cells whose slope lies
    within 1e-9 degrees of a band edge (the mask's guard band, SURVEY 8a
    rows a7/a8).  Other device masks count through the compaction that
    ``release_cells`` runs anyway (its cell list is kept on the mask)."""

    _payload = ("mask",)
    _dtypes = {"mask": (np.dtype(np.bool_), torch.bool)}

    def __init__(self, mask, *, _counts: torch.Tensor | None = None):
        super().__init__(mask=mask)
        object.__setattr__(self, "_count", None)
        object.__setattr__(self, "_borderline", None)
        object.__setattr__(self, "_counts_dev", _counts)
        object.__setattr__(self, "_cells", None)

    @property
    def nrows(self) -> int:
        return self.shape_of("mask")[0]

    @property
    def ncols(self) -> int:
        return self.shape_of("mask")[1]

    def _read_counts(self) -> None:
        n, near = _device.read_small(self._counts_dev)
        object.__setattr__(self, "_count", int(n))
        object.__setattr__(self, "_borderline", int(near))
        object.__setattr__(self, "_counts_dev", None)

    @property
    def count(self) -> int:
        if self._count is None:
            if self._counts_dev is not None:
                self._read_counts()
            elif self.on_device("mask"):
                object.__setattr__(self, "_count", int(release_cells(self).numel()))
            else:
                object.__setattr__(self, "_count", int(self._h["mask"].sum()))
        return self._count

    @property
    def borderline(self) -> int | None:
        """Lattice cells within 1e-9 degrees of a band edge (None for masks
        not produced from a slope band)."""
        if self._counts_dev is not None:
            self._read_counts()
        return self._borderline

    def __repr__(self) -> str:
        return f"ReleaseMask({self.nrows}x{self.ncols})"


class RunoutRaster(Resident):
    """Accumulated flow field: per-cell max vertical drop and hit count
    (simulate.py:159-190).  Invariants are checked by one device pass
    (wg_runout_stats) that also yields the avalanche stats."""

    _payload = ("z_delta_max", "hit_count")
    _dtypes = {
        "z_delta_max": (np.dtype(np.float64), torch.float64),
        "hit_count": (np.dtype(np.int64), torch.int64),
    }

    def __init__(self, z_delta_max, hit_count, *, _stats: tuple[int, int, float] | None = None,
                 _deferred: bool = False):
        zs = tuple(z_delta_max.shape) if isinstance(z_delta_max, torch.Tensor) else np.shape(z_delta_max)
        hs = tuple(hit_count.shape) if isinstance(hit_count, torch.Tensor) else np.shape(hit_count)
        if tuple(zs) != tuple(hs):
            raise SimulationError(f"layer shapes differ: {tuple(zs)} vs {tuple(hs)}")
        super().__init__(z_delta_max=z_delta_max, hit_count=hit_count)
        object.__setattr__(self, "_stats", _stats)
        object.__setattr__(self, "_stats_dev", None)
        self._validate(_deferred)

    def _validate(self, deferred: bool = False) -> None:
        """``deferred`` (rasters the trajectory kernel just wrote, whose
        invariants hold by construction): launch the stats pass and read it
        back only when a stat is first used, so the host does not wait for
        the simulation here."""
        if self._stats is not None:
            return
        if not (self.on_device("z_delta_max") or torch.cuda.is_available()):
            zd, hc = self._h["z_delta_max"], self._h["hit_count"]
            self._check_host(zd, hc)
            object.__setattr__(self, "_stats", (int(hc.sum()), int(np.count_nonzero(hc)), float(zd.max()) if zd.size else 0.0))
            return
        L = _lib.lib()
        z, h = self.dev("z_delta_max"), self.dev("hit_count")
        out = torch.zeros(4, dtype=torch.int64, device=z.device)
        _lib.check(L.wg_runout_stats(_lib.ptr(h), _lib.ptr(z), z.numel(), _lib.ptr(out), _lib.stream_ptr()),
                   SimulationError)
        if deferred:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            object.__setattr__(self, "_stats_dev", (out, ev))
            return
        self._resolve(out)

    def _resolve(self, out: torch.Tensor) -> None:
        s, nnz, zbits, bad = _device.read_small(out)
        if bad:
            # reproduce the reference's specific message
            self._check_host(self.z_delta_max, self.hit_count)
            raise SimulationError("invalid runout raster")
        zmax = float(np.array([zbits], dtype=np.int64).view(np.float64)[0])
        object.__setattr__(self, "_stats", (s, nnz, zmax))

    @staticmethod
    def _check_host(zd, hc) -> None:
        if not np.all(np.isfinite(zd)) or np.any(zd < 0):
            raise SimulationError("z_delta_max must be finite and non-negative")
        if np.any(hc < 0):
            raise SimulationError("hit_count must be non-negative")
        if np.any((zd > 0) & (hc == 0)):
            raise SimulationError("z_delta_max positive on a cell with no hits")

    @property
    def nrows(self) -> int:
        return self.shape_of("z_delta_max")[0]

    @property
    def ncols(self) -> int:
        return self.shape_of("z_delta_max")[1]

    def _stat(self, i: int):
        if self._stats is None:
            out, ev = self._stats_dev
            ev.synchronize()  # the stats pass may have run on another stream
            self._resolve(out)
            object.__setattr__(self, "_stats_dev", None)
        return self._stats[i]

    @property
    def total_hits(self) -> int:
        return self._stat(0)

    @property
    def cells_hit(self) -> int:
        return self._stat(1)

    @property
    def z_max(self) -> float:
        return self._stat(2)

    def __repr__(self) -> str:
        return f"RunoutRaster({self.nrows}x{self.ncols})"


@dataclass(frozen=True)
class Trajectory:
    """Positions of one particle, release point first (simulate.py:193-204)."""

    positions: np.ndarray
    stop_reason: StopReason

    def __post_init__(self):
        p = np.asarray(self.positions, dtype=np.float64)
        if p.ndim != 2 or p.shape[1] != 2 or p.shape[0] < 1:
            raise SimulationError(f"positions must be (n >= 1, 2), got {p.shape}")
        object.__setattr__(self, "positions", p)


def detect_release_points(
    slope: SlopeField,
    min_steepness_deg: float,
    max_steepness_deg: float,
    stride: int = 1,
) -> ReleaseMask:
    """Cells whose steepness lies in [min, max] (inclusive), thinned to every
    stride-th row and column (simulate.py:207-225); one device pass."""
    if stride < 1:
        raise ParamError(f"stride must be >= 1, got {stride}")
    if min_steepness_deg > max_steepness_deg:
        raise ParamError(f"empty steepness band [{min_steepness_deg}, {max_steepness_deg}]")
    L = _lib.lib()
    s = slope.dev("slope_deg")
    out = _device.empty(tuple(s.shape), torch.uint8)
    counts = _device.zeros((2,), torch.int64)
    _lib.check(
        L.wg_release_mask(_lib.ptr(s), slope.nrows, slope.ncols, float(min_steepness_deg), float(max_steepness_deg),
                          int(stride), _lib.ptr(out), _lib.ptr(counts), _lib.stream_ptr()),
        ParamError,
    )
    return ReleaseMask(out.view(torch.bool), _counts=counts)


def release_mask_from_dem(
    grid: DemGrid,
    min_steepness_deg: float,
    max_steepness_deg: float,
    stride: int = 1,
) -> ReleaseMask:
    """detect_release_points(steepness_deg(compute_normals(grid)), ...) bit for
    bit, computing the slope only at the stride-lattice cells the mask can
    set (wg_lattice_release_mask) -- for grids whose normal and slope fields
    are not needed otherwise (the 65536^2 config: 128 GiB of fields avoided)."""
    from .terrain import TerrainError

    if stride < 1:
        raise ParamError(f"stride must be >= 1, got {stride}")
    if min_steepness_deg > max_steepness_deg:
        raise ParamError(f"empty steepness band [{min_steepness_deg}, {max_steepness_deg}]")
    if grid.has_nodata():
        raise TerrainError("normals require a gap-free grid (nodata present)")
    L = _lib.lib()
    e = grid.device_elevations()
    out = _device.empty((grid.nrows, grid.ncols), torch.uint8)
    counts = _device.zeros((2,), torch.int64)
    cs = grid.cellsize
    _lib.check(
        L.wg_lattice_release_mask(_lib.ptr(e), grid.nrows, grid.ncols, cs, 2.0 * cs, float(min_steepness_deg),
                                  float(max_steepness_deg), int(stride), 0, grid.nrows, _lib.ptr(out),
                                  _lib.ptr(counts), _lib.stream_ptr()),
        ParamError,
    )
    return ReleaseMask(out.view(torch.bool), _counts=counts)


# -- the particle engine (csrc/traj.cu) ----------------------------------------


@dataclass(frozen=True)
class _Scalars:
    """Host-derived kernel scalars, computed as simulate.py:286-298 does."""

    nrows: int
    ncols: int
    ox: float
    oy: float
    cs: float
    xmax: float
    ymax: float
    tana: float
    p: float
    omp: float
    rscale: float
    rh: float
    max_steps: int


def kernel_scalars(grid: DemGrid, params: AvalancheParams) -> _Scalars:
    cs = grid.cellsize
    ox = grid.origin_x
    oy = grid.origin_y
    return _Scalars(
        nrows=grid.nrows,
        ncols=grid.ncols,
        ox=ox,
        oy=oy,
        cs=cs,
        xmax=ox + grid.ncols * cs,
        ymax=oy + grid.nrows * cs,
        tana=math.tan(math.radians(params.runout_angle_deg)),
        p=params.persistence,
        omp=1.0 - params.persistence,
        rscale=params.randomness,
        rh=params.randomness * _HALF_PI,
        max_steps=params.max_steps if params.max_steps is not None else 10 * max(grid.ncols, grid.nrows),
    )


def _sc_args(sc: _Scalars) -> tuple:
    return (sc.nrows, sc.ncols, float(sc.ox), float(sc.oy), float(sc.cs), float(sc.xmax), float(sc.ymax),
            float(sc.tana), float(sc.p), float(sc.omp), float(sc.rscale), float(sc.rh), int(sc.max_steps))


def release_cells(mask: ReleaseMask) -> torch.Tensor:
    """Row-major flat indices of the set mask cells (np.flatnonzero order,
    simulate.py:465) by device stream compaction (wg_mask_compact); kept on
    the (immutable) mask for later calls."""
    if mask._cells is not None:
        return mask._cells
    L = _lib.lib()
    m = mask.dev("mask").view(torch.uint8).reshape(-1)
    n = m.numel()
    cells = _device.empty((max(n, 1),), torch.int64)
    count = _device.zeros((1,), torch.int64)
    scratch = _device.empty((int(L.wg_compact_scratch_bytes(n)),), torch.uint8)
    _lib.check(L.wg_mask_compact(_lib.ptr(m), n, _lib.ptr(cells), _lib.ptr(count), _lib.ptr(scratch),
                                 _lib.stream_ptr()))
    k = int(_device.read_small(count.reshape(-1)[:1])[0])
    object.__setattr__(mask, "_cells", cells[:k])
    if mask._count is None:
        object.__setattr__(mask, "_count", k)
    return mask._cells


_LAYOUT_HEADROOM = 8 << 30  # HBM left free after a gather layout (NCCL, peers, the next rasters)


def _try_empty(n: int) -> torch.Tensor | None:
    """A float64 buffer of n elements, or None when it would leave less than
    _LAYOUT_HEADROOM of HBM free.  When this process's own allocations leave
    ample room the buffer is taken directly; near the limit the driver's
    free memory (other processes, the context, NCCL) plus what the caching
    allocator holds unused decides -- cudaMemGetInfo is kept off the common
    path, where it would cost a driver round trip per grid."""
    dev = _device.device()
    need = 8 * n + _LAYOUT_HEADROOM
    if torch.cuda.get_device_properties(dev).total_memory - torch.cuda.memory_allocated(dev) < 4 * need:
        free, _ = torch.cuda.mem_get_info(dev)
        spare = torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
        if need > free + spare:
            return None
    try:
        return _device.empty((n,), torch.float64)
    except torch.cuda.OutOfMemoryError:
        return None


def build_quad(grid: DemGrid) -> torch.Tensor | None:
    """Patch-corner layout of the DEM (wg_build_quad: 32 B per cell, four
    times the DEM) so every particle step gathers its bilinear patch with one
    256-bit load; None when it does not fit (see build_gather_layout)."""
    quad = _try_empty(grid.nrows * grid.ncols * 4)
    if quad is None:
        return None
    L = _lib.lib()
    _lib.check(L.wg_build_quad(_lib.ptr(grid.device_elevations()), grid.nrows, grid.ncols, _lib.ptr(quad),
                               _lib.stream_ptr()), ParamError)
    return quad


def build_pair(grid: DemGrid) -> torch.Tensor | None:
    """Row-pair layout of the DEM (wg_build_pair: 16 B per cell, twice the
    DEM): two 128-bit loads per step; None when it does not fit."""
    pair = _try_empty(grid.nrows * grid.ncols * 2)
    if pair is None:
        return None
    L = _lib.lib()
    _lib.check(L.wg_build_pair(_lib.ptr(grid.device_elevations()), grid.nrows, grid.ncols, _lib.ptr(pair),
                               _lib.stream_ptr()), ParamError)
    return pair


def build_gather_layout(grid: DemGrid) -> tuple[torch.Tensor | None, torch.Tensor | None]:
    """(quad, pair) for the trajectory gather: the patch-corner quads when
    they fit, else the row pairs, else neither (four loads from the DEM).
    The results are identical for every layout."""
    quad = build_quad(grid)
    if quad is not None:
        return quad, None
    return None, build_pair(grid)


_LAYOUT_GRIDS = 2  # grids that keep their gather layout (4x / 2x the DEM each)
_layout_owners: list = []  # weak references to them, oldest first


def gather_layout(grid: DemGrid) -> tuple[torch.Tensor | None, torch.Tensor | None, torch.Tensor]:
    """(quad, pair, absmax) of an immutable grid, built on first use and kept
    on the grid: the trajectory kernel's gather layout and the bits of max
    |z| (the operand bound of its divisions) -- one 1.6 ms / 10.7 GB pass at
    16384^2 per grid instead of per launch.  Only the _LAYOUT_GRIDS most
    recent grids keep theirs (an executor's cache may hold many grids; a
    layout is four times the DEM)."""
    cached = grid._gather
    if cached is not None:
        return cached
    L = _lib.lib()
    e = grid.device_elevations()
    absmax = _device.empty((1,), torch.int64)
    _lib.check(L.wg_absmax(_lib.ptr(e), e.numel(), _lib.ptr(absmax), _lib.stream_ptr()), ParamError)
    _layout_owners[:] = [r for r in _layout_owners if r() is not None]
    while len(_layout_owners) >= _LAYOUT_GRIDS:
        old = _layout_owners.pop(0)()
        if old is not None:
            object.__setattr__(old, "_gather", None)  # freed once its launches are done (stream-ordered)
    quad, pair = build_gather_layout(grid)
    cached = (quad, pair, absmax)
    object.__setattr__(grid, "_gather", cached)
    _layout_owners.append(weakref.ref(grid))
    return cached


def run_avalanche_device(
    grid: DemGrid,
    cells: torch.Tensor,
    params: AvalancheParams,
    *,
    i_lo: int = 0,
    i_hi: int | None = None,
    ranges: list[tuple[int, int]] | None = None,
    hits: torch.Tensor | None = None,
    zmax: torch.Tensor | None = None,
    touched: torch.Tensor | None = None,
    plan=None,
    rank: int = 0,
    stream: torch.cuda.Stream | None = None,
) -> tuple[torch.Tensor, torch.Tensor]:
    """Launch the trajectory kernel over the particles [i_lo, i_hi) (or the
    ascending disjoint `ranges`, a rank's bands) accumulating into (hits,
    zmax); with `touched` (and the shard.BandPlan `plan`, this being `rank`)
    also marking the tiles of other ranks' bands its visits land in.  No
    host sync."""
    L = _lib.lib()
    sc = kernel_scalars(grid, params)
    total = int(cells.numel()) * params.particles_per_release_cell
    if ranges is None:
        ranges = [(int(i_lo), total if i_hi is None else int(i_hi))]
    ranges = [(int(a), int(b)) for a, b in ranges]
    if hits is None:
        hits = _device.zeros((grid.nrows, grid.ncols), torch.int64)
    if zmax is None:
        zmax = _device.zeros((grid.nrows, grid.ncols), torch.float64)
    if all(b <= a for a, b in ranges):
        return hits, zmax
    if touched is not None and (plan is None or plan.nranks < 2):
        touched = None  # one rank: no other rank's bands to mark
    span_lo, span_hi = ranges[0][0], ranges[-1][1]
    scratch = _device.empty((int(L.wg_avalanche_scratch_bytes(params.particles_per_release_cell, span_lo,
                                                               span_hi)),), torch.uint8)
    dem = grid.device_elevations()
    quad, pair, absmax = gather_layout(grid)
    pairs = (ctypes.c_int64 * (2 * len(ranges)))(*[v for r in ranges for v in r])
    _lib.check(
        L.wg_run_avalanche(
            _lib.ptr(dem), _lib.ptr(quad), _lib.ptr(pair), *_sc_args(sc), _lib.ptr(cells),
            params.particles_per_release_cell, rng.seed_word(params.seed), pairs, len(ranges), _lib.ptr(absmax),
            _lib.ptr(hits), _lib.ptr(zmax), _lib.ptr(touched), plan.tile_log2 if plan else 0,
            plan.band_log2 if plan else 0, int(rank), plan.nranks if plan else 1, _lib.ptr(scratch),
            _lib.stream_ptr(stream),
        ),
        ParamError,
    )
    return hits, zmax


def run_avalanche(
    grid: DemGrid,
    mask: ReleaseMask,
    params: AvalancheParams,
    threads: int = 1,
    *,
    group=None,
) -> RunoutRaster:
    """Release particles from every marked cell and accumulate the flow
    (simulate.py:441-504).  ``threads`` is validated like the reference and
    otherwise ignored: the GPU result is bitwise independent of any schedule.
    ``group`` (a torch.distributed process group, one GPU per rank, every
    rank calling with the same grid and mask) shards the particles over its
    ranks; each rank returns the whole raster."""
    if (mask.nrows, mask.ncols) != (grid.nrows, grid.ncols):
        raise SimulationError(
            f"mask shape {(mask.nrows, mask.ncols)} does not match grid {(grid.nrows, grid.ncols)}"
        )
    if threads < 1:
        raise ParamError(f"threads must be >= 1, got {threads}")
    if grid.has_nodata():
        raise SimulationError("simulation requires a gap-free grid")
    cells = release_cells(mask)
    if group is not None:
        from . import shard

        run = shard.run_sharded(grid, cells, params, group)
        shard.gather_bands(run.hits, run.zmax, run.plan, group)
        return RunoutRaster(run.zmax, run.hits, _deferred=True)
    hits = _device.zeros((grid.nrows, grid.ncols), torch.int64)
    zmax = _device.zeros((grid.nrows, grid.ncols), torch.float64)
    if cells.numel() == 0:
        return RunoutRaster(zmax, hits, _deferred=True)
    run_avalanche_device(grid, cells, params, hits=hits, zmax=zmax)
    return RunoutRaster(zmax, hits, _deferred=True)


def simulate_particle(
    grid: DemGrid,
    start: tuple[float, float],
    params: AvalancheParams,
    stream: rng.CounterStream | None = None,
) -> Trajectory:
    """Trace a single particle and return its full trajectory
    (simulate.py:415-438); runs the kernel's step function on one lane."""
    if grid.has_nodata():
        raise SimulationError("simulation requires a gap-free grid")
    if not grid.contains(start[0], start[1]):
        raise SimulationError(f"start {start} outside grid extent")
    key = stream.key if stream is not None else rng.derive_key(params.seed, 0, 0)
    positions, code = trace(grid, start, params, key, grid.cellsize)
    return Trajectory(positions=positions, stop_reason=_REASON_BY_CODE[code])


def trace(grid: DemGrid, start: tuple[float, float], params: AvalancheParams, key: int,
          step: float) -> tuple[np.ndarray, int]:
    """One particle's path on the device (wg_trace_particle): (positions, stop code)."""
    L = _lib.lib()
    sc = kernel_scalars(grid, params)
    cap = int(sc.max_steps) + 2
    path = _device.empty((cap, 2), torch.float64)
    meta = _device.zeros((2,), torch.int64)
    _lib.check(
        L.wg_trace_particle(_lib.ptr(grid.device_elevations()), *_sc_args(sc), float(step), float(start[0]),
                            float(start[1]), int(key), _lib.ptr(path), cap, _lib.ptr(meta), _lib.stream_ptr()),
        ParamError,
    )
    n, code = meta.tolist()
    return path[:n].cpu().numpy(), code


def particle_records(
    grid: DemGrid, mask: ReleaseMask, params: AvalancheParams, lo: int, hi: int
) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Per-particle (stop reason code, steps, end position) for global
    particle indices [lo, hi): the trajectory-endpoint parity artefact."""
    L = _lib.lib()
    sc = kernel_scalars(grid, params)
    cells = release_cells(mask)
    n = hi - lo
    reason = _device.empty((n,), torch.int8)
    steps = _device.empty((n,), torch.int64)
    ends = _device.empty((n, 2), torch.float64)
    scratch = _device.empty((int(L.wg_avalanche_scratch_bytes(params.particles_per_release_cell, lo, hi)),),
                            torch.uint8)
    _lib.check(
        L.wg_particle_records(_lib.ptr(grid.device_elevations()), *_sc_args(sc), _lib.ptr(cells),
                              params.particles_per_release_cell, rng.seed_word(params.seed), int(lo), int(hi),
                              _lib.ptr(reason), _lib.ptr(steps), _lib.ptr(ends), _lib.ptr(scratch),
                              _lib.stream_ptr()),
        ParamError,
    )
    return reason.cpu().numpy(), steps.cpu().numpy(), ends.cpu().numpy()


def released_particles(mask: ReleaseMask, params: AvalancheParams) -> int:
    return mask.count * params.particles_per_release_cell


def total_particle_steps(raster: RunoutRaster, released: int) -> int:
    """Every hit beyond the per-particle release visit is one advance
    (simulate.py:511-514)."""
    return int(raster.total_hits) - released


# -- snow cover ------------------------------------------------------------


def _snow_scalars(params: SnowParams) -> tuple[float, float, float, float]:
    # simulate.py:525-536, evaluated with Python floats
    base = params.snow_line_m - params.altitude_blend_m
    alt_div = max(params.altitude_blend_m, 1e-6)
    top = params.max_steepness_deg + params.steepness_blend_deg
    sl_div = max(params.steepness_blend_deg, 1e-6)
    return float(base), float(alt_div), float(top), float(sl_div)


def snow_alpha(z, slope_deg, params: SnowParams) -> np.ndarray:
    """Snow opacity (simulate.py:520-537) on the device; host uint8 result."""
    zt = _device.as_device_tensor(z, torch.float64)
    st = _device.as_device_tensor(slope_deg, torch.float64)
    px = _snow_pixels(zt, st, params, False, 0.0)
    return _device.host_view(px[..., 3].contiguous())


def _snow_pixels(z: torch.Tensor, s: torch.Tensor, params: SnowParams, has_nodata: bool, nodata: float):
    L = _lib.lib()
    out = _device.empty(tuple(z.shape) + (4,), torch.uint8)
    base, alt_div, top, sl_div = _snow_scalars(params)
    _lib.check(
        L.wg_snow(_lib.ptr(z), _lib.ptr(s), z.numel(), base, alt_div, top, sl_div, int(has_nodata), float(nodata),
                  _lib.ptr(out), _lib.stream_ptr()),
        ParamError,
    )
    return out


def compute_snow(grid: DemGrid, normals: NormalField, params: SnowParams) -> OverlayTexture:
    """White snow overlay (simulate.py:540-545)."""
    return compute_snow_from_slope(grid, steepness_deg(normals), params)


def compute_snow_from_slope(grid: DemGrid, slope: SlopeField, params: SnowParams) -> OverlayTexture:
    """compute_snow for callers holding the steepness field (simulate.py:548-560);
    one fused device pass writes the RGBA texture."""
    px = _snow_pixels(grid.device_elevations(), slope.dev("slope_deg"), params, grid.has_nodata(),
                      float(grid.nodata))
    return OverlayTexture(px)


def scale_particles(params: AvalancheParams, particles: int) -> AvalancheParams:
    return replace(params, particles_per_release_cell=particles)

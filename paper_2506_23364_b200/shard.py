"""Multi-GPU trajectory sharding and the tile-sparse overlay merge.

Particles are pure functions of (DEM, key(seed, k, p)), and the overlay merge
is an integer sum plus a float64 max -- exact, associative, commutative -- so
any partition of the particle index space yields the bitwise-identical
raster (the reference's own thread-invariance contract, simulate.py:449-453,
489-503).

Partition: the grid's rows are cut into about ``nranks * bands_per_rank``
bands of a power-of-two number of rows (whole tiles); band b belongs to rank
b % nranks (cyclic, so terrain that is steep in one region spreads over all
ranks).  A rank simulates the
particles released in its bands -- release cells are numbered row-major, so
a band's particles are one contiguous range of the global particle index,
and a rank's share is a few ranges (csrc/traj.cu ``ranges``).

Merge: a particle travels ~80 cells, so a rank's visits stay in and near its
own bands.  The trajectory kernel marks every tile (64 x 64 cells) of
another rank's bands that a visit lands in; after the run each rank packs
those tiles, one NCCL all-to-all moves them to their owners, and the owners
add / max them into their rasters (csrc/merge.cu).  The owners' bands
then hold the exact single-GPU raster; nothing else moves.  ``gather_bands``
gives every rank the whole raster (the reference API's result) when a caller
needs it.  Under the gloo backend (CPU tests, several ranks on one GPU) the
collectives run on host copies.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

TILE_LOG2 = 6  # 64 x 64-cell tiles: 32 KiB of hits + 32 KiB of drops
BANDS_PER_RANK = 4


@dataclass(frozen=True)
class BandPlan:
    """Row bands of a (nrows, ncols) grid over nranks ranks."""

    nrows: int
    ncols: int
    nranks: int
    band_rows: int  # a power of two, a multiple of the tile height
    tile_log2: int = TILE_LOG2

    @property
    def band_log2(self) -> int:
        return self.band_rows.bit_length() - 1

    @property
    def nbands(self) -> int:
        return -(-self.nrows // self.band_rows)

    @property
    def tile(self) -> int:
        return 1 << self.tile_log2

    @property
    def tiles_x(self) -> int:
        return -(-self.ncols // self.tile)

    @property
    def tiles_y(self) -> int:
        return -(-self.nrows // self.tile)

    def owner(self, band: int) -> int:
        return band % self.nranks

    def rows(self, band: int) -> tuple[int, int]:
        r0 = band * self.band_rows
        return r0, min(self.nrows, r0 + self.band_rows)

    def owned_bands(self, rank: int) -> list[int]:
        return list(range(rank, self.nbands, self.nranks))

    def tile_bounds(self) -> list[int]:
        """First tile id of every band, plus the tile count (bands are whole tile rows)."""
        per = self.band_rows >> self.tile_log2
        return [min(b * per, self.tiles_y) * self.tiles_x for b in range(self.nbands)] + [self.tiles_y * self.tiles_x]

    def cell_bounds(self) -> list[int]:
        """First flat cell index of every band, plus the cell count."""
        return [self.rows(b)[0] * self.ncols for b in range(self.nbands)] + [self.nrows * self.ncols]


def plan_bands(nrows: int, ncols: int, nranks: int, bands_per_rank: int = BANDS_PER_RANK,
               tile_log2: int = TILE_LOG2) -> BandPlan:
    """Bands of the smallest power-of-two height (>= one tile) that makes at
    most nranks * bands_per_rank of them."""
    per = -(-nrows // (nranks * bands_per_rank))
    rows = 1 << max(tile_log2, (per - 1).bit_length())
    return BandPlan(nrows, ncols, nranks, rows, tile_log2)


def particle_ranges(cell_offsets: list[int], plan: BandPlan, rank: int, per_cell: int) -> list[tuple[int, int]]:
    """The global particle ranges of `rank`: cell_offsets[b] = ordinal of the
    first release cell at or below band b's first row (row-major order),
    cell_offsets[nbands] = the release-cell count."""
    out = []
    for b in plan.owned_bands(rank):
        lo, hi = cell_offsets[b] * per_cell, cell_offsets[b + 1] * per_cell
        if hi > lo:
            out.append((lo, hi))
    return out or [(0, 0)]


def exchange_segments(tile_offsets: list[int], plan: BandPlan, rank: int):
    """Send plan of `rank`'s touched-tile list (sorted tile ids; tile_offsets
    = band offsets into it): (segs, counts) with segs = (src_off, dst_off,
    count) triples grouping the foreign tiles by destination rank, and
    counts[d] = tiles sent to rank d (0 for itself)."""
    segs, counts = [], [0] * plan.nranks
    dst = 0
    for d in range(plan.nranks):
        if d == rank:
            continue
        for b in range(d, plan.nbands, plan.nranks):
            n = tile_offsets[b + 1] - tile_offsets[b]
            if n > 0:
                segs.append((tile_offsets[b], dst, n))
                dst += n
                counts[d] += n
    return segs, counts


# ---- device helpers ------------------------------------------------------------


def _sorted_offsets(ids: torch.Tensor, n: int, bounds: list[int]) -> list[int]:
    from . import _device, _lib

    L = _lib.lib()
    b = torch.tensor(bounds, dtype=torch.int64).to(ids.device, non_blocking=True)
    out = torch.empty(len(bounds), dtype=torch.int64, device=ids.device)
    _lib.check(L.wg_sorted_offsets(_lib.ptr(ids), int(n), _lib.ptr(b), len(bounds), _lib.ptr(out),
                                   _lib.stream_ptr()))
    return [int(v) for v in _device.read_small(out)]


def band_cell_offsets(cells: torch.Tensor, plan: BandPlan) -> list[int]:
    """Release-cell ordinal offsets of the bands (cells: the row-major list)."""
    return _sorted_offsets(cells, cells.numel(), plan.cell_bounds())


def touched_tiles(touched: torch.Tensor) -> tuple[torch.Tensor, int]:
    """Sorted ids of the touched tiles (device) and their count."""
    from . import _device, _lib

    L = _lib.lib()
    m = touched.reshape(-1)
    n = m.numel()
    ids = torch.empty(max(n, 1), dtype=torch.int64, device=m.device)
    count = torch.zeros(1, dtype=torch.int64, device=m.device)
    scratch = torch.empty(int(L.wg_compact_scratch_bytes(n)), dtype=torch.uint8, device=m.device)
    _lib.check(L.wg_mask_compact(_lib.ptr(m), n, _lib.ptr(ids), _lib.ptr(count), _lib.ptr(scratch),
                                 _lib.stream_ptr()))
    return ids, int(_device.read_small(count)[0])


def pack_foreign(hits: torch.Tensor, zmax: torch.Tensor, touched: torch.Tensor, plan: BandPlan, rank: int):
    """(counts, ids, data): this rank's touched tiles (all in other ranks'
    bands), grouped by destination rank; data holds a 2*T*T-word block per
    tile."""
    from . import _lib

    L = _lib.lib()
    ids, n = touched_tiles(touched)
    toffs = _sorted_offsets(ids, n, plan.tile_bounds())
    segs, counts = exchange_segments(toffs, plan, rank)
    nout = sum(counts)
    words = 2 * plan.tile * plan.tile
    out_ids = torch.empty(max(nout, 1), dtype=torch.int64, device=hits.device)
    data = torch.empty((max(nout, 1), words), dtype=torch.int64, device=hits.device)
    if nout:
        seg_t = torch.tensor(segs, dtype=torch.int64).reshape(-1).to(hits.device, non_blocking=True)
        _lib.check(L.wg_tiles_pack(_lib.ptr(hits), _lib.ptr(zmax), plan.nrows, plan.ncols, plan.tile_log2,
                                   _lib.ptr(ids), _lib.ptr(seg_t), len(segs), nout, _lib.ptr(out_ids),
                                   _lib.ptr(data), _lib.stream_ptr()))
    return counts, out_ids[:nout], data[:nout]


def accumulate_tiles(hits: torch.Tensor, zmax: torch.Tensor, plan: BandPlan, ids: torch.Tensor,
                     data: torch.Tensor) -> None:
    from . import _lib

    if ids.numel() == 0:
        return
    L = _lib.lib()
    _lib.check(L.wg_tiles_accumulate(_lib.ptr(hits), _lib.ptr(zmax), plan.nrows, plan.ncols, plan.tile_log2,
                                     _lib.ptr(ids), ids.numel(), _lib.ptr(data), _lib.stream_ptr()))


def clear_tiles(hits: torch.Tensor, zmax: torch.Tensor, touched: torch.Tensor, plan: BandPlan, rank: int) -> None:
    """Make a rank's rasters zero again for the next run without a
    full-raster memset: its own bands (1/N of the raster) and the foreign
    tiles it touched; then the touched map."""
    from . import _lib

    for b in plan.owned_bands(rank):
        r0, r1 = plan.rows(b)
        hits[r0:r1].zero_()
        zmax[r0:r1].zero_()
    ids, n = touched_tiles(touched)
    if n:
        L = _lib.lib()
        _lib.check(L.wg_tiles_zero(_lib.ptr(hits), _lib.ptr(zmax), plan.nrows, plan.ncols, plan.tile_log2,
                                   _lib.ptr(ids), n, _lib.stream_ptr()))
    touched.zero_()


# ---- collectives ---------------------------------------------------------------


def _world(group) -> tuple[int, int]:
    return dist.get_rank(group), dist.get_world_size(group)


def _on_host(group) -> bool:
    return dist.get_backend(group) != "nccl"


def _all_to_all(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group) -> torch.Tensor:
    if _on_host(group):
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), list(out_splits), list(in_splits), group=group)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, list(out_splits), list(in_splits), group=group)
    return out


def merge_tiles(hits: torch.Tensor, zmax: torch.Tensor, touched: torch.Tensor, plan: BandPlan, group=None) -> dict:
    """Send this rank's foreign touched tiles to their owners and fold the
    tiles received into its own bands; returns the traffic counts."""
    rank, world = _world(group)
    counts, ids, data = pack_foreign(hits, zmax, touched, plan, rank)
    dev = hits.device
    cin = torch.tensor(counts, dtype=torch.int64)
    cout = torch.empty(world, dtype=torch.int64)
    if _on_host(group):
        dist.all_to_all_single(cout, cin, group=group)
    else:
        c = cin.to(dev)
        co = torch.empty_like(c)
        dist.all_to_all_single(co, c, group=group)
        cout = co.cpu()
    recv = [int(v) for v in cout.tolist()]
    nrecv = sum(recv)
    words = data.shape[1] if data.dim() == 2 else 2 * plan.tile * plan.tile
    rids = torch.empty(nrecv, dtype=torch.int64, device=dev)
    rdata = torch.empty((nrecv, words), dtype=torch.int64, device=dev)
    _all_to_all(rids, ids, recv, counts, group)
    _all_to_all(rdata, data.reshape(-1, words), recv, counts, group)
    accumulate_tiles(hits, zmax, plan, rids, rdata)
    tile_bytes = words * 8
    return {"sent_tiles": sum(counts), "recv_tiles": nrecv, "sent_bytes": sum(counts) * tile_bytes,
            "dense_bytes": plan.nrows * plan.ncols * 16}


def band_stats(hits: torch.Tensor, zmax: torch.Tensor, plan: BandPlan, group=None) -> tuple[int, int, float]:
    """(total hits, cells hit, max drop) of the merged raster: each rank's
    stats pass over its own bands, then one all-reduce of the scalars."""
    from . import _device, _lib
    from .simulate import SimulationError

    rank, world = _world(group)
    L = _lib.lib()
    out = torch.zeros(4, dtype=torch.int64, device=hits.device)
    for b in plan.owned_bands(rank):
        r0, r1 = plan.rows(b)
        _lib.check(L.wg_runout_stats(_lib.ptr(hits[r0:r1]), _lib.ptr(zmax[r0:r1]), (r1 - r0) * plan.ncols,
                                     _lib.ptr(out), _lib.stream_ptr()), SimulationError)
    s, nnz, zb, bad = _device.read_small(out)
    v = torch.tensor([s, nnz, bad], dtype=torch.int64)
    m = torch.tensor([zb], dtype=torch.int64)
    if not _on_host(group):
        v, m = v.to(hits.device), m.to(hits.device)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)  # non-negative doubles order like their bits
    s, nnz, bad = (int(x) for x in v.tolist())
    if bad:
        raise SimulationError("invalid runout raster")
    return s, nnz, float(np.array([int(m.item())], dtype=np.int64).view(np.float64)[0])


def gather_bands(hits: torch.Tensor, zmax: torch.Tensor, plan: BandPlan, group=None) -> None:
    """Every rank receives every band from its owner (the full raster)."""
    for b in range(plan.nbands):
        r0, r1 = plan.rows(b)
        src = plan.owner(b)
        for t in (hits[r0:r1], zmax[r0:r1]):
            if _on_host(group):
                h = t.cpu()
                dist.broadcast(h, src, group=group)
                t.copy_(h)
            else:
                dist.broadcast(t, src, group=group)


@dataclass
class ShardedRun:
    """One rank's rasters after the merge: its own bands are final."""

    hits: torch.Tensor
    zmax: torch.Tensor
    touched: torch.Tensor
    plan: BandPlan
    ranges: list
    traffic: dict


def run_sharded(grid, cells: torch.Tensor, params, group=None, plan: BandPlan | None = None,
                hits: torch.Tensor | None = None, zmax: torch.Tensor | None = None,
                touched: torch.Tensor | None = None) -> ShardedRun:
    """This rank's bands of run_avalanche(grid, cells) (simulate.py:441-504):
    its particles into private rasters (zeroed, or given zeroed), then the
    tile-sparse merge.  Every rank passes the same grid and cell list."""
    from . import _device
    from .simulate import run_avalanche_device

    rank, world = _world(group)
    if plan is None:
        plan = plan_bands(grid.nrows, grid.ncols, world)
    if hits is None:
        hits = _device.zeros((grid.nrows, grid.ncols), torch.int64)
    if zmax is None:
        zmax = _device.zeros((grid.nrows, grid.ncols), torch.float64)
    if touched is None:
        touched = _device.zeros((plan.tiles_y, plan.tiles_x), torch.uint8)
    ranges = particle_ranges(band_cell_offsets(cells, plan), plan, rank, params.particles_per_release_cell)
    run_avalanche_device(grid, cells, params, ranges=ranges, hits=hits, zmax=zmax, touched=touched, plan=plan,
                         rank=rank)
    traffic = merge_tiles(hits, zmax, touched, plan, group)
    return ShardedRun(hits, zmax, touched, plan, ranges, traffic)


def local_particles(ranges: list[tuple[int, int]]) -> int:
    return sum(hi - lo for lo, hi in ranges)


# ---- the sharded upstream (bench N > 1) -----------------------------------------


def band_rows(nrows: int, stride: int, rank: int, nranks: int) -> tuple[int, int]:
    """Row band [r0, r1) of `rank` for the upstream nodes: equal shares
    rounded up to a multiple of the release lattice stride, so each band's
    first row is a lattice row."""
    per = -(-nrows // nranks)
    per = -(-per // stride) * stride
    r0 = min(nrows, rank * per)
    return r0, min(nrows, r0 + per)


def release_cells_banded(grid, min_deg: float, max_deg: float, stride: int, rank: int, nranks: int,
                         with_normals: bool = True, group=None) -> torch.Tensor:
    """Global release-cell list (row-major, == release_cells(detect_release_
    points(steepness(normals(grid)), ...))) with the upstream nodes sharded
    by row band: each rank computes normals + slope for its band (one halo
    row on each side, so interior band edges use central differences exactly
    like the full grid and global edges the one-sided rule), its band of the
    release mask and its cells; the per-band lists are all-gathered in rank
    (= row) order.  Bit-identical to the unsharded prefix."""
    from . import _device, _lib
    from .terrain import TerrainError

    if grid.has_nodata():
        raise TerrainError("normals require a gap-free grid (nodata present)")
    L = _lib.lib()
    H, W = grid.nrows, grid.ncols
    r0, r1 = band_rows(H, stride, rank, nranks)
    e = grid.device_elevations()
    local = torch.empty(0, dtype=torch.int64, device=e.device)
    if r1 > r0:
        a, b = max(r0 - 1, 0), min(r1 + 1, H)
        sub = e[a:b]
        cs = grid.cellsize
        mask = _device.empty((r1 - r0, W), torch.uint8)
        if with_normals:
            slope = _device.empty((b - a, W), torch.float64)
            nrm = _device.empty((b - a, W, 3), torch.float64)
            _lib.check(L.wg_normals(_lib.ptr(sub), b - a, W, cs, 2.0 * cs, _lib.ptr(nrm), _lib.ptr(slope),
                                    _lib.stream_ptr()), TerrainError)
            band = slope[r0 - a : r1 - a]
            _lib.check(L.wg_release_mask(_lib.ptr(band), r1 - r0, W, float(min_deg), float(max_deg), int(stride),
                                         _lib.ptr(mask), None, _lib.stream_ptr()))
        else:  # the slope at lattice cells only, straight from the band + halo rows
            _lib.check(L.wg_lattice_release_mask(_lib.ptr(sub), b - a, W, cs, 2.0 * cs, float(min_deg),
                                                 float(max_deg), int(stride), r0 - a, r1 - a, _lib.ptr(mask),
                                                 None, _lib.stream_ptr()), TerrainError)
        n = mask.numel()
        cells = _device.empty((max(n, 1),), torch.int64)
        count = _device.zeros((1,), torch.int64)
        scratch = _device.empty((int(L.wg_compact_scratch_bytes(n)),), torch.uint8)
        _lib.check(L.wg_mask_compact(_lib.ptr(mask), n, _lib.ptr(cells), _lib.ptr(count), _lib.ptr(scratch),
                                     _lib.stream_ptr()))
        k = int(_device.read_small(count)[0])
        local = cells[:k] + r0 * W
    sizes_t = torch.tensor([local.numel()], dtype=torch.int64)
    if _on_host(group):
        parts_sz = [torch.zeros_like(sizes_t) for _ in range(nranks)]
        dist.all_gather(parts_sz, sizes_t, group=group)
    else:
        st = sizes_t.to(e.device)
        parts_sz = [torch.zeros_like(st) for _ in range(nranks)]
        dist.all_gather(parts_sz, st, group=group)
    sizes = [int(c.item()) for c in parts_sz]
    m = max(sizes) if sizes else 0
    if m == 0:
        return torch.empty(0, dtype=torch.int64, device=e.device)
    padded = torch.zeros(m, dtype=torch.int64, device=e.device)
    padded[: local.numel()] = local
    if _on_host(group):
        padded = padded.cpu()
    parts = [torch.zeros_like(padded) for _ in range(nranks)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)]).to(e.device)


def merge_runout(hits: torch.Tensor, zmax: torch.Tensor, group=None, dst: int | None = None) -> None:
    """Dense merge of whole private rasters (hits SUM, drops MAX) -- the
    baseline the tile-sparse merge replaces; kept for callers holding
    rasters of arbitrary particle subsets."""
    if dst is None:
        dist.all_reduce(hits, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(zmax, op=dist.ReduceOp.MAX, group=group)
    else:
        dist.reduce(hits, dst, op=dist.ReduceOp.SUM, group=group)
        dist.reduce(zmax, dst, op=dist.ReduceOp.MAX, group=group)

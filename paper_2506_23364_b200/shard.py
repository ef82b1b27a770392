"""Multi-GPU trajectory sharding.

Particles are pure functions of (DEM, key(seed, k, p)), and the overlay merge
is an integer sum plus a float64 max -- exact, associative, commutative -- so
any partition of the particle index space yields the bitwise-identical
raster.  Each rank runs the trajectory kernel on its blocked-cyclic share of
release-point blocks (csrc/traj.cu, ``rank``/``nranks``/``shard_block``)
into a private int64 hit raster and float64 drop raster; this module merges
them with one NCCL all-reduce (or reduce to one rank) each (SUM for hits,
MAX for drops) over NVLink/NVSwitch.  Under the gloo backend (CPU tests) the same calls run on
host tensors.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def block_owner(block: int, nranks: int) -> int:
    """Rank owning shard block `block` (blocked-cyclic; mirrors traj.cu start())."""
    return block % nranks


def local_particles(total: int, block: int, rank: int, nranks: int) -> int:
    """Number of particles of [0, total) that `rank` simulates (traj.cu launch_traj)."""
    nb = (total + block - 1) // block
    if rank >= nb:
        return 0
    owned = (nb - rank + nranks - 1) // nranks
    n = owned * block
    if (nb - 1) % nranks == rank:
        n -= nb * block - total
    return n


def local_indices(total: int, block: int, rank: int, nranks: int) -> list[range]:
    """The particle index ranges `rank` owns, in claim order."""
    out = []
    for b in range(rank, (total + block - 1) // block, nranks):
        out.append(range(b * block, min((b + 1) * block, total)))
    return out


def merge_runout(hits: torch.Tensor, zmax: torch.Tensor, group=None, dst: int | None = None) -> None:
    """In-place merge of one rank's private rasters: hits SUM, drops MAX.
    All ranks receive the result (all-reduce), or only rank `dst` (reduce:
    half the NVLink traffic when one rank colorizes the overlay, as the
    reference's single process does)."""
    if dst is None:
        dist.all_reduce(hits, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(zmax, op=dist.ReduceOp.MAX, group=group)
    else:
        dist.reduce(hits, dst, op=dist.ReduceOp.SUM, group=group)
        dist.reduce(zmax, dst, op=dist.ReduceOp.MAX, group=group)


def band_rows(nrows: int, stride: int, rank: int, nranks: int) -> tuple[int, int]:
    """Row band [r0, r1) of `rank`: equal shares rounded up to a multiple of
    the release lattice stride, so each band's first row is a lattice row."""
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
                                         _lib.ptr(mask), _lib.stream_ptr()))
        else:  # the slope at lattice cells only, straight from the band + halo rows
            _lib.check(L.wg_lattice_release_mask(_lib.ptr(sub), b - a, W, cs, 2.0 * cs, float(min_deg),
                                                 float(max_deg), int(stride), r0 - a, r1 - a, _lib.ptr(mask),
                                                 _lib.stream_ptr()), TerrainError)
        n = mask.numel()
        cells = _device.empty((max(n, 1),), torch.int64)
        count = _device.zeros((1,), torch.int64)
        scratch = _device.empty((int(L.wg_compact_scratch_bytes(n)),), torch.uint8)
        _lib.check(L.wg_mask_compact(_lib.ptr(mask), n, _lib.ptr(cells), _lib.ptr(count), _lib.ptr(scratch),
                                     _lib.stream_ptr()))
        k = int(_device.read_small(count)[0])
        local = cells[:k] + r0 * W
    counts = torch.tensor([local.numel()], dtype=torch.int64, device=e.device)
    all_counts = [torch.zeros_like(counts) for _ in range(nranks)]
    dist.all_gather(all_counts, counts, group=group)
    sizes = [int(c.item()) for c in all_counts]
    m = max(sizes) if sizes else 0
    if m == 0:
        return torch.empty(0, dtype=torch.int64, device=e.device)
    padded = torch.zeros(m, dtype=torch.int64, device=e.device)
    padded[: local.numel()] = local
    parts = [torch.zeros_like(padded) for _ in range(nranks)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])

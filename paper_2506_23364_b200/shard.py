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

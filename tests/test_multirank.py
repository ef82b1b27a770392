"""World-size-2 gloo run of the multi-GPU merge path on the CPU: each rank
simulates its blocked-cyclic share of the particles (the CPU oracle stands in
for its GPU), merges with shard.merge_runout (the all-reduce the NCCL path
uses), and the merged raster must equal the single-process run bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, elev, mask, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import traj
        from paper_2506_23364_b200.shard import local_indices, merge_runout

        cells = np.ascontiguousarray(np.flatnonzero(mask.ravel()), dtype=np.int64)
        ppc = 96
        total = cells.size * ppc
        hits = np.zeros(elev.shape, dtype=np.int64)
        zmax = np.zeros(elev.shape, dtype=np.float64)
        for rg in local_indices(total, 256, rank, world):
            traj.run_range(elev, 0.0, 0.0, 10.0, cells, rg.start, rg.stop, hits, zmax, particles_per_release_cell=ppc,
                           seed=4, threads=2)
        h, z = torch.from_numpy(hits), torch.from_numpy(zmax)
        h2, z2 = h.clone(), z.clone()
        merge_runout(h, z)  # all-reduce: every rank holds the merged raster
        merge_runout(h2, z2, dst=0)  # reduce: rank 0 only (the bench's N>1 path)
        if rank == 0:
            out.put((h.numpy().copy(), z.numpy().copy(), h2.numpy().copy(), z2.numpy().copy()))
        else:
            out.put((h.numpy().copy(), z.numpy().copy(), None, None))
    finally:
        dist.destroy_process_group()


def test_two_rank_merge_equals_single_run():
    from oracle import traj
    from paper_2506_23364_b200.synth import synth_dem_host

    elev = synth_dem_host(192, 2)
    mask = np.zeros(elev.shape, dtype=bool)
    mask[::12, ::12] = True
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, elev, mask, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    z1, h1 = traj.run_avalanche(elev, 0.0, 0.0, 10.0, mask, particles_per_release_cell=96, seed=4)
    for h, z, h2, z2 in got:  # all-reduce: both ranks
        assert np.array_equal(h, h1)
        assert np.array_equal(z.view(np.int64), z1.view(np.int64))
    roots = [(h2, z2) for _, _, h2, z2 in got if h2 is not None]
    assert len(roots) == 1  # reduce: the root's rasters
    assert np.array_equal(roots[0][0], h1)
    assert np.array_equal(roots[0][1].view(np.int64), z1.view(np.int64))

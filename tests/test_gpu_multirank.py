"""The banded (rank-sharded) upstream of the multi-GPU bench path --
normals/slope/mask per row band with halos, cell lists all-gathered -- equals
the unsharded release-cell list, on the GPU with 2 and 3 ranks sharing one
device over gloo (NCCL refuses two ranks per device)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, e, stride, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_23364_b200 as wf
        from paper_2506_23364_b200.shard import release_cells_banded

        torch.cuda.set_device(0)
        g = wf.DemGrid(e.shape[1], e.shape[0], 0.0, 0.0, 10.0, -9999.0, e)
        cells = release_cells_banded(g, 30.0, 45.0, stride, rank, world)
        out.put((rank, cells.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,stride,shape", [(2, 32, (1000, 777)), (3, 7, (301, 450))])
def test_banded_release_cells_equal_full(gpu, world, stride, shape):
    import paper_2506_23364_b200 as wf
    from paper_2506_23364_b200.simulate import release_cells
    from paper_2506_23364_b200.synth import synth_dem_host

    e = synth_dem_host(max(shape), 3)[: shape[0], : shape[1]].copy()
    g = wf.DemGrid(shape[1], shape[0], 0.0, 0.0, 10.0, -9999.0, e)
    want = release_cells(wf.detect_release_points(wf.steepness_deg(wf.compute_normals(g)), 30.0, 45.0, stride))
    want = want.cpu().numpy()
    assert want.size > 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, e, stride, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, cells in got:
        assert np.array_equal(cells, want)


def _sharded_worker(rank, world, port, e, mask, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_23364_b200 as wf
        from paper_2506_23364_b200 import shard
        from paper_2506_23364_b200.simulate import release_cells

        torch.cuda.set_device(0)
        g = wf.DemGrid(e.shape[1], e.shape[0], 0.0, 0.0, 10.0, -9999.0, e)
        params = wf.AvalancheParams(particles_per_release_cell=128, seed=9)
        m = wf.ReleaseMask(mask)
        cells = release_cells(m)
        run = shard.run_sharded(g, cells, params, group=None, plan=shard.plan_bands(e.shape[0], e.shape[1], world,
                                                                                       3, 5))
        stats = shard.band_stats(run.hits, run.zmax, run.plan)
        bands = {b: (run.hits[slice(*run.plan.rows(b))].cpu().numpy(), run.zmax[slice(*run.plan.rows(b))].cpu().numpy())
                 for b in run.plan.owned_bands(rank)}
        full = wf.run_avalanche(g, m, params, group=dist.group.WORLD)  # the public opt-in API
        out.put((rank, bands, stats, run.traffic, full.hit_count.copy(), full.z_delta_max.copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_run_and_api_equal_single_gpu(gpu, world):
    """run_sharded (band partition + touched tiles + all-to-all merge) with
    `world` ranks on one GPU over gloo: each owner's bands, the all-reduced
    stats and the public run_avalanche(group=...) equal the single run."""
    import paper_2506_23364_b200 as wf
    from paper_2506_23364_b200.synth import synth_dem_host

    e = synth_dem_host(400, 6)[:, :350].copy()
    mask = np.zeros(e.shape, dtype=bool)
    mask[::9, ::9] = True
    g = wf.DemGrid(e.shape[1], e.shape[0], 0.0, 0.0, 10.0, -9999.0, e)
    params = wf.AvalancheParams(particles_per_release_cell=128, seed=9)
    want = wf.run_avalanche(g, wf.ReleaseMask(mask), params)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, e, mask, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2506_23364_b200 import shard

    plan = shard.plan_bands(e.shape[0], e.shape[1], world, 3, 5)
    seen = set()
    for rank, bands, stats, traffic, fh, fz in got:
        assert stats == (want.total_hits, want.cells_hit, want.z_max)
        assert 0 < traffic["sent_bytes"] < traffic["dense_bytes"]
        assert np.array_equal(fh, want.hit_count) and np.array_equal(fz.view(np.int64), want.z_delta_max.view(np.int64))
        for b, (h, z) in bands.items():
            r0, r1 = plan.rows(b)
            assert np.array_equal(h, want.hit_count[r0:r1])
            assert np.array_equal(z.view(np.int64), want.z_delta_max[r0:r1].view(np.int64))
            seen.add(b)
    assert seen == set(range(plan.nbands))

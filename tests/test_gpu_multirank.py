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

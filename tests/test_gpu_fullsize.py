"""Parity at BASELINE's full size (C3: synth_dem(16384, 0), band 30-45 deg,
stride 32, 2048 particles per release cell = 1.9e8 particles, 1.0e10 steps)
through size-independent properties and sampled oracle checks:

* accounting: the accumulating kernel's hit total == released particles +
  the per-particle step counts of the independent records kernel;
* shard composition: two blocked-cyclic shards (the multi-GPU split) sum /
  max to the single run bit for bit;
* sampled oracle: 128 evenly spaced 2048-particle chunks -- per-particle
  stop reason, step count and end point, and the chunks' accumulated rasters
  -- equal the C oracle (oracle/traj_oracle.c) bit for bit."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N, STRIDE, PPC, SEED = 16384, 32, 2048, 0


@pytest.fixture(scope="module")
def c3(gpu):
    import paper_2506_23364_b200 as wf
    from paper_2506_23364_b200.simulate import release_cells
    from paper_2506_23364_b200.synth import synth_dem_device
    from paper_2506_23364_b200.terrain import compute_normals_and_slope

    grid = wf.DemGrid(N, N, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(N, SEED))
    _, slope = compute_normals_and_slope(grid)
    mask = wf.detect_release_points(slope, 30.0, 45.0, STRIDE)
    cells = release_cells(mask)
    params = wf.AvalancheParams(particles_per_release_cell=PPC, seed=SEED)
    return wf, grid, mask, cells, params


def test_fullsize_accounting_and_shards(c3):
    wf, grid, mask, cells, params = c3
    from paper_2506_23364_b200.simulate import particle_records, run_avalanche_device

    total = int(cells.numel()) * PPC
    assert total > 1.5e8
    hits, zmax = run_avalanche_device(grid, cells, params)
    torch.cuda.synchronize()
    hit_total = int(hits.sum().item())
    _, steps, _ = particle_records(grid, mask, params, 0, total)
    assert hit_total == total + int(steps.sum())
    assert hit_total - total > 9e9
    h0, z0 = run_avalanche_device(grid, cells, params, rank=0, nranks=2, shard_block=2048)
    h1, z1 = run_avalanche_device(grid, cells, params, rank=1, nranks=2, shard_block=2048)
    assert torch.equal(h0 + h1, hits)
    assert torch.equal(torch.maximum(z0, z1), zmax)


def test_fullsize_sampled_chunks_match_oracle(c3):
    wf, grid, mask, cells, params = c3
    from oracle import traj

    from paper_2506_23364_b200.simulate import particle_records, run_avalanche_device

    total = int(cells.numel()) * PPC
    nchunks = total // PPC
    picks = np.linspace(0, nchunks - 1, 128).astype(np.int64)
    elev = grid.device_elevations().cpu().numpy()
    cells_h = cells.cpu().numpy().astype(np.int64)
    oh = np.zeros((N, N), dtype=np.int64)
    oz = np.zeros((N, N), dtype=np.float64)
    gh = torch.zeros((N, N), dtype=torch.int64, device="cuda")
    gz = torch.zeros((N, N), dtype=torch.float64, device="cuda")
    for c in picks:
        lo, hi = int(c) * PPC, int(c + 1) * PPC
        rr, st, en = particle_records(grid, mask, params, lo, hi)
        _, (orr, ost, oen) = traj.run_range(elev, 0.0, 0.0, 10.0, cells_h, lo, hi, oh, oz,
                                            particles_per_release_cell=PPC, seed=SEED, records=True)
        assert np.array_equal(rr, orr) and np.array_equal(st, ost)
        assert np.array_equal(en.view(np.int64), oen.view(np.int64))
        run_avalanche_device(grid, cells, params, i_lo=lo, i_hi=hi, hits=gh, zmax=gz)
    assert torch.equal(gh, torch.from_numpy(oh).cuda())
    assert torch.equal(gz.view(torch.int64), torch.from_numpy(oz).cuda().view(torch.int64))


def test_readme_example(gpu):
    """The README's usage snippet runs as written."""
    import paper_2506_23364_b200 as wf

    grid, mask = wf.gen_parabola()
    graph = wf.build_avalanche_graph(grid.extent, wf.AvalancheParams(), wf.MaskRelease(wf.ReleaseMask(mask)), zoom=1)
    graph.bind("world", grid)
    res = wf.Executor().execute(graph)
    runout = res.value("avalanche_overlay", "runout")
    assert runout.total_hits == 122_870 + int(mask.sum()) * 2048
    assert res.value("avalanche_overlay", "stats")["particle_steps"] == 122_870

"""Parity at BASELINE's full size (C3: synth_dem(16384, 0), band 30-45 deg,
stride 32, 2048 particles per release cell = 1.9e8 particles, 1.0e10 steps).

* The whole run against the C oracle (oracle/traj_oracle.c, pinned to the
  reference's shipped goldens): all 92,233 release cells, every particle --
  hit_count and z_delta_max bit for bit (the oracle takes ~2 minutes on the
  box's 16 host threads).
* The release mask of the full normals -> slope -> mask chain equals the
  numpy statement of the reference's (oracle/npref.py) and its guard band
  is empty.
* Per-particle records (stop reason, steps, end point) of sampled chunks
  equal the oracle's; the accounting identity hit total == released +
  steps holds against the independent records kernel."""

import os

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

    grid = wf.DemGrid.adopt(N, N, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(N, SEED))
    _, slope = compute_normals_and_slope(grid)
    mask = wf.detect_release_points(slope, 30.0, 45.0, STRIDE)
    del slope
    cells = release_cells(mask)
    params = wf.AvalancheParams(particles_per_release_cell=PPC, seed=SEED)
    return wf, grid, mask, cells, params


def test_fullsize_mask_equals_numpy_chain(c3):
    from oracle import npref

    wf, grid, mask, cells, params = c3
    e = grid.elevations
    want = npref.lattice_release_mask(e, 10.0, 30.0, 45.0, STRIDE)
    assert np.array_equal(mask.mask, want)
    assert mask.count == int(want.sum()) == cells.numel() == 92233
    assert mask.borderline == 0


def test_fullsize_raster_equals_oracle(c3):
    """Every particle of the headline config, GPU vs the C oracle."""
    from oracle import traj

    from paper_2506_23364_b200.simulate import run_avalanche_device

    wf, grid, mask, cells, params = c3
    hits, zmax = run_avalanche_device(grid, cells, params)
    gh = hits.cpu().numpy()
    gz = zmax.cpu().numpy()
    del hits, zmax
    elev = grid.elevations
    cells_h = cells.cpu().numpy().astype(np.int64)
    oh = np.zeros((N, N), dtype=np.int64)
    oz = np.zeros((N, N), dtype=np.float64)
    total = cells_h.size * PPC
    steps = traj.run_range(elev, 0.0, 0.0, 10.0, cells_h, 0, total, oh, oz, particles_per_release_cell=PPC,
                           seed=SEED, threads=os.cpu_count())
    assert steps > 1.0e10
    assert int(oh.sum()) == total + steps
    assert np.array_equal(gh, oh), f"hit_count differs in {int((gh != oh).sum())} cells"
    assert np.array_equal(gz.view(np.int64), oz.view(np.int64)), \
        f"z_delta_max differs in {int((gz.view(np.int64) != oz.view(np.int64)).sum())} cells"


def test_fullsize_records_and_accounting(c3):
    wf, grid, mask, cells, params = c3
    from oracle import traj

    from paper_2506_23364_b200.simulate import particle_records, run_avalanche_device

    total = int(cells.numel()) * PPC
    hits, _ = run_avalanche_device(grid, cells, params)
    hit_total = int(hits.sum().item())
    del hits
    _, steps, _ = particle_records(grid, mask, params, 0, total)
    assert hit_total == total + int(steps.sum())
    nchunks = total // PPC
    elev = grid.elevations
    cells_h = cells.cpu().numpy().astype(np.int64)
    oh = np.zeros((N, N), dtype=np.int64)
    oz = np.zeros((N, N), dtype=np.float64)
    for c in np.linspace(0, nchunks - 1, 32).astype(np.int64):
        lo, hi = int(c) * PPC, int(c + 1) * PPC
        rr, st, en = particle_records(grid, mask, params, lo, hi)
        _, (orr, ost, oen) = traj.run_range(elev, 0.0, 0.0, 10.0, cells_h, lo, hi, oh, oz,
                                            particles_per_release_cell=PPC, seed=SEED, records=True)
        assert np.array_equal(rr, orr) and np.array_equal(st, ost)
        assert np.array_equal(en.view(np.int64), oen.view(np.int64))


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

"""The trajectory launch may claim release cells in any order (csrc/traj.cu:
the long-first partition on short launches); the rasters must not depend on
it.  The same runs with the order forced off and forced on
(WG_CELL_ORDER=0 / 1, read by the library at each launch) give identical
hit_count and z_delta_max bit patterns -- single-range launches, a sharded
rank's banded launch, and the C4-sized overlay world."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wf(gpu):
    import paper_2506_23364_b200 as wf

    return wf


def _with_order(flag: str, fn):
    old = os.environ.get("WG_CELL_ORDER")
    os.environ["WG_CELL_ORDER"] = flag
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["WG_CELL_ORDER"]
        else:
            os.environ["WG_CELL_ORDER"] = old


def _rasters(run):
    return run.hit_count.copy(), run.z_delta_max.view(np.int64).copy()


@pytest.mark.parametrize("n,stride,ppc,seed,randomness", [(512, 4, 64, 3, 0.16), (1024, 8, 128, 5, 0.16),
                                                          (700, 5, 33, 7, 0.7)])
def test_order_does_not_change_the_rasters(wf, n, stride, ppc, seed, randomness):
    from paper_2506_23364_b200.synth import synth_dem_host

    grid = wf.DemGrid(ncols=n, nrows=n, origin_x=0.0, origin_y=0.0, cellsize=10.0, nodata=-9999.0,
                      elevations=np.ascontiguousarray(synth_dem_host(n, seed)))
    mask = wf.detect_release_points(wf.steepness_deg(wf.compute_normals(grid)), 30.0, 45.0, stride)
    params = wf.AvalancheParams(particles_per_release_cell=ppc, seed=seed, randomness=randomness)
    off = _with_order("0", lambda: _rasters(wf.run_avalanche(grid, mask, params)))
    on = _with_order("1", lambda: _rasters(wf.run_avalanche(grid, mask, params)))
    assert np.array_equal(off[0], on[0]) and np.array_equal(off[1], on[1])
    assert off[0].sum() > mask.count * ppc  # particles moved


def test_order_does_not_change_a_banded_launch(wf):
    """A rank's share as several whole-cell ranges (release-row bands)."""
    import torch

    from paper_2506_23364_b200 import shard
    from paper_2506_23364_b200.simulate import release_cells, run_avalanche_device
    from paper_2506_23364_b200.synth import synth_dem_device

    n = 2048
    grid = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, 4))
    mask = wf.detect_release_points(wf.steepness_deg(wf.compute_normals(grid)), 30.0, 45.0, 8)
    cells = release_cells(mask)
    params = wf.AvalancheParams(particles_per_release_cell=128, seed=4)
    plan = shard.plan_bands(n, n, 4)
    ranges = shard.particle_ranges(shard.band_cell_offsets(cells, plan), plan, 1, 128)
    assert len(ranges) > 1

    def run():
        h = torch.zeros((n, n), dtype=torch.int64, device="cuda")
        z = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        run_avalanche_device(grid, cells, params, ranges=ranges, hits=h, zmax=z)
        return h.cpu().numpy(), z.view(torch.int64).cpu().numpy()

    off = _with_order("0", run)
    on = _with_order("1", run)
    assert np.array_equal(off[0], on[0]) and np.array_equal(off[1], on[1])

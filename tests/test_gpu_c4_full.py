"""C4 at full size (BASELINE configs[3]: world synth_dem(8192, 1), zoom 2 =
16 stitched tiles, band 30-45 deg, stride 16, 256 particles per release
cell = 2.4e7 particles, 1.15e9 steps; colorize + 14-level mip): the stock
avalanche graph on the B200 against the reference chain restated on the
host -- npref normals / steepness / mask, the C oracle's trajectories (all
particles), npref colorize and mipmap -- bit for bit, stats included.  (The
parity-sized variant of C4 is checked against the reference itself in
test_gpu_baseline_configs.py.)"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, STRIDE, PPC, SEED = 8192, 16, 256, 0


def test_c4_full_overlay_equals_oracle_chain(gpu):
    import paper_2506_23364_b200 as wf
    from oracle import npref, traj

    from paper_2506_23364_b200.overlay import DEFAULT_RUNOUT_COLORMAP
    from paper_2506_23364_b200.synth import synth_dem_device, synth_dem_host

    world = wf.DemGrid.adopt(N, N, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(N, 1))
    params = wf.AvalancheParams(particles_per_release_cell=PPC, seed=SEED)
    graph = wf.build_avalanche_graph(world.extent, params, wf.SteepnessRelease(30.0, 45.0, stride=STRIDE), zoom=2)
    graph.bind("world", world)
    res = wf.Executor().execute(graph)
    run = res.value("avalanche_overlay", "runout")
    pyr = res.value("avalanche_overlay", "overlay")
    stats = res.value("avalanche_overlay", "stats")

    e = synth_dem_host(N, 1)
    assert np.array_equal(world.elevations, e)
    mask = npref.release_mask(npref.steepness(npref.normals(e, 10.0)), 30.0, 45.0, STRIDE)
    assert np.array_equal(res.value("release_points", "mask").mask, mask)
    cells = np.ascontiguousarray(np.flatnonzero(mask.ravel()), dtype=np.int64)
    oh = np.zeros((N, N), dtype=np.int64)
    oz = np.zeros((N, N), dtype=np.float64)
    steps = traj.run_range(e, 0.0, 0.0, 10.0, cells, 0, cells.size * PPC, oh, oz, particles_per_release_cell=PPC,
                           seed=SEED, threads=os.cpu_count())
    assert steps > 1.0e9 and stats["particle_steps"] == steps
    assert np.array_equal(run.hit_count, oh)
    assert np.array_equal(run.z_delta_max.view(np.int64), oz.view(np.int64))
    levels = npref.mipmap(npref.colorize(oz, DEFAULT_RUNOUT_COLORMAP.stops))
    assert len(pyr.levels) == len(levels) == 14
    for got, want in zip(pyr.levels, levels):
        assert np.array_equal(got.pixels, want)

"""C5 (BASELINE configs[4]): synth_dem(65536, 2), band 30-45 deg, stride 128,
2048 particles per release cell (~2e8 particles, ~1e10 steps) -- the
multi-GPU config, checked on one B200:

* the release mask from the slope at lattice cells only (the C5 prefix:
  128 GiB of normal / slope fields never materialised) equals the numpy
  statement of the reference's normals -> steepness -> mask chain
  (oracle/npref.py, fed the DEM rows it needs) bit for bit, guard band empty;
* the 2-rank split -- release-row bands, touched-tile maps, the foreign
  tiles packed and folded into their owners (the data the NCCL all-to-all
  moves) -- gives every band of its owner the 1-rank raster bit for bit
  (per-band device digests);
* 16 evenly spaced 2048-particle chunks equal the C oracle bit for bit
  (stop reasons, steps, end points), and so does the whole run's raster
  (every particle, ~2 minutes of the oracle on the box's host threads).

HBM: DEM 32 GiB + rasters 64 GiB (+ the packed tiles); the gather layout is
held at the plain DEM here (the bench uses the 64 GiB row-pair layout)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N, STRIDE, PPC, SEED = 65536, 128, 2048, 2


@pytest.fixture(scope="module")
def c5(gpu):
    import paper_2506_23364_b200 as wf
    from paper_2506_23364_b200 import _device, _lib
    from paper_2506_23364_b200.simulate import release_cells, release_mask_from_dem
    from paper_2506_23364_b200.synth import synth_dem_device

    grid = wf.DemGrid.adopt(N, N, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(N, SEED))
    mask = release_mask_from_dem(grid, 30.0, 45.0, STRIDE)
    cells = release_cells(mask)
    absmax = _device.empty((1,), torch.int64)
    e = grid.device_elevations()
    _lib.check(_lib.lib().wg_absmax(_lib.ptr(e), e.numel(), _lib.ptr(absmax), _lib.stream_ptr()))
    object.__setattr__(grid, "_gather", (None, None, absmax))  # plain-DEM gathers: keeps HBM for two raster sets
    params = wf.AvalancheParams(particles_per_release_cell=PPC, seed=SEED)
    return wf, grid, mask, cells, params


def test_c5_lattice_mask_equals_numpy_chain(c5):
    from oracle import npref

    wf, grid, mask, cells, params = c5
    e = grid.device_elevations()

    def rows_of(idx):
        return e[torch.from_numpy(np.ascontiguousarray(idx)).cuda()].cpu().numpy()

    want = npref.lattice_release_mask(None, 10.0, 30.0, 45.0, STRIDE, rows_of=rows_of, shape=(N, N))
    got = mask.mask
    assert np.array_equal(got, want)
    assert mask.count == int(want.sum()) == cells.numel() > 90_000
    assert mask.borderline == 0


def test_c5_two_rank_bands_equal_one_rank(c5):
    from paper_2506_23364_b200 import shard
    from paper_2506_23364_b200.simulate import run_avalanche_device
    from paper_2506_23364_b200.workflow import device_digest

    wf, grid, mask, cells, params = c5
    plan = shard.plan_bands(N, N, 2)
    hits = torch.zeros((N, N), dtype=torch.int64, device="cuda")
    zmax = torch.zeros((N, N), dtype=torch.float64, device="cuda")
    run_avalanche_device(grid, cells, params, hits=hits, zmax=zmax)
    want = {b: (device_digest(hits[slice(*plan.rows(b))]), device_digest(zmax[slice(*plan.rows(b))]))
            for b in range(plan.nbands)}
    total_hits = int(hits.sum().item())
    offs = shard.band_cell_offsets(cells, plan)
    touched = torch.zeros((plan.tiles_y, plan.tiles_x), dtype=torch.uint8, device="cuda")

    def run_rank(r):
        hits.zero_()
        zmax.zero_()
        touched.zero_()
        run_avalanche_device(grid, cells, params, ranges=shard.particle_ranges(offs, plan, r, PPC), hits=hits,
                             zmax=zmax, touched=touched, plan=plan, rank=r)

    # rank 1's tiles in rank 0's bands, then rank 0 with them folded in
    run_rank(1)
    counts1, ids1, data1 = shard.pack_foreign(hits, zmax, touched, plan, 1)
    run_rank(0)
    counts0, ids0, data0 = shard.pack_foreign(hits, zmax, touched, plan, 0)
    shard.accumulate_tiles(hits, zmax, plan, ids1, data1)
    got_hits = 0
    for b in plan.owned_bands(0):
        sl = slice(*plan.rows(b))
        assert (device_digest(hits[sl]), device_digest(zmax[sl])) == want[b], f"band {b}"
        got_hits += int(hits[sl].sum().item())
    del ids1, data1
    run_rank(1)
    shard.accumulate_tiles(hits, zmax, plan, ids0, data0)
    for b in plan.owned_bands(1):
        sl = slice(*plan.rows(b))
        assert (device_digest(hits[sl]), device_digest(zmax[sl])) == want[b], f"band {b}"
        got_hits += int(hits[sl].sum().item())
    assert got_hits == total_hits
    sent = (sum(counts0) + sum(counts1)) * 2 * plan.tile * plan.tile * 8
    assert sent < 0.15 * N * N * 16  # tile-sparse: well under one dense raster pair


def test_c5_sampled_chunks_equal_oracle(c5):
    from oracle import traj

    from paper_2506_23364_b200.simulate import particle_records

    wf, grid, mask, cells, params = c5
    elev = grid.elevations  # 32 GiB host view (staged download)
    cells_h = cells.cpu().numpy().astype(np.int64)
    nchunks = cells_h.size * PPC // 2048
    for c in np.linspace(0, nchunks - 1, 16).astype(np.int64):
        lo, hi = int(c) * 2048, int(c + 1) * 2048
        rr, st, en = particle_records(grid, mask, params, lo, hi)
        _, (orr, ost, oen) = traj.run_range(elev, 0.0, 0.0, 10.0, cells_h, lo, hi, None, None,
                                            particles_per_release_cell=PPC, seed=SEED, records=True)
        assert np.array_equal(rr, orr) and np.array_equal(st, ost), int(c)
        assert np.array_equal(en.view(np.int64), oen.view(np.int64)), int(c)


def test_c5_full_raster_equals_oracle(c5):
    """Every particle of C5 (2.2e8 particles, 1.09e10 steps), GPU vs the C
    oracle on the box's host threads (~2 minutes); compared band by band on
    the device (the host holds the 32 GiB DEM and the oracle's 64 GiB of
    rasters)."""
    import os

    from oracle import traj

    from paper_2506_23364_b200.simulate import run_avalanche_device

    wf, grid, mask, cells, params = c5
    hits = torch.zeros((N, N), dtype=torch.int64, device="cuda")
    zmax = torch.zeros((N, N), dtype=torch.float64, device="cuda")
    run_avalanche_device(grid, cells, params, hits=hits, zmax=zmax)
    elev = grid.elevations
    cells_h = cells.cpu().numpy().astype(np.int64)
    oh = np.zeros((N, N), dtype=np.int64)
    oz = np.zeros((N, N), dtype=np.float64)
    total = cells_h.size * PPC
    steps = traj.run_range(elev, 0.0, 0.0, 10.0, cells_h, 0, total, oh, oz, particles_per_release_cell=PPC, seed=SEED,
                           threads=os.cpu_count())
    assert steps > 1.0e10
    rows = 2048
    bh = torch.empty((rows, N), dtype=torch.int64, device="cuda")
    bz = torch.empty((rows, N), dtype=torch.float64, device="cuda")
    bad_h = bad_z = 0
    for r0 in range(0, N, rows):
        bh.copy_(torch.from_numpy(oh[r0:r0 + rows]))
        bz.copy_(torch.from_numpy(oz[r0:r0 + rows]))
        bad_h += int((hits[r0:r0 + rows] != bh).sum().item())
        bad_z += int((zmax[r0:r0 + rows].view(torch.int64) != bz.view(torch.int64)).sum().item())
    assert bad_h == 0 and bad_z == 0, (bad_h, bad_z)

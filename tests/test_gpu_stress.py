"""Randomised parity stress of the trajectory kernel against the C oracle:
60 seeded worlds (shapes 20-300, cellsizes 0.5-100, origins up to 1e6,
terraced terrain every 7th case, random release sets and parameters), every
one bit-exact in hit_count and z_delta_max."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = range(100, 160)


def stress_world(case: int):
    """The seeded world and parameters of one stress case."""
    from paper_2506_23364_b200.synth import synth_dem_host

    r = np.random.default_rng(1000 + case)
    nr, nc = int(r.integers(20, 300)), int(r.integers(20, 300))
    cs = float(r.choice([0.5, 3.7, 10.0, 25.0, 1.0 / 3.0, 100.0]))
    ox, oy = float(r.uniform(-1e6, 1e6)), float(r.uniform(-1e6, 1e6))
    e = synth_dem_host(max(nr, nc), int(case) % 50)[:nr, :nc] * float(r.uniform(0.01, 5.0)) * (cs / 10.0)
    e = e + r.uniform(-80, 80) * np.linspace(0, 1, nc)[None, :] + r.uniform(-80, 80) * np.linspace(0, 1, nr)[:, None]
    if case % 7 == 0:
        e = np.round(e, 1)  # terraces / plateaus
    e = np.ascontiguousarray(e)
    mask = r.random((nr, nc)) < float(r.uniform(0.002, 0.05))
    params = {"particles_per_release_cell": int(r.integers(1, 64)), "seed": int(r.integers(0, 2**63)),
              "persistence": float(r.uniform(0, 1)), "randomness": float(r.uniform(0, 1)),
              "runout_angle_deg": float(r.uniform(1, 60))}
    return e, ox, oy, cs, mask, params


def run_case(wf, case: int) -> bool:
    from oracle import traj

    e, ox, oy, cs, mask, params = stress_world(case)
    nr, nc = e.shape
    grid = wf.DemGrid(ncols=nc, nrows=nr, origin_x=ox, origin_y=oy, cellsize=cs, nodata=-9999.0, elevations=e)
    run = wf.run_avalanche(grid, wf.ReleaseMask(mask), wf.AvalancheParams(**params))
    z, h = traj.run_avalanche(e, ox, oy, cs, mask, **params)
    return bool(np.array_equal(run.hit_count, h)
                and np.array_equal(np.ascontiguousarray(run.z_delta_max).view(np.int64), z.view(np.int64)))


@pytest.mark.parametrize("case", CASES)
def test_stress_world_vs_oracle(gpu, case):
    import paper_2506_23364_b200 as wf

    assert run_case(wf, case)

"""Generate tests/golden/baseline_golden.json by running the REFERENCE
(/root/reference/pkg/src/demflow) on the BASELINE.md section-3 configs, in
this container (AVX-512 numpy 2.3.5, glibc 2.39).

The inputs are the synthetic DEMs of the measurement plan
(paper_2506_23364_b200.synth: separable, so the DEM is fixed by its 1-D
factors, whose SHA-256 is stored -- a GPU-box test regenerates them and checks
the hash before comparing anything else).  The arrays are too large to
commit, so the reference's outputs travel as SHA-256 digests of their bytes
(the reference's own `tobytes()` layouts) plus its stats:

* C2  synth_dem(4096, 0): stock snow graph, snow line = median height,
      blend 200 m, max steepness 50, blend 10, zoom 1 (4 tiles):
      normals, slope, 13-level pyramid (workflow.py:267-274).
* C3  synth_dem(16384, 0): compute_normals -> steepness_deg ->
      detect_release_points(30, 45, stride 32 and 256): the full-chain masks;
      run_avalanche at the parity size (stride 256, 64 particles per cell).
* C4  world synth_dem(8192, 1), zoom 2 (16 stitched tiles), band 30-45,
      parity size stride 128, 64 particles per cell, seed 0: stock avalanche
      graph -> runout, stats, 14-level pyramid, and every extract_tile of
      zooms 0..5 (workflow.py:242-264, overlay.py:190-252).

Run:  python tests/golden/make_baseline_golden.py   (about 10 minutes)
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent / "baseline_golden.json"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def factors_sha(n: int, seed: int) -> str:
    from paper_2506_23364_b200.synth import _factors

    rowf, colf, lin = _factors(n, seed, 10.0, 300.0, 4000.0)
    return sha(np.concatenate([rowf.ravel(), colf.ravel(), lin]))


def main() -> None:
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import demflow as d
    from demflow import overlay as ov
    from demflow.workflow import Executor, SteepnessRelease, build_avalanche_graph, build_snow_graph

    from paper_2506_23364_b200.synth import synth_dem_host

    meta: dict = {"numpy": np.__version__, "generator": "tests/golden/make_baseline_golden.py",
                  "timings_note": "reference wall times in the generating container (8-core Xeon, AVX-512)"}

    # ---- C2: snow graph at 4096^2 -------------------------------------------
    n = 4096
    z = synth_dem_host(n, 0)
    grid = d.DemGrid(ncols=n, nrows=n, origin_x=0.0, origin_y=0.0, cellsize=10.0, nodata=-9999.0, elevations=z)
    line = float(np.median(z))
    snow = d.SnowParams(snow_line_m=line, altitude_blend_m=200.0, max_steepness_deg=50.0, steepness_blend_deg=10.0)
    g = build_snow_graph(grid.extent, snow, zoom=1)
    g.bind("world", grid)
    t0 = time.perf_counter()
    res = Executor().execute(g)
    wall = time.perf_counter() - t0
    pyr = res.value("snow_overlay", "overlay")
    meta["c2"] = {
        "n": n, "seed": 0, "factors_sha": factors_sha(n, 0), "dem_sha": sha(z), "snow_line_m": line,
        "normals_sha": sha(res.value("surface_normals", "normals").normals),
        "slope_sha": sha(res.value("steepness", "slope").slope_deg),
        "levels_sha": [sha(lv.pixels) for lv in pyr.levels],
        "ref_wall_s": wall, "ref_node_ms": {r.node_id: r.elapsed_ms for r in res.report.records},
    }
    print("C2 done", wall, flush=True)
    del res, pyr, g, grid, z

    # ---- C4: stock avalanche graph over a stitched 8192^2 world --------------
    n = 8192
    z = synth_dem_host(n, 1)
    world = d.DemGrid(ncols=n, nrows=n, origin_x=0.0, origin_y=0.0, cellsize=10.0, nodata=-9999.0, elevations=z)
    params = d.AvalancheParams(particles_per_release_cell=64, seed=0)
    rel = SteepnessRelease(30.0, 45.0, stride=128)
    g = build_avalanche_graph(world.extent, params, rel, zoom=2)
    g.bind("world", world)
    t0 = time.perf_counter()
    res = Executor().execute(g)
    wall = time.perf_counter() - t0
    run = res.value("avalanche_overlay", "runout")
    pyr = res.value("avalanche_overlay", "overlay")
    mask = res.value("release_points", "mask")
    tiles = []
    zmax = ov.max_tile_zoom(pyr.width, pyr.height)
    for zoom in range(zmax + 1):
        k = 1 << zoom
        for ty in range(k):
            for tx in range(k):
                tiles.append(sha(ov.extract_tile(pyr, zoom, tx, ty).pixels))
    meta["c4"] = {
        "n": n, "seed": 1, "factors_sha": factors_sha(n, 1), "dem_sha": sha(z), "zoom": 2,
        "release": [30.0, 45.0, 128], "particles_per_release_cell": 64, "avalanche_seed": 0,
        "stitched_sha": sha(res.value("stitch_tiles", "dem").elevations),
        "mask_sha": sha(mask.mask), "release_cells": int(mask.count),
        "z_sha": sha(run.z_delta_max), "h_sha": sha(run.hit_count),
        "stats": res.value("avalanche_overlay", "stats"),
        "levels_sha": [sha(lv.pixels) for lv in pyr.levels],
        "tiles_max_zoom": zmax, "tiles_count": len(tiles),
        "tiles_sha": hashlib.sha256("".join(tiles).encode()).hexdigest(),
        "ref_wall_s": wall, "ref_node_ms": {r.node_id: r.elapsed_ms for r in res.report.records},
    }
    print("C4 done", wall, flush=True)
    del res, run, pyr, mask, g, world, z

    # ---- C3: full-chain masks at 16384^2, parity-sized trajectories ----------
    n = 16384
    z = synth_dem_host(n, 0)
    grid = d.DemGrid(ncols=n, nrows=n, origin_x=0.0, origin_y=0.0, cellsize=10.0, nodata=-9999.0, elevations=z)
    t0 = time.perf_counter()
    normals = d.compute_normals(grid)
    slope = d.steepness_deg(normals)
    t_slope = time.perf_counter() - t0
    del normals
    c3 = {"n": n, "seed": 0, "factors_sha": factors_sha(n, 0), "dem_sha": sha(z), "slope_sha": sha(slope.slope_deg),
          "ref_slope_s": t_slope}
    s = slope.slope_deg
    # distance of every lattice slope to the band edges (how close the
    # threshold decisions come to the slope's last bits)
    for stride in (32, 256):
        m = d.detect_release_points(slope, 30.0, 45.0, stride=stride)
        lat = s[::stride, ::stride]
        c3[f"stride{stride}"] = {"mask_sha": sha(m.mask), "release_cells": int(m.count),
                                 "min_edge_distance_deg": float(min(np.abs(lat - 30.0).min(), np.abs(lat - 45.0).min()))}
    m = d.detect_release_points(slope, 30.0, 45.0, stride=256)
    del slope, s
    params = d.AvalancheParams(particles_per_release_cell=64, seed=0)
    t0 = time.perf_counter()
    run = d.run_avalanche(grid, m, params, threads=8)
    c3["parity_run"] = {"stride": 256, "particles_per_release_cell": 64, "seed": 0,
                        "z_sha": sha(run.z_delta_max), "h_sha": sha(run.hit_count),
                        "released": d.simulate.released_particles(m, params),
                        "steps": d.simulate.total_particle_steps(run, d.simulate.released_particles(m, params)),
                        "ref_wall_s": time.perf_counter() - t0}
    meta["c3"] = c3
    print("C3 done", flush=True)
    OUT.write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", OUT)


if __name__ == "__main__":
    main()

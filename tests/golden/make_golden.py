"""Generate the golden fixtures of tests/golden/ by running the REFERENCE
implementation (/root/reference/pkg/src/demflow) in this container.

/root/reference does not exist on the GPU box, so its outputs travel as these
small committed fixtures.  Re-run with:  python tests/golden/make_golden.py
Every input array is stored next to the reference's outputs, so the fixtures
do not depend on how the inputs were generated.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def smooth_dem(seed: int, ncols: int, nrows: int):
    """Gaussian bumps over a tilted plane (same family as the reference's test
    terrains, generated independently here)."""
    r = np.random.default_rng(1000 + seed)
    cs = float(r.uniform(4.0, 25.0))
    ox = float(r.uniform(-1000.0, 1000.0))
    oy = float(r.uniform(-1000.0, 1000.0))
    xs = ox + (np.arange(ncols) + 0.5) * cs
    ys = oy + (nrows - 1 - np.arange(nrows) + 0.5) * cs
    X, Y = np.meshgrid(xs, ys)
    z = np.zeros((nrows, ncols))
    for _ in range(int(r.integers(4, 9))):
        cx, cy = float(r.uniform(xs.min(), xs.max())), float(r.uniform(ys.min(), ys.max()))
        amp = float(r.uniform(30.0, 200.0)) * float(r.choice([-1.0, 1.0]))
        sig = float(r.uniform(3.0, 10.0)) * cs
        z = z + amp * np.exp(-((X - cx) ** 2 + (Y - cy) ** 2) / (2.0 * sig * sig))
    z = z + (X - xs.min()) * float(r.uniform(-0.3, 0.3)) + (Y - ys.min()) * float(r.uniform(-0.3, 0.3))
    return z - z.min(), cs, ox, oy


def main() -> None:
    sys.path.insert(0, str(REF))
    import demflow as d
    from demflow import rng as drng
    from demflow.overlay import DEFAULT_RUNOUT_COLORMAP
    from demflow.workflow import Executor, MaskRelease, SteepnessRelease, build_avalanche_graph, build_snow_graph

    meta: dict = {"reference": str(REF), "numpy": np.__version__}

    # ---- parabola workflows (config 1 + the shipped golden run) -------------
    grid, mask = d.gen_parabola()
    par = {}
    for name, params in (("default", d.AvalancheParams()),
                         ("a12s7", d.AvalancheParams(runout_angle_deg=12.0, seed=7))):
        g = build_avalanche_graph(grid.extent, params, MaskRelease(d.ReleaseMask(mask)), zoom=1)
        g.bind("world", grid)
        res = Executor().execute(g)
        run = res.value("avalanche_overlay", "runout")
        pyr = res.value("avalanche_overlay", "overlay")
        par[name] = {
            "z_sha": sha(run.z_delta_max),
            "h_sha": sha(run.hit_count),
            "levels_sha": [sha(lv.pixels) for lv in pyr.levels],
            "stats": res.value("avalanche_overlay", "stats"),
            "slope_sha": sha(res.value("steepness", "slope").slope_deg),
            "normals_sha": sha(res.value("surface_normals", "normals").normals),
        }
    meta["parabola"] = par

    # ---- smooth terrains: every node of both stock graphs ---------------------
    cases = [(0, 61, 47), (1, 33, 90), (2, 128, 96), (3, 7, 5)]
    arrays: dict[str, np.ndarray] = {}
    smooth_meta = []
    for seed, nc, nr in cases:
        z, cs, ox, oy = smooth_dem(seed, nc, nr)
        dem = d.DemGrid(ncols=nc, nrows=nr, origin_x=ox, origin_y=oy, cellsize=cs, nodata=-9999.0, elevations=z)
        av = d.AvalancheParams(particles_per_release_cell=48, seed=seed, runout_angle_deg=15.0 + 3 * seed)
        rel = SteepnessRelease(5.0, 60.0, stride=3)
        g = build_avalanche_graph(dem.extent, av, rel, zoom=d.workflow.default_tile_zoom(dem))
        g.bind("world", dem)
        res = Executor().execute(g)
        snow = d.SnowParams(snow_line_m=float(np.median(z)), altitude_blend_m=40.0, max_steepness_deg=30.0,
                            steepness_blend_deg=8.0)
        gs = build_snow_graph(dem.extent, snow, zoom=d.workflow.default_tile_zoom(dem))
        gs.bind("world", dem)
        rs = Executor().execute(gs)
        k = f"s{seed}_"
        arrays[k + "dem"] = z
        arrays[k + "normals"] = res.value("surface_normals", "normals").normals
        arrays[k + "slope"] = res.value("steepness", "slope").slope_deg
        arrays[k + "mask"] = res.value("release_points", "mask").mask
        run = res.value("avalanche_overlay", "runout")
        arrays[k + "hits"] = run.hit_count
        arrays[k + "zmax"] = run.z_delta_max
        pyr = res.value("avalanche_overlay", "overlay")
        arrays[k + "tex"] = pyr.levels[0].pixels
        spyr = rs.value("snow_overlay", "overlay")
        arrays[k + "snow"] = spyr.levels[0].pixels
        # single-particle trajectories from the first release cells
        cells = np.flatnonzero(arrays[k + "mask"].ravel())[:3]
        paths = []
        for kk, flat in enumerate(cells):
            r, c = divmod(int(flat), nc)
            start = dem.cell_center(r, c)
            for p in (0, 5):
                key = drng.derive_key(av.seed, kk, p)
                tr = d.simulate_particle(dem, start, av, drng.CounterStream(key))
                arrays[f"{k}path_{kk}_{p}"] = tr.positions
                paths.append({"k": kk, "p": p, "key": key, "start": list(start), "reason": tr.stop_reason.value})
        smooth_meta.append({
            "seed": seed, "ncols": nc, "nrows": nr, "cs": cs, "ox": ox, "oy": oy,
            "avalanche": {"persistence": av.persistence, "randomness": av.randomness,
                          "runout_angle_deg": av.runout_angle_deg,
                          "particles_per_release_cell": av.particles_per_release_cell, "seed": av.seed},
            "release": [rel.min_steepness_deg, rel.max_steepness_deg, rel.stride],
            "snow": [snow.snow_line_m, snow.altitude_blend_m, snow.max_steepness_deg, snow.steepness_blend_deg],
            "stats": res.value("avalanche_overlay", "stats"),
            "levels_sha": [sha(lv.pixels) for lv in pyr.levels],
            "snow_levels_sha": [sha(lv.pixels) for lv in spyr.levels],
            "paths": paths,
        })
    meta["smooth"] = smooth_meta

    # ---- colorize / mipmap on awkward inputs ---------------------------------
    r = np.random.default_rng(77)
    tex_meta = []
    for i, (h, w) in enumerate([(1, 1), (1, 7), (9, 1), (37, 23), (64, 64), (5, 130)]):
        vals = r.gamma(1.5, 2.0, size=(h, w))
        vals[r.random((h, w)) < 0.3] = 0.0
        if i == 0:
            vals[:] = 0.0
        cm = d.colorize(vals, DEFAULT_RUNOUT_COLORMAP)
        arrays[f"c{i}_vals"] = vals
        arrays[f"c{i}_px"] = cm.pixels
        t = r.integers(0, 256, size=(h, w, 4), dtype=np.uint8)
        t[..., 3][r.random((h, w)) < 0.2] = 0
        pyr = d.build_mipmap(d.OverlayTexture(t))
        arrays[f"m{i}_tex"] = t
        for li, lv in enumerate(pyr.levels):
            arrays[f"m{i}_L{li}"] = lv.pixels
        tex_meta.append({"h": h, "w": w, "levels": len(pyr.levels)})
    meta["textures"] = tex_meta

    # ---- tiles ---------------------------------------------------------------
    world = d.RegionAABB(-5.0, -5.0, 5005.0, 1505.0)
    tcases = []
    for reg, zoom in (((0, 0, 100, 100), 2), ((-5.0, -5.0, 5005.0, 1505.0), 1), ((1000, 300, 3000, 900), 3),
                      ((2500.0, 750.0, 2500.0 + 1e-9, 750.0 + 1e-9), 1)):
        region = d.RegionAABB(*reg)
        tiles = d.select_tiles(region, world, zoom)
        tcases.append({"region": list(reg), "zoom": zoom, "tiles": [[t.zoom, t.tx, t.ty] for t in tiles]})
    g2, _ = d.gen_parabola()
    split = []
    for zoom in (0, 1, 2, 3):
        for t, sub in d.split_grid(g2, g2.extent, zoom):
            split.append([zoom, t.tx, t.ty, sub.ncols, sub.nrows, sub.origin_x, sub.origin_y])
    meta["tiles"] = {"world": [-5.0, -5.0, 5005.0, 1505.0], "select": tcases, "split_parabola": split}

    # ---- rng KATs ------------------------------------------------------------
    kat = []
    for seed, k, p in ((0, 0, 0), (7, 2, 2047), (2**63 + 5, 12345, 99), (1, 0, 1)):
        key = drng.derive_key(seed, k, p)
        kat.append({"seed": seed, "k": k, "p": p, "key": key,
                    "draws": [drng.draw_bits(key, n) for n in (0, 1, 99)],
                    "units": [drng.draw_unit(key, n) for n in (0, 1, 99)]})
    meta["rng"] = kat

    # ---- the drop-in boundary: OPS port/kind tables, stock graph JSON,
    #      validation codes of broken graphs ------------------------------------
    from demflow import workflow as W

    meta["ops"] = {
        name: {"inputs": {p: k.value for p, k in spec.inputs.items()},
               "outputs": {p: k.value for p, k in spec.outputs.items()}}
        for name, spec in W.OPS.items()
    }
    region = d.RegionAABB(0.0, 0.0, 100.0, 50.0)
    stock = {
        "avalanche_mask": W.graph_to_json(W.build_avalanche_graph(
            region, d.AvalancheParams(seed=3), W.MaskRelease(d.ReleaseMask(np.zeros((5, 10), bool))), zoom=1)),
        "avalanche_steep": W.graph_to_json(W.build_avalanche_graph(
            region, d.AvalancheParams(), W.SteepnessRelease(28.0, 44.0, 2), zoom=2,
            colormap=DEFAULT_RUNOUT_COLORMAP)),
        "snow": W.graph_to_json(W.build_snow_graph(region, d.SnowParams(snow_line_m=1200.0), zoom=0)),
    }
    meta["stock_graphs"] = stock
    broken = []
    base = W.graph_to_json(W.build_snow_graph(region, d.SnowParams(snow_line_m=1.0)))
    import copy

    def mutate(fn):
        doc = copy.deepcopy(base)
        fn(doc)
        g = W.graph_from_json(doc)
        return doc, [[v.code, v.node_id] for v in W.validate(g)]

    cases = {
        "dup": lambda doc: doc["nodes"].append(copy.deepcopy(doc["nodes"][0])),
        "unknown_op": lambda doc: doc["nodes"][3].__setitem__("op", "nope"),
        "unknown_node": lambda doc: doc["nodes"][4]["inputs"].__setitem__("normals", {"node": "ghost", "port": "x"}),
        "unknown_port": lambda doc: doc["nodes"][4]["inputs"].__setitem__(
            "normals", {"node": "surface_normals", "port": "nope"}),
        "unknown_source": lambda doc: doc["nodes"][0]["inputs"].__setitem__("region", {"source": "nope"}),
        "unknown_input": lambda doc: doc["nodes"][2]["inputs"].__setitem__("extra", {"source": "region"}),
        "unbound_input": lambda doc: doc["nodes"][3]["inputs"].pop("dem"),
        "kind_mismatch": lambda doc: doc["nodes"][4]["inputs"].__setitem__(
            "normals", {"node": "stitch_tiles", "port": "dem"}),
        "cycle": lambda doc: doc["nodes"][2]["inputs"].__setitem__("tiles", {"node": "stitch_tiles", "port": "dem"}),
    }
    for name, fn in cases.items():
        doc, codes = mutate(fn)
        broken.append({"name": name, "graph": doc, "violations": codes})
    meta["broken_graphs"] = broken

    np.savez_compressed(OUT / "golden_arrays.npz", **arrays)
    (OUT / "golden_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", OUT / "golden_arrays.npz", (OUT / "golden_arrays.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()

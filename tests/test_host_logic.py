"""Host-side logic of the drop-in boundary (no GPU): the OPS registry, graph
builders, JSON forms, validation codes, tile selection, parameter checks,
the host RNG, and the no-fallback rule."""

import json

import numpy as np
import pytest
import torch

import paper_2506_23364_b200 as wf
from paper_2506_23364_b200 import rng, workflow as W


def test_ops_registry_matches_reference(golden_meta):
    ours = {
        name: {"inputs": {p: k.value for p, k in spec.inputs.items()},
               "outputs": {p: k.value for p, k in spec.outputs.items()}}
        for name, spec in W.OPS.items()
    }
    assert ours == golden_meta["ops"]


def _json_roundtrip(doc):
    return json.loads(json.dumps(doc))


def test_stock_graphs_json_identical(golden_meta):
    region = wf.RegionAABB(0.0, 0.0, 100.0, 50.0)
    mine = {
        "avalanche_mask": W.graph_to_json(W.build_avalanche_graph(
            region, wf.AvalancheParams(seed=3), W.MaskRelease(wf.ReleaseMask(np.zeros((5, 10), bool))), zoom=1)),
        "avalanche_steep": W.graph_to_json(W.build_avalanche_graph(
            region, wf.AvalancheParams(), W.SteepnessRelease(28.0, 44.0, 2), zoom=2,
            colormap=wf.DEFAULT_RUNOUT_COLORMAP)),
        "snow": W.graph_to_json(W.build_snow_graph(region, wf.SnowParams(snow_line_m=1200.0), zoom=0)),
    }
    assert _json_roundtrip(mine) == golden_meta["stock_graphs"]


def test_reference_json_graphs_load_unchanged(golden_meta):
    """A workflow spec serialised by the reference loads and re-serialises
    identically (the 'runs unchanged' contract, workflow.py:886-1052)."""
    for name, doc in golden_meta["stock_graphs"].items():
        g = W.graph_from_json(doc)
        assert _json_roundtrip(W.graph_to_json(g)) == doc, name
        assert W.validate(g) == []


def test_validation_codes_match_reference(golden_meta):
    for case in golden_meta["broken_graphs"]:
        g = W.graph_from_json(case["graph"])
        got = [[v.code, v.node_id] for v in W.validate(g)]
        assert got == case["violations"], case["name"]


def test_executor_rejects_invalid_and_unbound_graphs():
    g = W.build_snow_graph(wf.RegionAABB(0, 0, 10, 10), wf.SnowParams(snow_line_m=1.0))
    with pytest.raises(W.WorkflowError, match="sources without values: world"):
        W.Executor().execute(g)
    bad = W.graph_from_json({"nodes": [{"id": "a", "op": "nope"}]})
    with pytest.raises(W.GraphValidationError) as ei:
        W.Executor().execute(bad)
    assert [v.code for v in ei.value.violations] == ["UNKNOWN_OP"]
    with pytest.raises(W.WorkflowError):
        W.Executor(max_entries=0)


def test_kind_checks_on_bind():
    g = W.build_snow_graph(wf.RegionAABB(0, 0, 10, 10), wf.SnowParams(snow_line_m=1.0))
    with pytest.raises(W.WorkflowError, match="kind DEM_GRID"):
        g.bind("world", np.zeros((4, 4)))
    with pytest.raises(W.WorkflowError):
        g.bind("nope", 1)


def test_params_and_json_forms():
    p = wf.AvalancheParams(persistence=0.5, seed=9, max_steps=77)
    assert W.params_from_json(_json_roundtrip(W.params_to_json(p))) == p
    s = wf.SnowParams(snow_line_m=900.0, steepness_blend_deg=0.0)
    assert W.params_from_json(W.params_to_json(s)) == s
    for kw in ({"persistence": 1.5}, {"randomness": -0.1}, {"runout_angle_deg": 90.0},
               {"particles_per_release_cell": 0}, {"max_steps": 0}):
        with pytest.raises(wf.ParamError):
            wf.AvalancheParams(**kw)
    with pytest.raises(wf.ParamError):
        wf.SnowParams(snow_line_m=1.0, max_steepness_deg=91.0)
    with pytest.raises(W.WorkflowError):
        W.params_from_json({"model": "glacier"})
    cm = W.colormap_from_json(W.colormap_to_json(wf.DEFAULT_RUNOUT_COLORMAP))
    assert cm == wf.DEFAULT_RUNOUT_COLORMAP
    with pytest.raises(wf.OverlayError):
        wf.Colormap(stops=((0.0, (0, 0, 0, 0)), (0.5, (1, 1, 1, 1))))
    r = W.region_from_json(W.region_to_json(wf.RegionAABB(-1.0, -2.0, 3.0, 4.0)))
    assert r == wf.RegionAABB(-1.0, -2.0, 3.0, 4.0)
    with pytest.raises(wf.GridError):
        wf.RegionAABB(1.0, 0.0, 1.0, 2.0)


def test_select_tiles_matches_reference(golden_meta):
    t = golden_meta["tiles"]
    world = wf.RegionAABB(*t["world"])
    for case in t["select"]:
        got = [[x.zoom, x.tx, x.ty] for x in wf.select_tiles(wf.RegionAABB(*case["region"]), world, case["zoom"])]
        assert got == case["tiles"]
    with pytest.raises(wf.TileError):
        wf.select_tiles(wf.RegionAABB(1e6, 1e6, 2e6, 2e6), world, 1)
    with pytest.raises(wf.TileError):
        wf.TileId(1, 2, 0)


def test_tile_ownership_ranges_match_reference(golden_meta):
    """Owned cell windows of every tile of the parabola at zooms 0-3
    (tiles.py:85-136) from host metadata alone."""
    from paper_2506_23364_b200.tiles import owned_columns, owned_rows, tile_extent

    class G:  # geometry of the bundled parabola (grid.py:195-221)
        ncols, nrows, origin_x, origin_y, cellsize = 501, 151, -5.0, -5.0, 10.0

    world = wf.RegionAABB(-5.0, -5.0, -5.0 + 5010.0, -5.0 + 1510.0)
    got = []
    for zoom in (0, 1, 2, 3):
        for ty in range(1 << zoom):
            for tx in range(1 << zoom):
                ext = tile_extent(world, wf.TileId(zoom, tx, ty))
                j0, j1 = owned_columns(G, ext.min_x, ext.max_x, tx == 0)
                i0, i1 = owned_rows(G, ext.min_y, ext.max_y, ty == 0)
                if j0 > j1 or i0 > i1:
                    continue
                got.append([zoom, tx, ty, j1 - j0 + 1, i1 - i0 + 1, G.origin_x + j0 * G.cellsize,
                            G.origin_y + (G.nrows - 1 - i1) * G.cellsize])
    assert got == golden_meta["tiles"]["split_parabola"]


def test_host_rng_kats(golden_meta):
    for kat in golden_meta["rng"]:
        key = rng.derive_key(kat["seed"], kat["k"], kat["p"])
        assert key == kat["key"]
        assert [rng.draw_bits(key, n) for n in (0, 1, 99)] == kat["draws"]
        assert [rng.draw_unit(key, n) for n in (0, 1, 99)] == kat["units"]
        arr = rng.derive_keys_array(kat["seed"], np.array([kat["k"]]), np.array([kat["p"]]))
        assert int(arr[0]) == key
        assert rng.draw_unit_array(arr, np.array([99]))[0] == kat["units"][2]
    assert rng.CounterStream.for_particle(7, 2, 2047).key == rng.derive_key(7, 2, 2047)


def test_demgrid_host_metadata_and_validation():
    e = np.arange(12, dtype=np.float64).reshape(3, 4)
    g = wf.DemGrid(4, 3, 10.0, 20.0, 2.0, -9999.0, e)
    assert g.extent == wf.RegionAABB(10.0, 20.0, 18.0, 26.0)
    assert g.cell_center(0, 0) == (11.0, 25.0)
    assert g.cell_of(11.0, 25.0) == (0, 0) and g.cell_of(-1e9, -1e9) == (2, 0)
    assert not g.has_nodata() and not e.flags.writeable
    with pytest.raises(wf.GridError):
        wf.DemGrid(1, 3, 0, 0, 1.0, -9999.0, np.zeros((3, 1)))
    with pytest.raises(wf.GridError):
        wf.DemGrid(4, 3, 0, 0, 0.0, -9999.0, e)
    with pytest.raises(wf.GridError):
        wf.DemGrid(4, 3, 0, 0, 1.0, -9999.0, np.zeros((4, 3)))
    bad = e.copy()
    bad[0, 0] = np.nan
    with pytest.raises(wf.GridError):
        wf.DemGrid(4, 3, 0, 0, 1.0, -9999.0, bad)
    holed = e.copy()
    holed[1, 1] = -9999.0
    assert wf.DemGrid(4, 3, 0, 0, 1.0, -9999.0, holed).has_nodata()
    with pytest.raises(Exception):
        g.ncols = 5
    assert wf.grid.sample_elevation(g, 13.0, 23.0) == pytest.approx(5.5 - 0.0, abs=3.0)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_compute_nodes_fail_loudly_without_gpu():
    from paper_2506_23364_b200._lib import NativeUnavailable

    grid, mask = wf.gen_parabola()
    with pytest.raises(NativeUnavailable):
        wf.compute_normals(grid)
    g = W.build_avalanche_graph(grid.extent, wf.AvalancheParams(), W.MaskRelease(wf.ReleaseMask(mask)))
    g.bind("world", grid)
    with pytest.raises(W.NodeExecutionError) as ei:
        W.Executor().execute(g)
    assert isinstance(ei.value.cause, NativeUnavailable)


def test_exchange_segments_group_foreign_tiles_by_owner():
    from paper_2506_23364_b200 import shard

    plan = shard.plan_bands(1024, 1024, 4, 2, 6)  # 8 bands of 128 rows = 2 tile rows
    rng = np.random.default_rng(1)
    ids = np.unique(rng.integers(0, plan.tiles_x * plan.tiles_y, 100))
    toffs = [int(v) for v in np.searchsorted(ids, plan.tile_bounds())]
    for rank in range(4):
        segs, counts = shard.exchange_segments(toffs, plan, rank)
        assert counts[rank] == 0
        out = np.concatenate([ids[s:s + n] for s, _, n in segs])
        # every foreign tile exactly once, grouped by destination rank in rank order
        owners = [plan.owner(int(t) // plan.tiles_x * plan.tile // plan.band_rows) for t in out]
        assert owners == sorted(owners) and rank not in owners
        foreign = [t for t in ids if plan.owner(int(t) // plan.tiles_x * plan.tile // plan.band_rows) != rank]
        assert sorted(out.tolist()) == sorted(int(t) for t in foreign)
        assert sum(counts) == len(out)
        assert [s[1] for s in segs] == list(np.cumsum([0] + [s[2] for s in segs])[:-1])

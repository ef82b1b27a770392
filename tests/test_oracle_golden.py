"""The CPU oracle pinned against the reference's goldens and reference-run
fixtures (tests/golden/make_golden.py).  No GPU."""

import hashlib
from pathlib import Path

import numpy as np
import pytest

from oracle import npref, traj


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# hashes of pkg/demos/out/{z_delta_max,hit_count}.asc as arrays
SHIPPED_A12S7 = (
    "00aaaac27cd75059b1208278d86ce6475682503e30fa5bff084890a6ef4f69fd",
    "db311426d1cff28df1307fc4ccb768bc3117d4562036d0ef913c44076a438bbe",
)


@pytest.mark.parametrize("name,kw", [("default", {}), ("a12s7", {"runout_angle_deg": 12.0, "seed": 7})])
def test_traj_oracle_parabola_goldens(parabola_host, golden_meta, name, kw):
    elev, mask, ox, oy, cs = parabola_host
    z, h = traj.run_avalanche(elev, ox, oy, cs, mask, **kw)
    g = golden_meta["parabola"][name]
    assert sha(z) == g["z_sha"]
    assert sha(h) == g["h_sha"]
    assert int(h.sum()) - int(mask.sum()) * 2048 == g["stats"]["particle_steps"]
    if name == "a12s7":
        assert (sha(z), sha(h)) == SHIPPED_A12S7


def test_traj_oracle_thread_invariance(parabola_host):
    elev, mask, ox, oy, cs = parabola_host
    a = traj.run_avalanche(elev, ox, oy, cs, mask, runout_angle_deg=20.0, seed=3, threads=1)
    b = traj.run_avalanche(elev, ox, oy, cs, mask, runout_angle_deg=20.0, seed=3, threads=7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_traj_oracle_smooth_fixtures(golden_meta, golden_arrays):
    for case in golden_meta["smooth"]:
        k = f"s{case['seed']}_"
        av = case["avalanche"]
        z, h = traj.run_avalanche(golden_arrays[k + "dem"], case["ox"], case["oy"], case["cs"],
                                  golden_arrays[k + "mask"], **av)
        assert np.array_equal(h, golden_arrays[k + "hits"]), case["seed"]
        assert np.array_equal(z.view(np.int64), golden_arrays[k + "zmax"].view(np.int64)), case["seed"]


def test_traj_oracle_single_particles(golden_meta, golden_arrays):
    codes = ["RUNOUT_ANGLE", "DOMAIN_EXIT", "FLAT", "MAX_STEPS"]
    for case in golden_meta["smooth"]:
        k = f"s{case['seed']}_"
        av = case["avalanche"]
        for p in case["paths"]:
            path, r = traj.simulate_particle(
                golden_arrays[k + "dem"], case["ox"], case["oy"], case["cs"], p["start"], p["key"],
                persistence=av["persistence"], randomness=av["randomness"], runout_angle_deg=av["runout_angle_deg"])
            ref = golden_arrays[f"{k}path_{p['k']}_{p['p']}"]
            assert codes[r] == p["reason"]
            assert np.array_equal(path, ref)


def test_rng_kats(golden_meta):
    for kat in golden_meta["rng"]:
        assert traj.derive_key(kat["seed"], kat["k"], kat["p"]) == kat["key"]
        for n, u in zip((0, 1, 99), kat["units"]):
            assert traj.lib().orc_draw_unit(kat["key"], n) == u


def test_npref_raster_nodes(golden_meta, golden_arrays):
    for case in golden_meta["smooth"]:
        k = f"s{case['seed']}_"
        dem = golden_arrays[k + "dem"]
        n = npref.normals(dem, case["cs"])
        assert np.array_equal(n, golden_arrays[k + "normals"])
        s = npref.steepness(n)
        assert np.array_equal(s, golden_arrays[k + "slope"])  # same numpy, same arccos
        lo, hi, stride = case["release"]
        assert np.array_equal(npref.release_mask(s, lo, hi, stride), golden_arrays[k + "mask"])
        px = npref.snow_texture(dem, s, -9999.0, False, *case["snow"])
        assert np.array_equal(px, golden_arrays[k + "snow"])


def test_npref_textures(golden_meta, golden_arrays):
    from paper_2506_23364_b200.overlay import DEFAULT_RUNOUT_COLORMAP

    for i, tm in enumerate(golden_meta["textures"]):
        got = npref.colorize(golden_arrays[f"c{i}_vals"], DEFAULT_RUNOUT_COLORMAP.stops)
        assert np.array_equal(got, golden_arrays[f"c{i}_px"])
        levels = npref.mipmap(golden_arrays[f"m{i}_tex"])
        assert len(levels) == tm["levels"]
        for li, lv in enumerate(levels):
            assert np.array_equal(lv, golden_arrays[f"m{i}_L{li}"])


def test_npref_parabola_pyramid_hashes(parabola_host, golden_meta):
    from paper_2506_23364_b200.overlay import DEFAULT_RUNOUT_COLORMAP

    elev, mask, ox, oy, cs = parabola_host
    z, _ = traj.run_avalanche(elev, ox, oy, cs, mask)
    levels = npref.mipmap(npref.colorize(z, DEFAULT_RUNOUT_COLORMAP.stops))
    assert [sha(lv) for lv in levels] == golden_meta["parabola"]["default"]["levels_sha"]


def test_ascii_oracle_matches_reference_fixtures():
    """oracle/asciigrid_ref.py (the CPU baseline of tools/bench_ascii.py)
    reproduces the reference-run ASCII fixtures."""
    import hashlib
    import json

    from oracle import asciigrid_ref

    g = json.loads((Path(__file__).resolve().parent / "golden" / "ascii_golden.json").read_text())
    for case in g["write"]:
        z = np.array([float.fromhex(h) for h in case["values_hex"]]).reshape(case["nrows"], case["ncols"])
        hdr = (case["ncols"], case["nrows"], case["origin_x"], case["origin_y"], case["cellsize"], case["nodata"])
        text = asciigrid_ref.write_text(hdr, z)
        assert hashlib.sha256(text.encode()).hexdigest() == case["sha"]
        back = asciigrid_ref.parse_body(text, case["nrows"], case["ncols"])
        assert np.array_equal(back, z)
    for case in g["parse"]:
        if "ok" in case and case["ok"]["values_hex"] is not None:
            ok = case["ok"]
            v = asciigrid_ref.parse_body(case["doc"], ok["nrows"], ok["ncols"])
            assert hashlib.sha256(v.tobytes()).hexdigest() == ok["sha"]

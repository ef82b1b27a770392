"""Hillshade base layer against reference-run fixtures
(tests/golden/hillshade_golden.json from tests/golden/make_hillshade_golden.py):
the gray image and every level of build_mipmap(texture_from_gray(gray)),
bit-exact."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent
CASES = json.loads((HERE / "golden" / "hillshade_golden.json").read_text())["cases"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def grids(gpu, golden_meta, golden_arrays):
    import paper_2506_23364_b200 as wf

    out = {"parabola": wf.gen_parabola()[0]}
    for c in golden_meta["smooth"]:
        out[f"smooth{c['seed']}"] = wf.DemGrid(ncols=c["ncols"], nrows=c["nrows"], origin_x=c["ox"], origin_y=c["oy"],
                                               cellsize=c["cs"], nodata=-9999.0,
                                               elevations=golden_arrays[f"s{c['seed']}_dem"])
    return out


@pytest.mark.parametrize("case", CASES, ids=[f"{c['grid']}-{c['azimuth']:g}-{c['altitude']:g}" for c in CASES])
def test_hillshade_and_pyramid_match_reference(grids, case):
    from paper_2506_23364_b200.terrain import hillshade, hillshade_pyramid

    g = grids[case["grid"]]
    assert sha(hillshade(g, case["azimuth"], case["altitude"])) == case["gray_sha"]
    pyr = hillshade_pyramid(g, case["azimuth"], case["altitude"])
    assert [sha(lv.pixels) for lv in pyr.levels] == case["levels_sha"]

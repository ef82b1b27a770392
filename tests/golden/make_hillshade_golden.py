"""Golden fixtures for the hillshade base layer and its
served tiles (extract_tile, §8f row 2), made
by running the REFERENCE (terrain.py:287-299 hillshade; service.py:527-538
build_mipmap(texture_from_gray(gray))) in this container:
tests/golden/hillshade_golden.json.  Inputs: the bundled parabola and the
smooth-terrain DEMs already stored in golden_arrays.npz.
Re-run: python tests/golden/make_hillshade_golden.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, str(REF))
    from demflow import gen_parabola
    from demflow.grid import DemGrid
    from demflow.overlay import build_mipmap, extract_tile, max_tile_zoom, texture_from_gray
    from demflow.terrain import hillshade

    meta = json.loads((HERE / "golden_meta.json").read_text())
    arrays = dict(np.load(HERE / "golden_arrays.npz"))
    cases = []
    grid, _ = gen_parabola()
    grids = [("parabola", grid, None)]
    for c in meta["smooth"]:
        k = f"s{c['seed']}_dem"
        grids.append((f"smooth{c['seed']}", DemGrid(ncols=c["ncols"], nrows=c["nrows"], origin_x=c["ox"],
                                                    origin_y=c["oy"], cellsize=c["cs"], nodata=-9999.0,
                                                    elevations=arrays[k]), k))
    for name, g, key in grids:
        for az, alt in ((315.0, 45.0), (90.0, 30.0), (200.0, 70.0)):
            gray = hillshade(g, az, alt)
            pyr = build_mipmap(texture_from_gray(gray))
            case = {"grid": name, "array": key, "azimuth": az, "altitude": alt, "gray_sha": sha(gray),
                    "levels_sha": [sha(lv.pixels) for lv in pyr.levels]}
            if az == 315.0:  # the service's tiles of this base layer (extract_tile, overlay.py:231-252)
                tiles = {}
                for tile_px in (256, 64):
                    zmax = max_tile_zoom(pyr.width, pyr.height, tile_px)
                    for z in range(zmax + 1):
                        for ty in range(1 << z):
                            for tx in range(1 << z):
                                tiles[f"{tile_px}/{z}/{tx}/{ty}"] = sha(extract_tile(pyr, z, tx, ty, tile_px).pixels)
                case["tiles_sha"] = tiles
            cases.append(case)
    (HERE / "hillshade_golden.json").write_text(json.dumps({"reference": str(REF), "cases": cases}, indent=1) + "\n")
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()

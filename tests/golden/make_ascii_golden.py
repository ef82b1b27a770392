"""Golden fixtures for the ASCII grid reader/writer, produced by running the
REFERENCE (/root/reference/pkg/src/demflow/asciigrid.py) in this container:
tests/golden/ascii_golden.json.  Re-run: python tests/golden/make_ascii_golden.py

* parse cases: document text -> either the parsed header + sha256 of the
  elevation bytes, or the AsciiGridError message / line / column;
* write cases: seeded grids (the inputs are stored as raw float64 hex so the
  fixture does not depend on how they were generated) -> sha256 of the
  canonical text, plus the text itself for the small ones;
* the parabola DEM: sha256 of write_ascii_grid(gen_parabola()) and whether it
  equals the shipped pkg/data/parabola/dem.asc byte for byte.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "ascii_golden.json"

CANONICAL = ("ncols 3\nnrows 2\nxllcorner -5\nyllcorner 100.5\ncellsize 10\nNODATA_value -9999\n"
             "1 2 3.25\n4 -9999 6e-05\n")


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def header(n_cols=3, n_rows=2, extra=""):
    return (f"ncols {n_cols}\nnrows {n_rows}\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n" + extra)


def parse_docs() -> list[tuple[str, str]]:
    r = np.random.default_rng(5)
    docs = [
        ("canonical", CANONICAL),
        ("keys_case", CANONICAL.replace("ncols", "NCOLS").replace("NODATA_value", "nodata_VALUE")),
        ("split_lines_ws", header(extra="1 2\n3\n  4\t5 6\n")),
        ("crlf", CANONICAL.replace("\n", "\r\n")),
        ("cr_only", CANONICAL.replace("\n", "\r")),
        ("vt_ff_seps", header(extra="1\x0b2\x0c3\x1c4\x1d5\x1e6\x1f")),
        ("no_final_newline", CANONICAL[:-1]),
        ("sci_underscore_sign", header(extra="1e3 -2.5E-3 +7 1_000.5 .5 5.\n")),
        ("inf_token", header(extra="1 2 3 4 5 inf\n")),
        ("nan_token", header(extra="1 2 3 NaN 5 6\n")),
        ("nodata_holes", header(extra="-9999 2 3 4 -9999 6\n")),
        ("long_digits", header(extra="0.1000000000000000055511151231257827 2.5000000000000004 "
                                     "9007199254740993 1e-320 1.7976931348623157e308 123456789012345678901234\n")),
        ("header_out_of_order", CANONICAL.replace("ncols 3", "nrows 3", 1).replace("nrows 2", "ncols 2", 1)),
        ("truncated_header", "ncols 3\nnrows 2\n"),
        ("empty", ""),
        ("header_only_5", "ncols 3\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1"),
        ("header_only_6", "ncols 3\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999"),
        ("non_integer_dim", CANONICAL.replace("nrows 2", "nrows two")),
        ("float_dim", CANONICAL.replace("ncols 3", "ncols 3.0")),
        ("zero_dim", CANONICAL.replace("nrows 2", "nrows 0")),
        ("negative_dim", CANONICAL.replace("ncols 3", "ncols -3")),
        ("bad_header_value", CANONICAL.replace("xllcorner -5", "xllcorner abc")),
        ("inf_header", CANONICAL.replace("cellsize 10", "cellsize inf")),
        ("nan_nodata", CANONICAL.replace("NODATA_value -9999", "NODATA_value nan")),
        ("three_token_header", CANONICAL.replace("cellsize 10", "cellsize 10 20")),
        ("wrong_key", CANONICAL.replace("yllcorner", "ylcorner")),
        ("zero_cellsize", CANONICAL.replace("cellsize 10", "cellsize 0")),
        ("too_few", CANONICAL.rsplit("6e-05", 1)[0] + "\n"),
        ("too_few_blank_lines", CANONICAL.rsplit("6e-05", 1)[0] + "\n\n\n"),
        ("too_many", CANONICAL[:-1] + " 7\n"),
        ("too_many_next_line", CANONICAL + "  \t 8 9\n"),
        ("bad_token", CANONICAL.replace("3.25", "3.2.5")),
        ("bad_token_second_row", CANONICAL.replace("6e-05", "6e-0x5")),
        ("two_bad_tokens", CANONICAL.replace("2 ", "x ").replace("3.25", "y")),
        ("bad_and_count", CANONICAL.replace("3.25", "3.2.5")[:-1] + " 7\n"),
        ("one_by_two", "ncols 1\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n1\n2\n"),
        ("underscore_bad", header(extra="1 2 3 4 5 1__0\n")),
        ("tabs_header", "ncols\t3\nnrows   2\nxllcorner\t-5\nyllcorner 100.5\ncellsize 10\nNODATA_value -9999\n"
                        "1 2 3.25\n4 -9999 6e-05\n"),
    ]
    vals = r.uniform(-500, 4800, 12 * 9)
    body = "\n".join(" ".join(repr(float(v)) for v in vals[i * 12:(i + 1) * 12]) for i in range(9))
    docs.append(("random_repr", header(12, 9, body + "\n")))
    return docs


def write_grids():
    """(name, ncols, nrows, ox, oy, cs, nodata, values) -- arbitrary values."""
    out = []
    for seed in range(12):
        r = np.random.default_rng(100 + seed)
        ncols, nrows = int(r.integers(2, 30)), int(r.integers(2, 30))
        z = r.uniform(-5000.0, 9000.0, size=(nrows, ncols))
        flat = z.ravel()
        idx = r.integers(0, flat.size, size=max(1, flat.size // 5))
        flat[idx] = r.choice([0.0, -0.0, 1.0, 123456789.0, 0.1, 1e-12, 2.5, 1e16, 1e16 - 2, 9007199254740993.0,
                              5e-324, 1.7976931348623157e308, -1e-5, 1e-4, 123456.789, 1e22, 1e23], size=idx.size)
        nodata = float(r.choice([-9999.0, -999.25, 3.5e38]))
        holes = r.integers(0, flat.size, size=max(1, flat.size // 11))
        flat[holes] = nodata
        out.append((f"random{seed}", ncols, nrows, float(r.uniform(-1e6, 1e6)), float(r.uniform(-1e6, 1e6)),
                    float(r.uniform(0.01, 500.0)), nodata, z))
    # raw bit patterns (every finite double class)
    r = np.random.default_rng(7)
    bits = r.integers(0, 2**63, size=40 * 25, dtype=np.int64).astype(np.uint64)
    bits |= (r.integers(0, 2, size=bits.size).astype(np.uint64) << np.uint64(63))
    z = bits.view(np.float64)
    z[~np.isfinite(z)] = 1.5
    out.append(("bitpatterns", 40, 25, 0.0, 0.0, 1.0, -9999.0, z.reshape(25, 40)))
    return out


def main() -> None:
    sys.path.insert(0, str(REF))
    from demflow import gen_parabola
    from demflow.asciigrid import AsciiGridError, parse_ascii_grid, write_ascii_grid
    from demflow.grid import DemGrid

    parse = []
    for name, doc in parse_docs():
        case = {"name": name, "doc": doc}
        try:
            g = parse_ascii_grid(doc)
            case["ok"] = {"ncols": g.ncols, "nrows": g.nrows, "origin_x": g.origin_x, "origin_y": g.origin_y,
                          "cellsize": g.cellsize, "nodata": g.nodata, "sha": sha(g.elevations.tobytes()),
                          "values_hex": [float(v).hex() for v in g.elevations.ravel()]
                          if g.elevations.size <= 200 else None}
        except AsciiGridError as e:
            case["error"] = {"message": str(e), "line": e.line, "column": e.column}
        parse.append(case)

    write = []
    for name, ncols, nrows, ox, oy, cs, nd, z in write_grids():
        g = DemGrid(ncols=ncols, nrows=nrows, origin_x=ox, origin_y=oy, cellsize=cs, nodata=nd, elevations=z)
        text = write_ascii_grid(g)
        write.append({"name": name, "ncols": ncols, "nrows": nrows, "origin_x": ox, "origin_y": oy, "cellsize": cs,
                      "nodata": nd, "values_hex": [float(v).hex() for v in z.ravel()],
                      "sha": sha(text.encode()), "text": text if len(text) < 4000 else None})

    pg, _ = gen_parabola()
    ptext = write_ascii_grid(pg)
    shipped = (REF.parent / "data" / "parabola" / "dem.asc").read_bytes()
    meta = {
        "reference": str(REF),
        "parse": parse,
        "write": write,
        "parabola": {"sha": sha(ptext.encode()), "bytes": len(ptext), "equals_shipped_dem_asc": ptext.encode() == shipped,
                     "shipped_sha": sha(shipped), "elev_sha": sha(pg.elevations.tobytes())},
    }
    OUT.write_text(json.dumps(meta, indent=1) + "\n")
    print(f"wrote {OUT}: {len(parse)} parse cases, {len(write)} write cases, "
          f"parabola equals shipped: {meta['parabola']['equals_shipped_dem_asc']}")


if __name__ == "__main__":
    main()

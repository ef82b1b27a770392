"""TEST INFRASTRUCTURE -- CPU restatement of the reference's ASCII grid
reader/writer body path (/root/reference/pkg/src/demflow/asciigrid.py:86-157):
tokens by str.split() over the body lines, np.array(tokens, dtype=float64),
and " ".join(format_number(v)) per row.  Used as the checker in tests and as
the timed CPU baseline of tools/bench_ascii.py; never imported by the
package.  Parity pinned by tests/test_oracle_golden.py::test_ascii_oracle_*
against tests/golden/ascii_golden.json (made by running the reference)."""

from __future__ import annotations

import numpy as np


def format_number(v: float) -> str:  # asciigrid.py:160-167
    f = float(v)
    if f == int(f) and abs(f) < 1e16:
        return str(int(f))
    return repr(f)


def parse_body(text: str, nrows: int, ncols: int) -> np.ndarray:
    """asciigrid.py:86-137 for a well-formed document: the values array."""
    lines = text.splitlines()
    tokens: list[str] = []
    for line in lines[6:]:
        tokens.extend(line.split())
    if len(tokens) != nrows * ncols:
        raise ValueError(f"expected {nrows * ncols} elevation values, found {len(tokens)}")
    return np.array(tokens, dtype=np.float64).reshape(nrows, ncols)


def write_text(header: tuple, elev: np.ndarray) -> str:
    """asciigrid.py:146-157."""
    keys = ("ncols", "nrows", "xllcorner", "yllcorner", "cellsize", "NODATA_value")
    out = [f"{k} {format_number(v)}" for k, v in zip(keys, header)]
    for row in elev:
        out.append(" ".join(format_number(v) for v in row))
    return "\n".join(out) + "\n"

"""CPU-side checks of the ASCII grid path: the header rules (host code) against
the reference-run fixtures, and the device number parser/formatter source
(csrc/wg_numconv.cuh) compiled for the host with g++ and compared with
CPython float() / the reference's format_number."""

import json
import random
import shutil
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((ROOT / "tests" / "golden" / "ascii_golden.json").read_text())

# cases whose error the reference raises while reading the header (no body work)
HEADER_ERRORS = [c for c in GOLDEN["parse"] if "error" in c and c["error"]["line"] is not None
                 and ("header" in c["error"]["message"] or "must be" in c["error"]["message"])]


@pytest.mark.parametrize("case", HEADER_ERRORS, ids=[c["name"] for c in HEADER_ERRORS])
def test_header_errors_match_reference(case):
    from paper_2506_23364_b200.asciigrid import AsciiGridError, parse_ascii_grid

    with pytest.raises(AsciiGridError) as ei:
        parse_ascii_grid(case["doc"])
    assert str(ei.value) == case["error"]["message"]
    assert (ei.value.line, ei.value.column) == (case["error"]["line"], case["error"]["column"])


def test_line_helpers_match_splitlines():
    from paper_2506_23364_b200.asciigrid import _count_lines, _line_col

    r = random.Random(4)
    for _ in range(300):
        s = "".join(r.choice(["a", "b", " ", "\n", "\r", "\r\n", "\x0b", "\x0c", "\x1c", "\x1f"])
                    for _ in range(r.randint(0, 30)))
        data = s.encode()
        assert _count_lines(data) == len(s.splitlines())
        for off in range(len(data)):
            if data[off:off + 1] not in (b"a", b"b"):
                continue
            lines = s[:off + 1].splitlines()
            # line of the char at off: the number of lines of the prefix ending at it
            assert _line_col(data, off)[0] == len(lines)
            assert _line_col(data, off)[1] == len(lines[-1])


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_numconv_host_build_matches_cpython():
    import sys

    sys.path.insert(0, str(ROOT / "tools" / "numconv"))
    import check  # tools/numconv/check.py

    lib = check.build()
    r = random.Random(2)
    toks = [check.rand_decimal(r) for _ in range(60_000)] + check.halfway_cases(r, 400)
    got, st = check.parse_many(lib, toks)
    for t, g, s in zip(toks, got, st):
        w, ws = check.ref_parse(t)
        assert ws == s and (s != 0 or check.same(w, g)), t
    # the SWAR fast path (plain numerals): whenever it takes a token, float()'s value
    reprs = [repr(float(v)) for v in np.random.default_rng(7).uniform(-5e3, 5e3, 20_000)]
    simple, sst = check.parse_simple_many(lib, toks + reprs)
    assert sst.sum() > 20_000
    for t, g, s in zip(toks + reprs, simple, sst):
        if s:
            w, ws = check.ref_parse(t)
            assert ws == 0 and check.same(w, g), t
    bits = np.random.default_rng(5).integers(0, 2**64, size=60_000, dtype=np.uint64).view(np.float64)
    vals = np.concatenate([bits[np.isfinite(bits)], np.round(np.random.default_rng(6).uniform(-500, 4800, 20_000), 2)])
    for v, s in zip(vals, check.format_many(lib, vals)):
        assert s == check.format_number(v)

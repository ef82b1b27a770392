"""ESRI ASCII grid I/O on the GPU against the
reference-run golden fixtures (tests/golden/ascii_golden.json, made by
tests/golden/make_ascii_golden.py from /root/reference/.../asciigrid.py) and
against CPython float() / the reference's format_number on large random
documents.  Bit-exact values, byte-exact text, identical error messages."""

import hashlib
import json
import random
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "ascii_golden.json").read_text())


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def ref_format(v: float) -> str:  # asciigrid.py:160-167
    f = float(v)
    if f == int(f) and abs(f) < 1e16:
        return str(int(f))
    return repr(f)


@pytest.fixture(scope="module")
def ag(gpu):
    from paper_2506_23364_b200 import asciigrid

    return asciigrid


@pytest.mark.parametrize("case", GOLDEN["parse"], ids=[c["name"] for c in GOLDEN["parse"]])
def test_parse_matches_reference(ag, case):
    if "ok" in case:
        g = ag.parse_ascii_grid(case["doc"])
        ok = case["ok"]
        assert (g.ncols, g.nrows) == (ok["ncols"], ok["nrows"])
        assert (g.origin_x, g.origin_y, g.cellsize, g.nodata) == (ok["origin_x"], ok["origin_y"], ok["cellsize"],
                                                                  ok["nodata"])
        assert sha(np.ascontiguousarray(g.elevations).tobytes()) == ok["sha"]
        if ok["values_hex"] is not None:
            want = np.array([float.fromhex(h) for h in ok["values_hex"]])
            assert np.array_equal(np.asarray(g.elevations).ravel().view(np.int64), want.view(np.int64))
    else:
        with pytest.raises(ag.AsciiGridError) as ei:
            ag.parse_ascii_grid(case["doc"])
        err = case["error"]
        assert str(ei.value) == err["message"]
        assert (ei.value.line, ei.value.column) == (err["line"], err["column"])


def test_parse_accepts_bytes(ag):
    doc = GOLDEN["parse"][0]["doc"]
    a = ag.parse_ascii_grid(doc)
    b = ag.parse_ascii_grid(doc.encode())
    assert np.array_equal(np.asarray(a.elevations), np.asarray(b.elevations))


def test_huge_header_small_body(ag):
    """A header promising 10^12 values over a tiny body raises the
    reference's count error (its messages, run here: 'found 3 (line 7)',
    'found 0 (line 6)') without sizing any buffer by the header."""
    head = "ncols 1000000\nnrows 1000000\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n"
    for body, msg in (("1 2 3\n", "expected 1000000000000 elevation values, found 3 (line 7)"),
                      ("", "expected 1000000000000 elevation values, found 0 (line 6)")):
        with pytest.raises(ag.AsciiGridError) as ei:
            ag.parse_ascii_grid(head + body)
        assert str(ei.value) == msg


UNICODE = json.loads((Path(__file__).resolve().parent / "golden" / "ascii_unicode_golden.json").read_text())


@pytest.mark.parametrize("case", UNICODE, ids=[c["name"] for c in UNICODE])
def test_non_ascii_documents_like_reference(ag, case):
    """Unicode separators / digits parse as the reference's str.split and
    float() read them; other characters give its messages and positions
    (tests/golden/make_ascii_unicode_golden.py ran the reference)."""
    if "ok" in case:
        g = ag.parse_ascii_grid(case["doc"])
        assert (g.ncols, g.nrows) == (case["ok"]["ncols"], case["ok"]["nrows"])
        assert np.asarray(g.elevations).ravel().tolist() == case["ok"]["values"]
    else:
        with pytest.raises(ag.AsciiGridError) as ei:
            ag.parse_ascii_grid(case["doc"])
        assert str(ei.value) == case["error"]


def test_non_ascii_bytes_rejected(ag):
    with pytest.raises(ag.AsciiGridError):
        ag.parse_ascii_grid(GOLDEN["parse"][0]["doc"].encode().replace(b"1 2", b"1\xc2\xa02"))


@pytest.mark.parametrize("case", GOLDEN["write"], ids=[c["name"] for c in GOLDEN["write"]])
def test_write_matches_reference(ag, case):
    from paper_2506_23364_b200 import DemGrid

    z = np.array([float.fromhex(h) for h in case["values_hex"]]).reshape(case["nrows"], case["ncols"])
    g = DemGrid(ncols=case["ncols"], nrows=case["nrows"], origin_x=case["origin_x"], origin_y=case["origin_y"],
                cellsize=case["cellsize"], nodata=case["nodata"], elevations=z)
    text = ag.write_ascii_grid(g)
    if case["text"] is not None:
        assert text == case["text"]
    assert sha(text.encode()) == case["sha"]
    # canonical text is a fixed point and parses back bitwise (-0.0 prints as "0")
    h = ag.parse_ascii_grid(text)
    back = np.asarray(h.elevations)
    assert np.array_equal(back, z) and np.array_equal(back.view(np.int64)[z != 0], z.view(np.int64)[z != 0])
    assert ag.write_ascii_grid(h) == text


def test_parabola_text_equals_shipped_dem(ag):
    from paper_2506_23364_b200 import gen_parabola

    grid, _ = gen_parabola()
    text = ag.write_ascii_grid(grid)
    p = GOLDEN["parabola"]
    assert p["equals_shipped_dem_asc"] and sha(text.encode()) == p["shipped_sha"] == p["sha"]
    g = ag.parse_ascii_grid(text)
    assert sha(np.ascontiguousarray(g.elevations).tobytes()) == p["elev_sha"]


def test_large_random_document_matches_cpython(ag):
    """1.2 M values of every double class written on the device == the
    reference writer's text; parsed back == the written values."""
    from paper_2506_23364_b200 import DemGrid

    r = np.random.default_rng(11)
    nrows, ncols = 600, 2000
    parts = [
        r.integers(0, 2**64, size=200_000, dtype=np.uint64).view(np.float64),
        np.round(r.uniform(-500, 4800, 400_000) * 10.0 ** (k := r.integers(0, 6, 400_000))) / 10.0 ** k,
        r.uniform(0, 1, 200_000),
        r.integers(-10**15, 10**15, 200_000).astype(np.float64),
        np.exp(r.uniform(-700, 700, 200_000)),
    ]
    z = np.concatenate(parts)
    z[~np.isfinite(z)] = 0.5
    z = z[: nrows * ncols].reshape(nrows, ncols)
    g = DemGrid(ncols=ncols, nrows=nrows, origin_x=0.0, origin_y=0.0, cellsize=1.0, nodata=-9999.0, elevations=z)
    text = ag.write_ascii_grid(g)
    body = "\n".join(" ".join(ref_format(v) for v in row) for row in z) + "\n"
    head = "ncols 2000\nnrows 600\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n"
    assert text == head + body
    back = np.asarray(ag.parse_ascii_grid(text).elevations)
    nz = z != 0
    assert np.array_equal(back.view(np.int64)[nz], z.view(np.int64)[nz]) and np.all(back[~nz] == 0)


def rand_token(r: random.Random) -> str:
    nd = r.choice([1, 2, 3, 5, 9, 15, 16, 17, 18, 19, 20, 24, 30])
    digits = "".join(r.choice("0123456789") for _ in range(nd))
    p = r.randint(0, nd)
    body = digits[:p] + ("." if r.random() < 0.7 else "") + digits[p:]
    if body in (".", ""):
        body = "0"
    if r.random() < 0.03 and len(body) > 2 and body[0].isdigit() and body[1].isdigit():
        body = body[0] + "_" + body[1:]
    e = ""
    if r.random() < 0.4:
        e = r.choice("eE") + r.choice(["", "-", "+"]) + str(r.choice([0, 1, 7, 22, 23, 100, 300, 307, 308, 309,
                                                                      320, 323, 324, 330, 342, 343]))
    return r.choice(["", "", "-", "+"]) + body + e


def test_random_tokens_parse_like_cpython(ag):
    """600 k tokens of many shapes (long significands, extreme exponents,
    underscores, signs): the device values == np.array(tokens, float64)."""
    r = random.Random(3)
    ncols, nrows = 1000, 600
    toks = [rand_token(r) for _ in range(ncols * nrows)]
    seps = [" ", " ", "  ", "\t", " \n "]
    body = "".join(t + r.choice(seps) for t in toks)
    doc = f"ncols {ncols}\nnrows {nrows}\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n" + body
    want = np.array(toks, dtype=np.float64)
    fin = np.isfinite(want)
    if not fin.all():  # overflowing tokens: the reference rejects the grid (non-finite)
        with pytest.raises(ag.AsciiGridError, match="non-nodata elevations must be finite"):
            ag.parse_ascii_grid(doc)
        toks = [t if f else "1" for t, f in zip(toks, fin)]
        body = "".join(t + " " for t in toks)
        doc = f"ncols {ncols}\nnrows {nrows}\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n" + body
        want = np.array(toks, dtype=np.float64)
    got = np.asarray(ag.parse_ascii_grid(doc).elevations).ravel()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def test_bytes_buffer_round_trip(ag):
    """write_ascii_grid_bytes -> parse_ascii_grid without a str in between."""
    from paper_2506_23364_b200 import gen_parabola

    grid, _ = gen_parabola()
    buf = ag.write_ascii_grid_bytes(grid)
    assert hashlib.sha256(buf).hexdigest() == GOLDEN["parabola"]["sha"]
    g = ag.parse_ascii_grid(buf)
    assert sha(np.ascontiguousarray(g.elevations).tobytes()) == GOLDEN["parabola"]["elev_sha"]
    with pytest.raises(ag.AsciiGridError, match="invalid elevation value"):
        raw = bytes(buf)
        i = raw.rindex(b" ")
        ag.parse_ascii_grid(memoryview(raw[:i] + b" x" + raw[i + 1:]))


def test_reader_tile_boundaries(ag):
    """The fused reader's 4 KiB tiles: whitespace runs longer than a tile
    (tiles without a token start), tokens longer than a tile (zero-padded
    significands), tokens straddling tile edges at every phase, and the error
    positions of an extra token / an invalid token far into the body."""
    from paper_2506_23364_b200.asciigrid import _line_col

    r = random.Random(9)
    ws = [" ", "\t", "\n", "\r\n", "\x0b", "\x0c", "\x1c", "\x1f"]
    toks, parts = [], []
    ncols, nrows = 700, 30
    for i in range(ncols * nrows):
        k = r.random()
        if k < 0.002:
            v = r.uniform(-9, 9)
            t = ("-" if v < 0 else "") + "0" * r.randint(4000, 9000) + repr(abs(v))  # longer than a tile
        elif k < 0.3:
            t = str(r.randint(-99999, 99999))
        else:
            t = repr(r.uniform(-5000, 5000))
        toks.append(t)
        sep = "".join(r.choice(ws) for _ in range(r.randint(1, 4)))
        if r.random() < 0.003:
            sep += " " * r.randint(4097, 12000)  # a whole tile of whitespace
        parts.append(t + sep)
    head = f"ncols {ncols}\nnrows {nrows}\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n"
    doc = head + "".join(parts)
    want = np.array([float(t) for t in toks])
    got = np.asarray(ag.parse_ascii_grid(doc).elevations).ravel()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    # leading whitespace so the first token starts at every phase of a tile
    head2 = head.replace(f"ncols {ncols}\nnrows {nrows}\n", "ncols 40\nnrows 10\n")
    for pad in (1, 7, 4095, 4096, 4097):
        d2 = head2 + " " * pad + "".join(parts[:400])
        g2 = np.asarray(ag.parse_ascii_grid(d2).elevations).ravel()
        assert np.array_equal(g2.view(np.int64), want[:400].view(np.int64))
    # one extra token: reported at its own line / column
    j = len(parts) * 3 // 4
    extra = head + "".join(parts[:j]) + "7 " + "".join(parts[j:])
    off = len(extra) - len(parts[-1])  # token #expected: the last one
    with pytest.raises(ag.AsciiGridError) as ei:
        ag.parse_ascii_grid(extra)
    assert (ei.value.line, ei.value.column) == _line_col(extra.encode(), off)
    assert str(ei.value).startswith(f"expected {ncols * nrows} elevation values, found {ncols * nrows + 1}")
    # invalid tokens far into the body: the first one is reported
    bad = parts.copy()
    for q in (len(bad) - 5, len(bad) // 2 + 3):
        bad[q] = "1.2.3" + parts[q][len(toks[q]):]
    bdoc = head + "".join(bad)
    with pytest.raises(ag.AsciiGridError) as ei:
        ag.parse_ascii_grid(bdoc)
    q = len(bad) // 2 + 3
    boff = len(head) + sum(len(p) for p in bad[:q])
    assert str(ei.value).startswith("invalid elevation value '1.2.3'")
    assert (ei.value.line, ei.value.column) == _line_col(bdoc.encode(), boff)

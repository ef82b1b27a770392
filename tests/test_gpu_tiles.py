"""Tile serving on the GPU: extract_tile against the
reference's slicing rule (restated below, overlay.py:231-252, and the
reference-run tile fixtures), and the device PNG encoder by decoding its
files with Pillow + zlib and checking every chunk CRC.  The reference's
Pillow byte stream is not pinned; the decoded image is."""

import struct
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def ref_extract(level: np.ndarray, zoom_level_pixels_unused=None, tx=0, ty=0, tile_px=256):
    src = level[ty * tile_px : (ty + 1) * tile_px, tx * tile_px : (tx + 1) * tile_px]
    canvas = np.zeros((tile_px, tile_px, 4), dtype=np.uint8)
    canvas[: src.shape[0], : src.shape[1]] = src
    return canvas


def check_png(data: bytes, want: np.ndarray):
    """Structure, CRCs, Adler (zlib) and pixels of one PNG file."""
    from PIL import Image
    import io

    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, chunks = 8, []
    while pos < len(data):
        (n,) = struct.unpack(">I", data[pos : pos + 4])
        typ = data[pos + 4 : pos + 8]
        body = data[pos + 8 : pos + 8 + n]
        (crc,) = struct.unpack(">I", data[pos + 8 + n : pos + 12 + n])
        assert crc == zlib.crc32(typ + body), typ
        chunks.append((typ, body))
        pos += 12 + n
    assert [c[0] for c in chunks] == [b"IHDR", b"IDAT", b"IEND"]
    w, h, depth, ctype, comp, filt, inter = struct.unpack(">IIBBBBB", chunks[0][1])
    assert (w, h, depth, ctype, comp, filt, inter) == (want.shape[1], want.shape[0], 8, 6, 0, 0, 0)
    raw = zlib.decompress(chunks[1][1])  # checks the Adler-32
    assert len(raw) == h * (4 * w + 1)
    img = np.array(Image.open(io.BytesIO(data)).convert("RGBA"))
    assert np.array_equal(img, want)


def textures():
    r = np.random.default_rng(3)
    out = []
    # smooth overlay-like: gradient blobs with transparent background
    y, x = np.mgrid[0:700, 0:900]
    a = np.clip(255 - np.hypot(x - 400, y - 300) / 2, 0, 255).astype(np.uint8)
    t = np.zeros((700, 900, 4), np.uint8)
    t[..., 0] = (x * 255 // 899).astype(np.uint8)
    t[..., 1] = (y * 255 // 699).astype(np.uint8)
    t[..., 2] = 128
    t[..., 3] = a
    t[a == 0] = 0
    out.append(t)
    out.append(r.integers(0, 256, size=(300, 520, 4), dtype=np.uint8))  # noise: worst case
    out.append(np.zeros((257, 257, 4), np.uint8))  # all transparent, odd size
    z = np.zeros((64, 2100, 4), np.uint8)  # rows wider than one 256-texel chunk, runs across chunks
    z[:, 1000:1600] = (10, 20, 30, 255)
    z[5, :] = r.integers(0, 256, size=(2100, 4), dtype=np.uint8)
    out.append(z)
    out.append(np.full((1, 1, 4), 7, np.uint8))
    return out


@pytest.mark.parametrize("k", range(5))
def test_encode_png_decodes_to_the_texture(gpu, k):
    import paper_2506_23364_b200 as wf

    t = textures()[k]
    data = wf.encode_png(wf.OverlayTexture(t))
    check_png(data, t)
    assert np.array_equal(np.asarray(wf.decode_png(data).pixels), t)


def test_tiles_of_a_pyramid(gpu):
    """Every tile of every zoom of a colorized runout pyramid: extract_tile ==
    the reference slicing; tile_pngs decode to exactly those tiles."""
    import paper_2506_23364_b200 as wf

    t = textures()[0]
    pyr = wf.build_mipmap(wf.OverlayTexture(t))
    zmax = wf.max_tile_zoom(pyr.width, pyr.height)
    total = 0
    for zoom in range(zmax + 1):
        level = np.asarray(pyr.levels[zmax - zoom].pixels)
        pngs = wf.tile_pngs(pyr, zoom)
        assert len(pngs) == 4 ** zoom
        for (tx, ty), data in pngs.items():
            want = ref_extract(level, tx=tx, ty=ty)
            got = np.asarray(wf.extract_tile(pyr, zoom, tx, ty).pixels)
            assert np.array_equal(got, want)
            check_png(data, want)
            total += 1
    assert total == sum(4 ** z for z in range(zmax + 1))


def test_tile_range_errors(gpu):
    import paper_2506_23364_b200 as wf

    pyr = wf.build_mipmap(wf.OverlayTexture(textures()[2]))
    with pytest.raises(wf.TileRangeError):
        wf.extract_tile(pyr, 3, 0, 0)
    with pytest.raises(wf.TileRangeError):
        wf.tile_pngs(pyr, 1, [(2, 0)])
    with pytest.raises(wf.TileRangeError):
        wf.extract_tile(pyr, 0, 1, 0)


def test_reference_tile_fixtures(gpu, golden_meta, golden_arrays):
    """The reference-run served tiles of the hillshade base layer
    (tests/golden/hillshade_golden.json: extract_tile for tile_px 256 and 64,
    every zoom and tile): device extract_tile and the decoded tile_pngs
    reproduce them."""
    import hashlib
    import io
    import json
    from pathlib import Path

    from PIL import Image

    import paper_2506_23364_b200 as wf
    from paper_2506_23364_b200.terrain import hillshade_pyramid

    cases = json.loads((Path(__file__).resolve().parent / "golden" / "hillshade_golden.json").read_text())["cases"]
    smooth = {f"smooth{c['seed']}": c for c in golden_meta["smooth"]}
    n = 0
    for case in cases:
        if "tiles_sha" not in case:
            continue
        if case["grid"] == "parabola":
            g = wf.gen_parabola()[0]
        else:
            c = smooth[case["grid"]]
            g = wf.DemGrid(ncols=c["ncols"], nrows=c["nrows"], origin_x=c["ox"], origin_y=c["oy"], cellsize=c["cs"],
                           nodata=-9999.0, elevations=golden_arrays[case["array"]])
        pyr = hillshade_pyramid(g, case["azimuth"], case["altitude"])
        by_zoom = {}
        for key, want in case["tiles_sha"].items():
            tile_px, z, tx, ty = map(int, key.split("/"))
            got = np.asarray(wf.extract_tile(pyr, z, tx, ty, tile_px).pixels)
            assert hashlib.sha256(np.ascontiguousarray(got).tobytes()).hexdigest() == want, key
            by_zoom.setdefault((tile_px, z), {})[(tx, ty)] = want
        for (tile_px, z), want in by_zoom.items():
            for (tx, ty), data in wf.tile_pngs(pyr, z, list(want), tile_px).items():
                img = np.array(Image.open(io.BytesIO(data)).convert("RGBA"))
                assert hashlib.sha256(np.ascontiguousarray(img).tobytes()).hexdigest() == want[(tx, ty)]
                n += 1
    assert n > 50

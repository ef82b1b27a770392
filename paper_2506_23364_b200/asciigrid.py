"""ESRI ASCII grid (.asc) reading and writing with the body on the GPU
(reference: /root/reference/pkg/src/demflow/asciigrid.py).

The six header lines are read and written on the host with the reference's
own rules (they are a few dozen bytes); the body -- nrows x ncols numerals,
hundreds of millions at the survey's sizes -- is tokenised, converted and
formatted by csrc/asciigrid.cu:

* ``parse_ascii_grid`` uploads the body bytes once, finds the tokens
  (``str.split()`` semantics) and converts them with CPython ``float()``
  semantics, correctly rounded (wg_numconv.cuh), straight into the device
  elevation raster of the returned ``DemGrid``;
* ``write_ascii_grid`` formats every elevation with ``format_number``'s rules
  (integral values as integers, the rest as the shortest round-trip repr) on
  the device and downloads the text once.

Errors are the reference's ``AsciiGridError`` messages with the same 1-based
line / column positions (computed on the host, on the error path only).
A ``str`` document with non-ASCII characters is first translated one
character for one (``_asciify``), the way CPython's own float() reads text:
Unicode whitespace becomes a space (non-ASCII line boundaries a newline, so
``splitlines`` numbering is kept), Unicode decimal digits their ASCII digit,
anything else a character float() rejects -- so the tokens, values, line /
column positions and rejected tokens are the reference's (``str.split`` /
``float``); byte input must be ASCII.
"""

from __future__ import annotations

import math
import re
import unicodedata

import numpy as np
import torch

from . import _device, _lib
from .grid import DemGrid, GridError

_HEADER_KEYS = ("ncols", "nrows", "xllcorner", "yllcorner", "cellsize", "nodata_value")
_CANONICAL_KEYS = ("ncols", "nrows", "xllcorner", "yllcorner", "cellsize", "NODATA_value")
# str.splitlines() boundaries within ASCII (\r\n counts once)
_LINE_BREAK = re.compile(rb"\r\n|[\n\r\x0b\x0c\x1c\x1d\x1e]")
_NO_BAD = (1 << 64) - 1

__all__ = ["AsciiGridError", "parse_ascii_grid", "write_ascii_grid", "write_ascii_grid_bytes", "format_number"]


class AsciiGridError(ValueError):
    """Parse failure; line and column are 1-based document positions
    (asciigrid.py:29-39)."""

    def __init__(self, message: str, line: int | None = None, column: int | None = None):
        if line is not None:
            where = f"line {line}"
            if column is not None:
                where += f", column {column}"
            message = f"{message} ({where})"
        super().__init__(message)
        self.line = line
        self.column = column


def format_number(v: float) -> str:
    """Shortest numeral that round-trips: bare integers, repr otherwise
    (asciigrid.py:160-167; header values -- the body uses the device twin)."""
    f = float(v)
    if f == int(f) and abs(f) < 1e16:
        return str(int(f))
    return repr(f)


# str.splitlines() boundaries outside ASCII
_UNICODE_LINE_BREAKS = frozenset("\x85\u2028\u2029")


def _asciify(text: str) -> bytes:
    """One ASCII byte per character of `text`, with the structure str.split /
    str.splitlines / float() see in it: non-ASCII line boundaries -> '\\n',
    other Unicode whitespace -> ' ', Unicode decimal digits -> their ASCII
    digit (float() converts them: CPython's _PyUnicode_TransformDecimalAndSpaceToASCII),
    any other non-ASCII character -> '?' (which float() rejects, as it
    rejects the character).  Offsets are preserved, so positions and
    offending tokens map back to the original text."""
    table = {}
    for ch in set(text):
        if ch.isascii():
            continue
        if ch in _UNICODE_LINE_BREAKS:
            table[ord(ch)] = "\n"
        elif ch.isspace():
            table[ord(ch)] = " "
        else:
            d = unicodedata.decimal(ch, None)
            table[ord(ch)] = str(d) if d is not None else "?"
    return text.translate(table).encode("ascii")


def _as_bytes(text):
    if isinstance(text, (bytes, bytearray)):
        return text
    if isinstance(text, memoryview):
        return text if text.contiguous and text.format in ("B", "b", "c") else text.tobytes()
    if not text.isascii():
        return _asciify(text)
    return text.encode("ascii")


def _count_lines(data: bytes) -> int:
    """len(text.splitlines()) for an ASCII document."""
    breaks = (data.count(b"\n") + data.count(b"\r") - data.count(b"\r\n") + data.count(b"\x0b")
              + data.count(b"\x0c") + data.count(b"\x1c") + data.count(b"\x1d") + data.count(b"\x1e"))
    if data and not _LINE_BREAK.fullmatch(data[-2:] if data.endswith(b"\r\n") else data[-1:]):
        breaks += 1
    return breaks


def _line_col(data: bytes, off: int) -> tuple[int, int]:
    """1-based line and column of byte `off` (splitlines numbering)."""
    line_start = 0
    line = 1
    for m in _LINE_BREAK.finditer(data, 0, off):
        line += 1
        line_start = m.end()
    return line, off - line_start + 1


def _header(data: bytes) -> tuple[dict, int, list[bytes]]:
    """The six header lines (asciigrid.py:44-85 restated); returns the values,
    the body's byte offset and the header lines."""
    lines: list[bytes] = []
    pos = 0
    for m in _LINE_BREAK.finditer(data):
        lines.append(data[pos:m.start()])
        pos = m.end()
        if len(lines) == 6:
            break
    body_off = pos
    if len(lines) < 6:
        if pos < len(data):  # a last header line without a line break
            lines.append(data[pos:])
            body_off = len(data)
        if len(lines) < 6:
            raise AsciiGridError(f"expected 6 header lines, document has {len(lines)}", line=len(lines) or 1)
    header: dict[str, float] = {}
    for idx, want in enumerate(_HEADER_KEYS):
        text = lines[idx].decode("ascii")
        parts = text.split()
        if len(parts) != 2:
            raise AsciiGridError(f"header line must be 'key value', got {text!r}", line=idx + 1)
        key, value = parts
        if key.lower() != want:
            raise AsciiGridError(f"expected header key {want!r}, got {key!r}", line=idx + 1)
        col = text.index(value, len(key)) + 1
        if want in ("ncols", "nrows"):
            try:
                header[want] = int(value)
            except ValueError:
                raise AsciiGridError(f"{want} must be an integer, got {value!r}", line=idx + 1, column=col) from None
            if header[want] <= 0:
                raise AsciiGridError(f"{want} must be positive, got {value!r}", line=idx + 1, column=col)
        else:
            try:
                header[want] = float(value)
            except ValueError:
                raise AsciiGridError(f"{want} must be a number, got {value!r}", line=idx + 1, column=col) from None
            if not math.isfinite(header[want]):
                raise AsciiGridError(f"{want} must be finite, got {value!r}", line=idx + 1, column=col)
    return header, body_off, lines


def parse_ascii_grid(text: str | bytes) -> DemGrid:
    """Parse an ASCII grid document into a device-resident DemGrid
    (asciigrid.py:42-143)."""
    data = _as_bytes(text)
    original = text if isinstance(text, str) and not text.isascii() else None  # for offending tokens
    if isinstance(data, memoryview):
        head = bytes(data[: 1 << 16])
        try:
            header, body_off, lines = _header(head)
        except AsciiGridError:
            header = None
        if header is None or (len(lines) == 6 and body_off == len(head) < len(data)):
            head = bytes(data)  # a header longer than 64 KiB: read it from the whole document
            header, body_off, _ = _header(head)
        full = lambda: bytes(data)  # noqa: E731  (error paths only)
    else:
        header, body_off, _ = _header(data)
        full = lambda: data  # noqa: E731
    ncols, nrows = int(header["ncols"]), int(header["nrows"])
    expected = ncols * nrows
    L = _lib.lib()
    dev = _device.device()
    n = len(data)
    # a body of m bytes holds at most (m + 1) // 2 tokens: a header that
    # promises more cannot be satisfied, and must not size the allocations
    # (the reader then only counts, and the reference's message follows)
    cap = min(expected, (n - body_off + 1) // 2)
    t = _device.upload(np.frombuffer(data, dtype=np.uint8))
    values = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    info = torch.empty(4, dtype=torch.int64, device=dev)
    scratch = torch.empty(int(L.wg_ascii_read_scratch_bytes(n, cap)), dtype=torch.uint8, device=dev)
    _lib.check(L.wg_ascii_read(_lib.ptr(t), n, body_off, _lib.ptr(values), cap, _lib.ptr(info),
                               _lib.ptr(scratch), _lib.stream_ptr()), AsciiGridError)
    found, nonascii, extra_off, bad_off = (v & _NO_BAD for v in _device.read_small(info))
    if nonascii:
        raise AsciiGridError("document is not ASCII")
    if found != expected:
        if found < expected:
            raise AsciiGridError(f"expected {expected} elevation values, found {found}",
                                 line=_count_lines(full()))
        line, col = _line_col(full(), extra_off)
        raise AsciiGridError(f"expected {expected} elevation values, found {found}", line=line, column=col)
    if bad_off != _NO_BAD:
        data = full()
        end = bad_off
        while end < n and data[end:end + 1] not in (b" ", b"\t", b"\n", b"\x0b", b"\x0c", b"\r", b"\x1c", b"\x1d",
                                                       b"\x1e", b"\x1f"):
            end += 1
        line, col = _line_col(data, bad_off)
        token = original[bad_off:end] if original is not None else data[bad_off:end].decode("ascii")
        raise AsciiGridError(f"invalid elevation value {token!r}", line=line, column=col)
    del t, scratch
    try:
        return DemGrid.adopt(ncols, nrows, header["xllcorner"], header["yllcorner"], header["cellsize"],
                             header["nodata_value"], values.view(nrows, ncols))
    except GridError as exc:
        raise AsciiGridError(str(exc)) from exc


def write_ascii_grid_bytes(grid: DemGrid) -> memoryview:
    """The canonical ASCII grid document as a bytes-like buffer (body
    formatted on the GPU); write it to a file or pass it to
    ``parse_ascii_grid`` without a copy."""
    header_values = (grid.ncols, grid.nrows, grid.origin_x, grid.origin_y, grid.cellsize, grid.nodata)
    head = "".join(f"{key} {format_number(val)}\n" for key, val in zip(_CANONICAL_KEYS, header_values)).encode()
    L = _lib.lib()
    v = grid.device_elevations().contiguous().view(-1)
    count = v.numel()
    scratch = _device.empty((int(L.wg_ascii_format_scratch_bytes(count)),), torch.uint8)
    nb = _device.empty((1,), torch.int64)
    cap = int(L.wg_ascii_format_capacity(count))
    full = _device.empty((len(head) + cap,), torch.uint8)  # upper bound; the used prefix is downloaded
    full[: len(head)].copy_(torch.tensor(list(head), dtype=torch.uint8))
    _lib.check(L.wg_ascii_format(_lib.ptr(v), count, grid.ncols, _lib.ptr(full[len(head):]), cap, _lib.ptr(nb),
                                 _lib.ptr(scratch), _lib.stream_ptr()))
    nbytes = int(_device.read_small(nb)[0])
    out = full[: len(head) + nbytes]
    # staged through pinned chunks by a thread pool (_device.download): a
    # single pageable copy into fresh host memory is bound by first-touch
    # page faults at multi-GB sizes (tools/host_xfer_probe.py)
    buf = _device.download(out)
    return memoryview(buf)


def write_ascii_grid(grid: DemGrid) -> str:
    """Serialize a DemGrid to the canonical ASCII grid text
    (asciigrid.py:146-157)."""
    return str(write_ascii_grid_bytes(grid), "ascii")


def read_ascii_grid(path) -> DemGrid:
    """Parse the ASCII grid file at `path` (bytes read straight from disk)."""
    with open(path, "rb") as f:
        return parse_ascii_grid(f.read())


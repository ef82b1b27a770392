"""Throughput of the executor's device digest (csrc/digest.cu) on a 2 GiB
f64 raster (the C3 DEM size), contiguous and as a strided window; CUDA events,
best of 5.  Prints one JSON line.  Usage: python tools/bench_digest.py"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2506_23364_b200 import _lib  # noqa: E402


def timed(t, rows, row_bytes, ld):
    L = _lib.lib()
    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    ms = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(L.wg_digest2d(t.data_ptr(), rows, row_bytes, ld, out.data_ptr(), _lib.stream_ptr()))
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return min(ms[1:])


def main():
    _lib.build()
    n = 16384
    x = torch.empty((n, n), dtype=torch.float64, device="cuda").uniform_()
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    ms = timed(x, n, n * 8, n * 8)
    w = x[:, 1:n - 1]  # strided window (rows 8-byte aligned, a partial last tile)
    msw = timed(w, n, (n - 2) * 8, n * 8)
    w2 = x[:, 16:n - 1008]  # strided window of whole tiles, 128-byte aligned rows
    msw2 = timed(w2, n, (n - 1024) * 8, n * 8)
    gbs = n * n * 8 / ms / 1e6
    print(json.dumps({"metric": "digest GB/s", "bytes": n * n * 8, "contiguous_ms": ms, "contiguous_gbs": gbs,
                      "window_ms": msw, "window_gbs": n * (n - 2) * 8 / msw / 1e6,
                      "window_tiles_gbs": n * (n - 1024) * 8 / msw2 / 1e6, "peak_gbs": peak,
                      "frac": gbs / peak}))


if __name__ == "__main__":
    main()

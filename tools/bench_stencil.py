"""Kernel times of the raster stencil at C3 size (16384^2 synth_dem):
normals (+ fused slope), normals alone, steepness from normals; CUDA events,
best of 5, with the algorithmic HBM bytes.  Usage: python tools/bench_stencil.py"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2506_23364_b200 import _lib  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402


def best(fn, reps=6):
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return min(ms[1:])


def main():
    L = _lib.lib()
    n = 16384
    e = synth_dem_device(n, 0)
    nrm = torch.empty((n, n, 3), dtype=torch.float64, device="cuda")
    slope = torch.empty((n, n), dtype=torch.float64, device="cuda")
    s = _lib.stream_ptr
    res = {}
    res["normals+slope_ms"] = best(lambda: _lib.check(L.wg_normals(e.data_ptr(), n, n, 10.0, 20.0, nrm.data_ptr(),
                                                                    slope.data_ptr(), s())))
    res["normals_ms"] = best(lambda: _lib.check(L.wg_normals(e.data_ptr(), n, n, 10.0, 20.0, nrm.data_ptr(), None, s())))
    res["slope_only_ms"] = best(lambda: _lib.check(L.wg_normals(e.data_ptr(), n, n, 10.0, 20.0, None,
                                                                 slope.data_ptr(), s())))
    res["steepness_ms"] = best(lambda: _lib.check(L.wg_steepness(nrm.data_ptr(), n * n, slope.data_ptr(), s())))
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    cells = n * n
    for k, b in (("normals+slope_ms", 40), ("normals_ms", 32), ("slope_only_ms", 16), ("steepness_ms", 32)):
        res[k.replace("_ms", "_frac")] = cells * b / (res[k] / 1e3) / 1e9 / peak
    print(json.dumps(res))


if __name__ == "__main__":
    main()

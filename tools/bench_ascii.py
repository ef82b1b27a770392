"""Measurement of the ASCII grid row at C3 size:
write and parse a synth_dem(16384, 0) document (every value a 13-17 digit
repr) on the GPU, kernel-only (device-resident text / values, CUDA events)
and end to end (host bytes in / host bytes out), with the reference
algorithm (oracle/asciigrid_ref.py) timed on the host cores on a 1024^2
sample beside it.  Prints one JSON line.  Usage: python tools/bench_ascii.py
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200 import _device, _lib, asciigrid  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402


def events():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    return a, b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-size", type=int, default=1024)
    a = ap.parse_args()
    _lib.build()
    L = _lib.lib()
    n = a.size
    g = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, 0))
    count = n * n

    # ---- writer: kernels only (values resident, text stays on the device)
    v = g.device_elevations().view(-1)
    scratch = _device.empty((int(L.wg_ascii_format_scratch_bytes(count)),), torch.uint8)
    nb = _device.empty((1,), torch.int64)
    cap = int(L.wg_ascii_format_capacity(count))
    body = _device.empty((cap,), torch.uint8)
    wt = []
    for _ in range(a.reps + 1):
        e0, e1 = events()
        e0.record()
        L.wg_ascii_format(_lib.ptr(v), count, n, _lib.ptr(body), cap, _lib.ptr(nb), _lib.ptr(scratch),
                          _lib.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        wt.append(e0.elapsed_time(e1))
    write_ms = min(wt[1:])
    nbytes = int(_device.read_small(nb)[0])
    del scratch, body

    # ---- writer end to end: DemGrid -> bytes on the host
    # (first call: includes the one-time pinned staging ring of _device)
    we = []
    for _ in range(2):
        t0 = time.perf_counter()
        doc = asciigrid.write_ascii_grid_bytes(g)
        we.append((time.perf_counter() - t0) * 1e3)
    write_e2e_first_ms, write_e2e_ms = we[0], min(we)

    # ---- reader: kernels only (text resident on the device)
    head_len = len(doc) - nbytes
    t = _device.upload(np.frombuffer(doc, dtype=np.uint8))
    info = _device.empty((4,), torch.int64)
    sc = _device.empty((int(L.wg_ascii_read_scratch_bytes(len(doc), count)),), torch.uint8)
    vals = _device.empty((count,), torch.float64)
    pt = []
    for _ in range(a.reps + 1):
        e0, e1 = events()
        e0.record()
        L.wg_ascii_read(_lib.ptr(t), len(doc), head_len, _lib.ptr(vals), count, _lib.ptr(info), _lib.ptr(sc),
                        _lib.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        pt.append(e0.elapsed_time(e1))
    parse_ms = min(pt[1:])
    assert int(_device.read_small(info)[0]) == count
    assert torch.equal(vals.view(torch.int64), v.view(torch.int64)), "parse(write(g)) != g"
    del t, sc, vals

    # ---- reader end to end: host bytes -> DemGrid (incl. H2D + validation)
    pe = []
    for _ in range(2):
        t0 = time.perf_counter()
        h = asciigrid.parse_ascii_grid(doc)
        torch.cuda.synchronize()
        pe.append((time.perf_counter() - t0) * 1e3)
    parse_e2e_ms = min(pe)
    assert torch.equal(h.device_elevations().view(-1).view(torch.int64), v.view(torch.int64))

    # ---- CPU baseline: the reference algorithm on a sample, host cores
    from oracle import asciigrid_ref

    m = a.cpu_size
    sample = g.device_elevations()[:m, :m].cpu().numpy()
    t0 = time.perf_counter()
    text = asciigrid_ref.write_text((m, m, 0.0, 0.0, 10.0, -9999.0), sample)
    cpu_write_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    back = asciigrid_ref.parse_body(text, m, m)
    cpu_parse_s = time.perf_counter() - t0
    assert np.array_equal(back, sample)

    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    text_b = len(doc)
    parse_bytes = text_b + 8 * count  # algorithmic: read the text, write the values
    write_bytes = 8 * count + nbytes  # read the values, write the text
    line = {
        "metric": "ascii grid values/s", "unit": "values/s", "config": {
            "workload": f"synth_dem({n}, 0) as canonical ESRI ASCII grid ({text_b / 1e9:.2f} GB, "
                        f"{count} values, {text_b / count:.1f} B/value)"},
        "parse": {"kernel_ms": parse_ms, "value": count / (parse_ms / 1e3), "e2e_ms": parse_e2e_ms,
                  "e2e_value": count / (parse_e2e_ms / 1e3),
                  "roofline": {"bound": "hbm", "achieved": parse_bytes / (parse_ms / 1e3) / 1e9, "peak": peak,
                               "unit": "GB/s", "frac": parse_bytes / (parse_ms / 1e3) / 1e9 / peak,
                               "bytes_per_unit": parse_bytes / count}},
        "write": {"kernel_ms": write_ms, "value": count / (write_ms / 1e3), "e2e_ms": write_e2e_ms,
                  "e2e_value": count / (write_e2e_ms / 1e3),
                  "e2e_first_call_ms": write_e2e_first_ms,
                  "roofline": {"bound": "hbm", "achieved": write_bytes / (write_ms / 1e3) / 1e9, "peak": peak,
                               "unit": "GB/s", "frac": write_bytes / (write_ms / 1e3) / 1e9 / peak,
                               "bytes_per_unit": write_bytes / count}},
        "cpu_baseline": {"kind": "port", "cores": 1, "sample": f"{m}x{m} values of the same DEM, oracle/asciigrid_ref.py "
                         "(the reference's str.split + np.array / format_number join)",
                         "parse_value": m * m / cpu_parse_s, "write_value": m * m / cpu_write_s, "unit": "values/s"},
        "roundtrip": "parse(write(g)) == g bitwise on the device",
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()

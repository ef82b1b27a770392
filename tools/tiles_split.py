"""Host-side split of overlay.tile_pngs on the stock 8192^2 overlay pyramid
(zoom 5, 1024 tiles): allocation, kernels, length readback, packing, D2H and
bytes objects.  usage: python tools/tiles_split.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200 import _device, _lib, overlay  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402

n = 8192
dem = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, 1))
g = wf.build_avalanche_graph(dem.extent, wf.AvalancheParams(particles_per_release_cell=256, seed=0),
                             wf.SteepnessRelease(30.0, 45.0, stride=16), zoom=2)
g.bind("world", dem)
pyr = wf.Executor().execute(g).value("avalanche_overlay", "overlay")
L = _lib.lib()
zmax = overlay.max_tile_zoom(pyr.width, pyr.height, 256)
for rep in range(3):
    t = [time.perf_counter()]
    tiles = [(tx, ty) for ty in range(32) for tx in range(32)]
    level = pyr.levels[zmax - 5].dev("pixels").contiguous()
    cap = int(L.wg_png_capacity(256, 256))
    txy = torch.tensor([v for p in tiles for v in p], dtype=torch.int32).to(level.device)
    out = _device.empty((cap * len(tiles),), torch.uint8)
    lens = _device.empty((len(tiles),), torch.int64)
    scratch = _device.empty((int(L.wg_png_scratch_bytes(256, 256, len(tiles))),), torch.uint8)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    L.wg_png_tiles(_lib.ptr(level), int(level.shape[1]), int(level.shape[0]), 256, _lib.ptr(txy), len(tiles),
                   _lib.ptr(out), cap, _lib.ptr(lens), _lib.ptr(scratch), _lib.stream_ptr())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    ln = lens.cpu().tolist()
    t.append(time.perf_counter())
    packed = torch.cat([out[i * cap: i * cap + k] for i, k in enumerate(ln)])
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    host = _device.download(packed)
    t.append(time.perf_counter())
    res, off = [], 0
    for k in ln:
        res.append(host[off: off + k].tobytes())
        off += k
    t.append(time.perf_counter())
    names = ["alloc", "kernels", "lens", "pack(cat)", "download", "bytes"]
    print({nm: round((t[i + 1] - t[i]) * 1e3, 2) for i, nm in enumerate(names)},
          "MB", round(sum(ln) / 1e6, 1), "scratch GB", round(scratch.numel() / 1e9, 2), "out GB",
          round(out.numel() / 1e9, 2))

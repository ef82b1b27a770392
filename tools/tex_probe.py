"""Texture kernels on the C4 overlay's own data: the stitched 8192^2 world's
runout raster (stock graph inputs: band 30-45, stride 16, 256 particles per
cell), then colorize and the full mip pyramid timed with CUDA events over
REPS launches each (min / median ms, fraction of the measured HBM peak at the
algorithmic bytes: colorize 12 B/texel, mip 4 B/texel read + 4/3 B written).
usage: python tools/tex_probe.py [--reps 20]"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200 import overlay  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402


def timed(fn, reps):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    n = 8192
    world = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, 1))
    g = wf.build_avalanche_graph(world.extent, wf.AvalancheParams(particles_per_release_cell=256, seed=0),
                                 wf.SteepnessRelease(30.0, 45.0, stride=16), zoom=2)
    g.bind("world", world)
    res = wf.Executor().execute(g)
    run = res.value("avalanche_overlay", "runout")
    tex = overlay.colorize(run, wf.DEFAULT_RUNOUT_COLORMAP)
    col = timed(lambda: overlay.colorize(run, wf.DEFAULT_RUNOUT_COLORMAP), a.reps)
    mip = timed(lambda: overlay.build_mipmap(tex), a.reps)
    peak = 6551.0
    try:
        peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:  # noqa: BLE001
        pass
    texels = n * n
    digest = int(torch.as_tensor(overlay.build_mipmap(tex).levels[3].pixels).to(torch.int64).sum())
    out = {"colorize_ms": [round(min(col), 4), round(statistics.median(col), 4)],
           "colorize_hbm_frac": round(12 * texels / (min(col) * 1e-3) / 1e9 / peak, 3),
           "mip_ms": [round(min(mip), 4), round(statistics.median(mip), 4)],
           "mip_hbm_frac": round((4 + 4 / 3) * texels / (min(mip) * 1e-3) / 1e9 / peak, 3),
           "level3_sum": digest}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

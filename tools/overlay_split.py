"""Wall-clock split of the avalanche_overlay op on the stitched 8192^2 world
(host time between synchronised stages) to find host-side gaps.
usage: python tools/overlay_split.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200 import overlay, simulate, workflow  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402

marks = []


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        marks.append((name, round((t1 - t0) * 1e3, 3), round((t2 - t0) * 1e3, 3)))
        return r
    setattr(mod, name, g)


from paper_2506_23364_b200 import _device  # noqa: E402

for mod, name in ((simulate, "_try_empty"), (_device, "empty"), (simulate, "build_quad"), (workflow, "run_avalanche"), (workflow, "colorize"), (workflow, "build_mipmap"),
                  (workflow, "avalanche_stats"), (simulate, "release_cells"), (simulate, "build_gather_layout"),
                  (simulate, "run_avalanche_device")):
    if hasattr(mod, name):
        wrap(mod, name)

world = wf.DemGrid.adopt(8192, 8192, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(8192, 1))
for rep in range(3):
    marks.clear()
    g = wf.build_avalanche_graph(world.extent, wf.AvalancheParams(particles_per_release_cell=256, seed=rep),
                                 wf.SteepnessRelease(30.0, 45.0, stride=16), zoom=2)
    g.bind("world", world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = wf.Executor().execute(g)
    ms = (time.perf_counter() - t0) * 1e3
print(f"execute {ms:.2f} ms", {r.node_id: round(r.elapsed_ms, 3) for r in res.report.records})
for m in marks:
    if m[2] > 0.05:
        print("  %-24s host %8.3f ms  +device %8.3f ms" % m)
print("allocator", {k: v for k, v in torch.cuda.memory_stats().items()
                    if k in ("num_alloc_retries", "num_device_alloc", "num_device_free", "num_sync_all_streams")})

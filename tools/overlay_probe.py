"""Run the stock avalanche graph on a stitched 8192^2 synthetic world once
(warm) and print per-node times; used under ncu for the overlay launch list.
usage: python tools/overlay_probe.py [n] [stride] [ppc] [reps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ppc = int(sys.argv[3]) if len(sys.argv) > 3 else 256
world = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, 1))
for rep in range(int(sys.argv[4]) if len(sys.argv) > 4 else 3):
    g = wf.build_avalanche_graph(world.extent, wf.AvalancheParams(particles_per_release_cell=ppc, seed=rep),
                                 wf.SteepnessRelease(30.0, 45.0, stride=stride), zoom=2)
    g.bind("world", world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = wf.Executor().execute(g)
    ms = (time.perf_counter() - t0) * 1e3
    print(f"rep {rep} cold {ms:.2f} ms", {r.node_id: round(r.elapsed_ms, 3) for r in res.report.records})

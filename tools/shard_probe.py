"""Trajectory-kernel time of one rank's share vs the full run, with and
without the touched-tile map, repeated in alternating order (separates the
cost of the map from that of the band partition and from first-launch
effects).  usage: python tools/shard_probe.py [--config c3|c5] [--world 2] [--reps 3]"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200 import shard  # noqa: E402
from paper_2506_23364_b200.simulate import release_cells, release_mask_from_dem, run_avalanche_device  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["c3", "c5"], default="c3")
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n, stride, seed = (16384, 32, 0) if a.config == "c3" else (65536, 128, 2)
    grid = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, seed))
    cells = release_cells(release_mask_from_dem(grid, 30.0, 45.0, stride))
    params = wf.AvalancheParams(particles_per_release_cell=2048, seed=seed)
    plan = shard.plan_bands(n, n, a.world)
    offs = shard.band_cell_offsets(cells, plan)
    hits = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    zmax = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    touched = torch.zeros((plan.tiles_y, plan.tiles_x), dtype=torch.uint8, device="cuda")
    cases = {"full": None}
    for r in range(a.world):
        cases[f"rank{r}"] = shard.particle_ranges(offs, plan, r, 2048)
    # a contiguous half of the index space, for comparison with the bands
    total = int(cells.numel()) * 2048
    cases["first_half"] = [(0, total // 2 // 2048 * 2048)]
    out = {k: {"plain": [], "touch": []} for k in cases}
    for _ in range(a.reps):
        for name, ranges in cases.items():
            for mode in ("plain", "touch"):
                hits.zero_()
                zmax.zero_()
                touched.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                run_avalanche_device(grid, cells, params, ranges=ranges, hits=hits, zmax=zmax,
                                     touched=touched if mode == "touch" else None, plan=plan, rank=max(
                                         0, int(name[4:]) if name.startswith("rank") else 0))
                e1.record()
                torch.cuda.synchronize()
                steps = int(hits.sum().item()) - sum(hi - lo for lo, hi in (ranges or [(0, total)]))
                out[name][mode].append((round(e0.elapsed_time(e1), 2), round(steps / e0.elapsed_time(e1) / 1e6, 1)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""One-GPU simulation of the multi-GPU split (shard.py) at C3 or C5: for
N = 2, 4, 8 every rank's release-row bands run in turn on this GPU into
private rasters with their touched-tile map; per rank it reports the
trajectory-kernel time and particle steps (load balance), and the foreign
tiles it would send (merge bytes per rank vs the dense raster pair).  The
ranks' kernels run one after another, so their times are independent
measurements of each rank's share -- no collective is exercised here (the
exchange itself is tested in tests/test_gpu_c5.py and test_gpu_multirank.py).

usage: python tools/shard_sim.py [--config c3|c5] [--ns 2,4,8] [--bands-per-rank 4]
"""

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


def timed(fn) -> float:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["c3", "c5"], default="c3")
    ap.add_argument("--ns", default="2,4,8")
    ap.add_argument("--bands-per-rank", type=int, default=shard.BANDS_PER_RANK)
    a = ap.parse_args()
    n, stride, seed = (16384, 32, 0) if a.config == "c3" else (65536, 128, 2)
    grid = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, seed))
    cells = release_cells(release_mask_from_dem(grid, 30.0, 45.0, stride))
    params = wf.AvalancheParams(particles_per_release_cell=2048, seed=seed)
    hits = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    zmax = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    run_avalanche_device(grid, cells, params, hits=hits, zmax=zmax)  # warm (builds the gather layout)
    hits.zero_()
    zmax.zero_()
    full_ms = timed(lambda: run_avalanche_device(grid, cells, params, hits=hits, zmax=zmax))
    total_steps = int(hits.sum().item()) - int(cells.numel()) * 2048
    out = {"config": a.config, "n": n, "stride": stride, "release_cells": int(cells.numel()),
           "particle_steps": total_steps, "one_gpu_traj_ms": full_ms, "bands_per_rank": a.bands_per_rank,
           "dense_bytes": n * n * 16, "splits": {}}
    for world in (int(x) for x in a.ns.split(",")):
        plan = shard.plan_bands(n, n, world, a.bands_per_rank)
        offs = shard.band_cell_offsets(cells, plan)
        touched = torch.zeros((plan.tiles_y, plan.tiles_x), dtype=torch.uint8, device="cuda")
        ranks = []
        for r in range(world):
            hits.zero_()
            zmax.zero_()
            touched.zero_()
            ranges = shard.particle_ranges(offs, plan, r, 2048)
            ms = timed(lambda: run_avalanche_device(grid, cells, params, ranges=ranges, hits=hits, zmax=zmax,
                                                    touched=touched, plan=plan, rank=r))
            particles = shard.local_particles(ranges)
            steps = int(hits.sum().item()) - particles
            ids, nt = shard.touched_tiles(touched)
            toffs = shard._sorted_offsets(ids, nt, plan.tile_bounds())
            _, counts = shard.exchange_segments(toffs, plan, r)
            sent = sum(counts) * 2 * plan.tile * plan.tile * 8
            ranks.append({"traj_ms": round(ms, 2), "particles": particles, "steps": steps,
                          "touched_tiles": nt, "sent_tiles": sum(counts), "sent_bytes": sent,
                          "sent_frac_of_dense": round(sent / (n * n * 16), 4)})
        slowest = max(x["traj_ms"] for x in ranks)
        out["splits"][str(world)] = {
            "band_rows": plan.band_rows, "nbands": plan.nbands, "ranks": ranks,
            "max_rank_traj_ms": slowest, "traj_speedup_vs_1gpu": round(full_ms / slowest, 2),
            "traj_efficiency": round(full_ms / slowest / world, 3),
            "steps_imbalance_max_over_mean": round(max(x["steps"] for x in ranks)
                                                  / (sum(x["steps"] for x in ranks) / world), 3),
            "max_sent_frac_of_dense": max(x["sent_frac_of_dense"] for x in ranks),
        }
        print(json.dumps({world: out["splits"][str(world)]["traj_efficiency"]}), file=sys.stderr)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

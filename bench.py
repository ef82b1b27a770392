"""Benchmark: trajectory steps/sec (+ overlay latency) of the avalanche hot
path on a synthetic 16384^2 DEM (BASELINE.json configs[2]), B200 vs host CPU.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

One step = one pass of the hot path over the DEM: fused normals+steepness ->
release_points (band 30-45 deg, stride 32) -> release ordinal compaction ->
avalanche trajectories (2048 particles per release cell, default physics) ->
runout invariants + stats.  Multi-GPU: the particles are sharded by
release-row bands (cyclic over ranks); each rank's private rasters are merged
tile-sparsely into the band owners by an NCCL all-to-all of the touched
foreign tiles (strong scaling: total work fixed).

value: device-resident inputs.  e2e: the same metric through the public API
(DemGrid from a pinned host array -> compute_normals -> steepness_deg ->
detect_release_points -> run_avalanche -> host read of the RunoutRaster),
host<->device copies inside the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "trajectory steps/sec"
UNIT = "particle-steps/s"
BYTES_PER_STEP = 64  # 32 B DEM patch + 16 B hit RMW + 16 B drop RMW
# FP64-pipe instructions per particle-step (DFMA+DMUL+DADD+DSETP per active
# thread) from the ncu SASS capture of traj_kernel (profiles/r01_traj_ncu_summary.txt),
# and the measured FP64 instruction peak (profiles/fp64_peak.json, DADD/DMUL rate)
FP64_OPS_PER_STEP = 168  # 143 DFMA+DMUL+DADD + 25 DSETP (ncu source page, round-2 final build)
FP64_PEAK_OPS = 1.853e13
# the step's memory operations alone (one 32-B gather + RED.ADD.64 + RED.MAX.64
# to random slots of a 96 MiB L2-resident working set, 32 warps/SM): the L2
# access-rate ceiling of a trajectory step (tools/micro/l2_peak.cu, profiles/l2_peak.json)
L2_STEP_PEAK = 6.7024e10
# DRAM bytes per traj_kernel launch from ncu --set full (dram__bytes_read+write, r01)
TRAJ_DRAM_BYTES = 6.60e9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--stride", type=int, default=32)
    ap.add_argument("--ppc", type=int, default=2048)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-chunks", type=int, default=8192, help="2048-particle chunks in the CPU sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-overlay", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", choices=["c3", "c5"], default="c3",
                    help="c3: 16384^2 stride 32 (default, BASELINE configs[2]); "
                         "c5: 65536^2 stride 128 seed 2 (configs[4]; lattice-slope mask prefix, no e2e/CPU legs)")
    ap.add_argument("--overlay-size", type=int, default=8192)
    a = ap.parse_args()
    a.slope_only = False
    if a.config == "c5":
        # 65536^2: DEM 32 GiB + slope 32 GiB + rasters 64 GiB; the 96 GiB
        # normal field would not fit next to them, so the prefix computes
        # the slope field directly (same arithmetic, normals not stored)
        a.size, a.stride, a.seed = 65536, 128, 2
        a.slope_only = a.no_e2e = a.no_cpu = a.no_overlay = True
    return a


def workload(a) -> dict:
    if a.config == "c5":
        which = "BASELINE configs[4], mask from the slope at lattice cells"
    elif (a.size, a.stride, a.ppc, a.seed) == (16384, 32, 2048, 0):
        which = "BASELINE configs[2]"
    else:
        which = f"non-BASELINE size: stride {a.stride}, {a.ppc} particles per cell"
    gib = a.size * a.size * 8 / 2**30
    return {
        "workload": f"avalanche release points + trajectories, synthetic {a.size}x{a.size} DEM ({which})",
        "dem": f"synth_dem({a.size}, seed={a.seed}, cs=10, H=300, lambda0=4000, 4 octaves)",
        "release": f"SteepnessRelease(30, 45, stride={a.stride})",
        "params": f"AvalancheParams(particles_per_release_cell={a.ppc}, seed={a.seed}) (defaults: p=0.9, r=0.16, alpha=25)",
        "l2": (f"inputs larger than L2 (DEM {gib:g} GiB, rasters {2 * gib:g} GiB per step)" if a.size >= 8192
               else "inputs may fit in L2"),
    }


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, float, str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), ",".join(parts[3:7])))
                except ValueError:
                    pass

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, flags in self.samples:
            for n, f in zip(names, flags.split(",")):
                if f.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples)}


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "src": "measured (MEASURED_PEAKS.json)", "sm_max_mhz": d.get("sm_max_mhz")}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0}


# ------------------------------------------------------------------ CPU side


def cpu_sample(elev: np.ndarray, mask: np.ndarray, a, chunks: int, threads: int | None = None) -> dict:
    """The oracle port (oracle/traj_oracle.c, the reference's engine restated
    in C) over `chunks` evenly spaced 2048-particle chunks of the workload,
    all host threads, bit-identical work to the GPU's for those particles."""
    from oracle import traj

    cells = np.ascontiguousarray(np.flatnonzero(mask.ravel()), dtype=np.int64)
    total = cells.size * a.ppc
    nchunks = (total + 2047) // 2048
    pick = np.unique(np.linspace(0, nchunks - 1, min(chunks, nchunks)).astype(np.int64))
    threads = threads or os.cpu_count() or 1
    hits = np.zeros(elev.shape, dtype=np.int64)
    zmax = np.zeros(elev.shape, dtype=np.float64)
    steps = 0
    t = 0.0
    for c in pick:
        lo, hi = int(c) * 2048, min(int(c) * 2048 + 2048, total)
        t0 = time.perf_counter()
        steps += traj.run_range(elev, 0.0, 0.0, 10.0, cells, lo, hi, hits, zmax, particles_per_release_cell=a.ppc,
                                seed=a.seed, threads=threads)
        t += time.perf_counter() - t0
    return {"value": steps / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(pick)} evenly spaced 2048-particle chunks of {nchunks} ({steps} steps, {t:.1f} s), "
                      f"C oracle (oracle/traj_oracle.c) of the reference engine, {threads} threads",
            "seconds": t, "steps": steps}


def host_inputs(a):
    from oracle import npref

    from paper_2506_23364_b200.synth import synth_dem_host

    e = synth_dem_host(a.size, a.seed)
    m = npref.lattice_release_mask(e, 10.0, 30.0, 45.0, a.stride)
    return e, m


def run_reference(a) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    e, m = host_inputs(a)
    vals = []
    for i in range(a.warmup + a.steps):
        r = cpu_sample(e, m, a, max(4, a.cpu_chunks // 4))
        if i >= a.warmup:
            vals.append(r)
    v = sum(r["steps"] for r in vals) / sum(r["seconds"] for r in vals)
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "higher_is_better": True, "data": "synthetic", "dtype": "f64",
        "config": workload(a),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[0]["cores"], "kind": "port",
                         "sample": vals[0]["sample"] + " per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ GPU side


def main() -> None:
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import paper_2506_23364_b200 as wf
    from paper_2506_23364_b200 import _lib, shard
    from paper_2506_23364_b200.simulate import release_cells, release_mask_from_dem, run_avalanche_device
    from paper_2506_23364_b200.synth import synth_dem_device
    from paper_2506_23364_b200.terrain import compute_normals_and_slope

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # WG_BENCH_BACKEND=gloo: code-path check of the N>1 bench with every rank
    # on one GPU (NCCL refuses two ranks per device); never a measurement
    backend = os.environ.get("WG_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    _lib.build()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    elev_dev = synth_dem_device(a.size, a.seed)
    grid = wf.DemGrid.adopt(a.size, a.size, 0.0, 0.0, 10.0, -9999.0, elev_dev)
    params = wf.AvalancheParams(particles_per_release_cell=a.ppc, seed=a.seed)
    plan = shard.plan_bands(a.size, a.size, world) if world > 1 else None
    # N > 1: persistent private rasters + touched-tile map, cleared tile-
    # sparsely after each step (no full-raster memset per step)
    bufs = None
    if world > 1:
        bufs = (torch.zeros((a.size, a.size), dtype=torch.int64, device=dev),
                torch.zeros((a.size, a.size), dtype=torch.float64, device=dev),
                torch.zeros((plan.tiles_y, plan.tiles_x), dtype=torch.uint8, device=dev))

    def upstream(g):
        if world > 1:  # normals / slope / mask sharded by row band, cell lists all-gathered
            return shard.release_cells_banded(g, 30.0, 45.0, a.stride, rank, world, with_normals=not a.slope_only)
        if a.slope_only:  # C5: the slope only where the mask can be set
            mask = release_mask_from_dem(g, 30.0, 45.0, a.stride)
        else:
            _, slope = compute_normals_and_slope(g)
            mask = wf.detect_release_points(slope, 30.0, 45.0, a.stride)
            del slope
        return release_cells(mask)

    def hot_path(g):
        """One step; returns (total hits, cells, traj events, merge events, traffic)."""
        cells = upstream(g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world == 1:
            hits = torch.zeros((g.nrows, g.ncols), dtype=torch.int64, device=dev)
            zmax = torch.zeros((g.nrows, g.ncols), dtype=torch.float64, device=dev)
            e0.record(stream)
            run_avalanche_device(g, cells, params, hits=hits, zmax=zmax)
            e1.record(stream)
            run = wf.RunoutRaster(zmax, hits)  # invariants + stats pass
            return run.total_hits, cells, (e0, e1), None, None
        hits, zmax, touched = bufs
        offs = shard.band_cell_offsets(cells, plan)
        ranges = shard.particle_ranges(offs, plan, rank, a.ppc)
        e0.record(stream)
        run_avalanche_device(g, cells, params, ranges=ranges, hits=hits, zmax=zmax, touched=touched, plan=plan,
                             rank=rank)
        e1.record(stream)
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        traffic = shard.merge_tiles(hits, zmax, touched, plan)
        m1.record(stream)
        total_hits, _, _ = shard.band_stats(hits, zmax, plan)  # invariants + stats of the owned bands
        shard.clear_tiles(hits, zmax, touched, plan, rank)
        return total_hits, cells, (e0, e1), (m0, m1), dict(traffic, ranges=len(ranges),
                                                           local_particles=shard.local_particles(ranges))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        total_hits, cells, _, _, traffic = hot_path(grid)
    released = int(cells.numel()) * params.particles_per_release_cell
    total_steps = total_hits - released

    # timed: device-resident
    barrier()
    launches0 = _lib.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        t0.record(stream)
        evs, mevs = [], []
        for _ in range(a.steps):
            _, cells, ev, mev, traffic = hot_path(grid)
            evs.append(ev)
            mevs.append(mev)
        t1.record(stream)
        barrier()
    launches = _lib.launch_count() - launches0
    ms = t0.elapsed_time(t1)
    traj_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    traj_avg = sum(traj_ms) / len(traj_ms)  # average launch duration (roofline contract)
    local_steps = total_steps
    merge_avg = None
    if world > 1:
        # this rank's particle steps (its own kernel's roofline): one untimed
        # pass into fresh private rasters, summed before any merge
        h = torch.zeros((a.size, a.size), dtype=torch.int64, device=dev)
        z = torch.zeros((a.size, a.size), dtype=torch.float64, device=dev)
        ranges = shard.particle_ranges(shard.band_cell_offsets(cells, plan), plan, rank, a.ppc)
        run_avalanche_device(grid, cells, params, ranges=ranges, hits=h, zmax=z)
        local_steps = wf.RunoutRaster(z, h).total_hits - shard.local_particles(ranges)
        del h, z
        torch.cuda.empty_cache()
        merge_avg = sum(m0.elapsed_time(m1) for m0, m1 in mevs) / len(mevs)
        tt = torch.tensor([ms, traj_avg, merge_avg], dtype=torch.float64, device=dev)
        if backend != "nccl":
            tt = tt.cpu()
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)  # max over ranks
        ms, traj_max, merge_avg = tt.tolist()
    ms_per_step = ms / a.steps
    value = total_steps / (ms_per_step / 1e3)

    # e2e through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e = e2e_leg(a, wf, shard, grid, params, plan, world, rank, total_steps, released, backend)

    # latency legs (rank 0, N = 1): C4 overlay, C2 snow, C1 parabola, each with its CPU baseline
    overlay = snow = c1 = None
    if not a.no_overlay and rank == 0 and world == 1:
        overlay = overlay_latency(wf, a)
        snow = snow_latency(wf)
        c1 = c1_latency(wf, a)

    if rank == 0:
        pk = peaks()
        traj_s = traj_avg / 1e3
        achieved = BYTES_PER_STEP * local_steps / traj_s / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload(a),
            "parallelism": (f"release-row bands over {world} GPUs ({plan.nbands} bands of {plan.band_rows} rows, "
                            f"cyclic), touched-tile all-to-all merge to the band owners ({backend})"
                            if world > 1 else "1 GPU"),
            "particle_steps_per_step": total_steps,
            "released_particles": released,
            "traj_kernel_ms": traj_avg,
            "merge_ms": merge_avg,
            "merge_traffic": traffic if world > 1 else None,
            "traj_kernel_ms_per_launch": [round(t, 3) for t in traj_ms],
            "e2e": e2e,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"],
                         "traffic": TRAJ_DRAM_BYTES if a.config == "c3" and world == 1 else None,
                         "traffic_note": "DRAM bytes per launch, ncu --set full (profiles/); the gather and "
                                         "atomics are served by the 126 MB L2",
                         "peak_src": pk["src"], "kernel": "traj_kernel", "bytes_per_unit": BYTES_PER_STEP,
                         "note": "algorithmic 64 B/particle-step; the binding pipe is FP64 (roofline_fp64)"},
            "roofline_fp64": {"achieved": FP64_OPS_PER_STEP * local_steps / traj_s,
                              "peak": FP64_PEAK_OPS, "unit": "FP64 instr/s",
                              "frac": FP64_OPS_PER_STEP * local_steps / traj_s / FP64_PEAK_OPS,
                              "ops_per_unit": FP64_OPS_PER_STEP,
                              "peak_src": "measured DADD rate, tools/micro/fp64_peak.cu (profiles/fp64_peak.json)"},
            "roofline_l2": {"achieved": local_steps / traj_s, "peak": L2_STEP_PEAK, "unit": "particle-steps/s",
                            "frac": local_steps / traj_s / L2_STEP_PEAK,
                            "note": "a step's L2 operations (32-B gather + 2 atomics) vs the same operations alone "
                                    "at random L2-resident slots",
                            "peak_src": "measured, tools/micro/l2_peak.cu (profiles/l2_peak.json)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if overlay is not None:
            line["overlay_latency_ms"] = overlay
        if snow is not None:
            line["snow_latency_ms"] = snow
        if c1 is not None:
            line["c1_latency_ms"] = c1
        if not a.no_cpu:
            e, m = host_inputs(a)
            line["cpu_baseline"] = cpu_baseline(e, m, a)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def e2e_leg(a, wf, shard, grid, params, plan, world, rank, total_steps, released, backend) -> dict:
    """The same metric through the public API from pinned host memory: DEM
    upload -> DemGrid -> normals -> steepness -> release points ->
    run_avalanche -> rasters to pinned host, every step.  N = 1: two CUDA
    streams, step i+1's upload overlapping step i's download.  N > 1: the
    sharded path; each rank uploads the DEM and downloads its own bands."""
    import torch
    import torch.distributed as dist

    cell_bytes = a.size * a.size * 8
    host = torch.empty((a.size, a.size), dtype=torch.float64, pin_memory=True)
    host.copy_(grid.device_elevations().cpu())
    dev = grid.device_elevations().device
    e2e_n = max(2, a.steps)
    if world == 1:
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        outs = [(torch.empty((a.size, a.size), dtype=torch.int64, pin_memory=True),
                 torch.empty((a.size, a.size), dtype=torch.float64, pin_memory=True)) for _ in streams]
        done = [None, None]

        def step(i):
            j = i % 2
            if done[j] is not None:
                done[j].synchronize()  # this stream's result buffers are free again
            with torch.cuda.stream(streams[j]):
                g = wf.DemGrid(a.size, a.size, 0.0, 0.0, 10.0, -9999.0, host)  # pinned host tensor
                slope = wf.steepness_deg(wf.compute_normals(g))
                mask = wf.detect_release_points(slope, 30.0, 45.0, a.stride)
                r = wf.run_avalanche(g, mask, params)
                outs[j][0].copy_(r.dev("hit_count"), non_blocking=True)
                outs[j][1].copy_(r.dev("z_delta_max"), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(streams[j])
                done[j] = ev

        step(0)
        step(1)
        for ev in done:
            ev.synchronize()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for i in range(e2e_n):
            step(i)
        for ev in done:
            ev.synchronize()
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - w0) * 1e3 / e2e_n
        assert int(outs[0][0].sum()) == int(outs[1][0].sum()) == total_steps + released
        d2h = 2 * cell_bytes
        note = ("public API per step: pinned-host DEM -> DemGrid -> normals -> steepness -> release points -> "
                "run_avalanche -> both rasters to pinned host; wall clock over all steps, two CUDA streams")
    else:
        own = plan.owned_bands(rank)
        rows = sum(plan.rows(b)[1] - plan.rows(b)[0] for b in own)
        out_h = torch.empty((rows, a.size), dtype=torch.int64, pin_memory=True)
        out_z = torch.empty((rows, a.size), dtype=torch.float64, pin_memory=True)

        def step():
            g = wf.DemGrid(a.size, a.size, 0.0, 0.0, 10.0, -9999.0, host)
            cells = shard.release_cells_banded(g, 30.0, 45.0, a.stride, rank, world, with_normals=not a.slope_only)
            run = shard.run_sharded(g, cells, params, plan=plan)
            o = 0
            for b in own:
                r0, r1 = plan.rows(b)
                out_h[o:o + r1 - r0].copy_(run.hits[r0:r1], non_blocking=True)
                out_z[o:o + r1 - r0].copy_(run.zmax[r0:r1], non_blocking=True)
                o += r1 - r0
            torch.cuda.current_stream().synchronize()

        step()
        torch.cuda.synchronize()
        dist.barrier()
        w0 = time.perf_counter()
        for _ in range(e2e_n):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        e2e_ms = (time.perf_counter() - w0) * 1e3 / e2e_n
        tt = torch.tensor([e2e_ms], dtype=torch.float64)
        if backend == "nccl":
            tt = tt.to(dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
        d2h = rows * a.size * 16
        note = ("sharded public path per step: pinned-host DEM -> DemGrid on every rank -> banded normals / "
                "steepness / release points -> run_sharded (tile-sparse merge) -> each rank's own bands to pinned "
                "host; wall clock, max over ranks; bytes per rank")
    return {"value": total_steps / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
            "h2d_bytes_per_step": cell_bytes, "d2h_bytes_per_step": d2h, "note": note}


# ------------------------------------------------------------------ CPU baselines


def lscpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


def cpu_baseline(e: np.ndarray, m: np.ndarray, a) -> dict:
    """The C port of the reference engine on the box's host cores: all
    threads over a.cpu_chunks evenly spaced chunks, and one thread over an
    eighth of them; both rates are sampled (the full run is ~10^10 steps)."""
    nthreads = os.cpu_count() or 1
    many = cpu_sample(e, m, a, a.cpu_chunks, nthreads)
    one = cpu_sample(e, m, a, max(8, a.cpu_chunks // 64), 1)
    return {"value": many["value"], "unit": UNIT, "cores": nthreads, "kind": "port",
            "sample": many["sample"], "cpu_model": lscpu_model(),
            "threads_1": {"value": one["value"], "sample": one["sample"]}}


def cpu_overlay_latency(e: np.ndarray, stride: int, ppc: int, seed: int, threads: int,
                        runout: np.ndarray | None = None) -> tuple[dict, np.ndarray]:
    """The stock avalanche graph's compute on the host -- the reference's
    node functions restated (oracle/npref.py: normals, steepness, mask,
    colorize, mipmap; the C oracle: trajectories), timed per node; returns
    the timings and the runout drop raster.  threads = 1: the trajectories
    are timed over 64 evenly spaced chunks and extrapolated (labelled), and
    colorize / mipmap run on the given full-run raster."""
    from oracle import npref, traj

    from paper_2506_23364_b200.overlay import DEFAULT_RUNOUT_COLORMAP

    t = {}
    t0 = time.perf_counter()
    n = npref.normals(e, 10.0)
    t["surface_normals"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    s = npref.steepness(n)
    t["steepness"] = time.perf_counter() - t0
    del n
    t0 = time.perf_counter()
    mask = npref.release_mask(s, 30.0, 45.0, stride)
    t["release_points"] = time.perf_counter() - t0
    del s
    cells = np.ascontiguousarray(np.flatnonzero(mask.ravel()), dtype=np.int64)
    total = cells.size * ppc
    hits = np.zeros(e.shape, dtype=np.int64)
    zmax = np.zeros(e.shape, dtype=np.float64)
    extrapolated = None
    t0 = time.perf_counter()
    if runout is None:
        traj.run_range(e, 0.0, 0.0, 10.0, cells, 0, total, hits, zmax, particles_per_release_cell=ppc, seed=seed,
                       threads=threads)
        t["trajectories"] = time.perf_counter() - t0
    else:
        nch = -(-total // 2048)
        pick = np.unique(np.linspace(0, nch - 1, min(64, nch)).astype(np.int64))
        for c in pick:
            traj.run_range(e, 0.0, 0.0, 10.0, cells, int(c) * 2048, min(int(c) * 2048 + 2048, total), hits, zmax,
                           particles_per_release_cell=ppc, seed=seed, threads=threads)
        t["trajectories"] = (time.perf_counter() - t0) * nch / len(pick)
        extrapolated = f"trajectories extrapolated from {len(pick)} of {nch} 2048-particle chunks"
        zmax = runout
    t0 = time.perf_counter()
    px = npref.colorize(zmax, DEFAULT_RUNOUT_COLORMAP.stops)
    t["colorize"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    npref.mipmap(px)
    t["mipmap"] = time.perf_counter() - t0
    out = {"ms": sum(t.values()) * 1e3, "node_ms": {k: round(v * 1e3, 1) for k, v in t.items()}, "threads": threads}
    if extrapolated:
        out["extrapolated"] = extrapolated
    return out, zmax


def cpu_leg(fn, *args) -> dict:
    """A CPU baseline at all host threads, then at one thread (reusing the
    all-thread run's raster where the one-thread run samples)."""
    nthreads = os.cpu_count() or 1
    many, runout = fn(*args, nthreads)
    one, _ = fn(*args, 1, runout)
    return {"kind": "port", "cores": nthreads, "cpu_model": lscpu_model(), "threads_n": many, "threads_1": one}


def overlay_latency(wf, a) -> dict:
    """Cold and warm-steering latency of the stock avalanche graph (7 nodes)
    on a stitched 8192^2 world (BASELINE configs[3]: zoom 2 = 16 tiles, band
    30-45 stride 16, 256 particles per cell), colorize + 14-level mip; and
    the same graph's compute on the host cores (cpu_baseline)."""
    import torch

    from paper_2506_23364_b200.synth import synth_dem_device, synth_dem_host

    n = a.overlay_size
    world = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, synth_dem_device(n, 1))
    rel = wf.SteepnessRelease(30.0, 45.0, stride=16)

    def graph(seed):
        g = wf.build_avalanche_graph(world.extent, wf.AvalancheParams(particles_per_release_cell=256, seed=seed),
                                     rel, zoom=2)
        g.bind("world", world)
        return g

    wf.Executor().execute(graph(0))  # warm the CUDA context / allocator
    torch.cuda.synchronize()
    cold = []
    for s in range(2):
        ex = wf.Executor()
        t0 = time.perf_counter()
        res = ex.execute(graph(s))
        cold.append((time.perf_counter() - t0) * 1e3)
    warm = []
    for s in range(3):
        t0 = time.perf_counter()
        rep = ex.execute(graph(100 + s)).report
        warm.append((time.perf_counter() - t0) * 1e3)
    nodes = {r.node_id: round(r.elapsed_ms, 3) for r in res.report.records}
    out = {"config": f"stock avalanche graph, synth_dem({n}, 1) world, zoom 2 (16 tiles), band 30-45 stride 16, "
                     "256 particles/cell, colorize + full mip (BASELINE configs[3])",
           "cold": min(cold), "warm_steering": min(warm), "warm_cache_hits": rep.cache_hits,
           "stats": res.value("avalanche_overlay", "stats"), "node_ms_cold": nodes}
    if not a.no_cpu:
        e = synth_dem_host(n, 1)
        out["cpu_baseline"] = cpu_leg(cpu_overlay_latency, e, 16, 256, 1)
        out["cpu_baseline"]["note"] = ("same graph on the host: npref normals / steepness / mask / colorize / "
                                       "mipmap (numpy, one thread) + C-oracle trajectories; no digests, no tiling "
                                       "copies")
    return out


def cpu_snow_latency(z: np.ndarray, line: float, threads: int, _unused=None) -> tuple[dict, None]:
    from oracle import npref

    t = {}
    t0 = time.perf_counter()
    n = npref.normals(z, 10.0)
    t["surface_normals"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    s = npref.steepness(n)
    t["steepness"] = time.perf_counter() - t0
    del n
    t0 = time.perf_counter()
    px = npref.snow_texture(z, s, -9999.0, False, line, 200.0, 50.0, 10.0)
    t["snow"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    npref.mipmap(px)
    t["mipmap"] = time.perf_counter() - t0
    return {"ms": sum(t.values()) * 1e3, "node_ms": {k: round(v * 1e3, 1) for k, v in t.items()},
            "threads": 1}, None


def snow_latency(wf) -> dict:
    """Cold latency of the stock snow graph at SURVEY §8d C2: synth_dem(4096, 0),
    snow line at the median height, zoom 1 (4 tiles), full 13-level mip; and
    the numpy restatement of the same nodes on the host."""
    import torch

    from paper_2506_23364_b200.synth import synth_dem_device

    n = 4096
    z = synth_dem_device(n, 0)
    world = wf.DemGrid.adopt(n, n, 0.0, 0.0, 10.0, -9999.0, z)
    line = float(torch.median(z.view(-1)).item())
    params = wf.SnowParams(snow_line_m=line, altitude_blend_m=200.0, max_steepness_deg=50.0, steepness_blend_deg=10.0)

    def graph():
        g = wf.build_snow_graph(world.extent, params, zoom=1)
        g.bind("world", world)
        return g

    wf.Executor().execute(graph())  # warm
    torch.cuda.synchronize()
    cold = []
    for _ in range(3):
        ex = wf.Executor()
        t0 = time.perf_counter()
        res = ex.execute(graph())
        cold.append((time.perf_counter() - t0) * 1e3)
    nodes = {r.node_id: round(r.elapsed_ms, 3) for r in res.report.records}
    cpu, _ = cpu_snow_latency(world.elevations, line, 1)
    cpu.update(kind="port", cores=1, cpu_model=lscpu_model(),
               note="npref normals / steepness / snow / mipmap (numpy is single-threaded on these ufuncs)")
    return {"config": "stock snow graph (6 nodes), synth_dem(4096, 0), snow line = median height, zoom 1, "
                      "13-level mip (BASELINE configs[1])",
            "cold": min(cold), "node_ms_cold": nodes, "cpu_baseline": cpu}


def c1_latency(wf, a) -> dict:
    """BASELINE configs[0], the reference's own benchmark (cli.py:229-264,
    the paper's 13.5 ms case): the stock avalanche graph over the bundled
    parabola slope (501 x 151, 3 release cells x 2048 particles) for the
    defaults and the shipped golden run (alpha 12, seed 7).  GPU cold graph,
    warm steering (only the params change: 5 cache hits + 1 executed), and
    the C-oracle trajectories on the host at 1 and all threads."""
    import torch

    from oracle import traj

    grid, mask = wf.gen_parabola()
    out = {"config": "stock avalanche graph, bundled parabola (pkg/data/parabola), MaskRelease(3 cells), zoom 1",
           "reference_recorded_s": {"alpha12_seed7": 0.86, "source": "pkg/test_output.txt:13 (1 thread)"}}
    for name, kw in (("defaults", {}), ("alpha12_seed7", {"runout_angle_deg": 12.0, "seed": 7})):
        params = wf.AvalancheParams(**kw)

        def graph(p):
            g = wf.build_avalanche_graph(grid.extent, p, wf.MaskRelease(wf.ReleaseMask(mask)), zoom=1)
            g.bind("world", grid)
            return g

        wf.Executor().execute(graph(params))
        torch.cuda.synchronize()
        cold = []
        for _ in range(3):
            t0 = time.perf_counter()
            res = wf.Executor().execute(graph(params))
            cold.append((time.perf_counter() - t0) * 1e3)
        ex = wf.Executor()
        ex.execute(graph(params))
        warm = []
        for s in range(3):
            t0 = time.perf_counter()
            ex.execute(graph(wf.AvalancheParams(**dict(kw, seed=1000 + s))))
            warm.append((time.perf_counter() - t0) * 1e3)
        stats = res.value("avalanche_overlay", "stats")
        cpu = {}
        for th in (1, os.cpu_count() or 1):
            t0 = time.perf_counter()
            traj.run_avalanche(grid.elevations, grid.origin_x, grid.origin_y, grid.cellsize, mask,
                               particles_per_release_cell=2048, threads=th, **kw)
            cpu[f"threads_{th}"] = (time.perf_counter() - t0) * 1e3
        out[name] = {"cold": min(cold), "warm_steering": min(warm), "particle_steps": stats["particle_steps"],
                     "node_ms_cold": {r.node_id: round(r.elapsed_ms, 3) for r in res.report.records},
                     "cpu_trajectories_ms": cpu}
    return out


if __name__ == "__main__":
    main()

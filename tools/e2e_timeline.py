"""Timeline of the bench's end-to-end loop (C3): CUDA events after each stage
on each stream plus host timestamps, to see what the e2e step waits on.
Usage: python tools/e2e_timeline.py [--steps 4]."""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200 import _lib  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--stride", type=int, default=32)
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    _lib.build()
    host = torch.empty((a.size, a.size), dtype=torch.float64, pin_memory=True)
    host.copy_(synth_dem_device(a.size, 0).cpu())
    params = wf.AvalancheParams(seed=0)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [(torch.empty((a.size, a.size), dtype=torch.int64, pin_memory=True),
             torch.empty((a.size, a.size), dtype=torch.float64, pin_memory=True)) for _ in streams]
    done = [None, None]
    t_origin = torch.cuda.Event(enable_timing=True)
    t_origin.record()
    host0 = time.perf_counter()
    log = []

    def mark(i, name, s):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        log.append((i, name, e, (time.perf_counter() - host0) * 1e3))

    from paper_2506_23364_b200 import simulate as sim

    cur = {}

    def wrap(fn, name):
        def inner(*args, **kw):
            r = fn(*args, **kw)
            mark(cur["i"], name, cur["s"])
            return r
        return inner

    sim.release_cells = wrap(sim.release_cells, "  release_cells")
    sim.build_quad = wrap(sim.build_quad, "  build_quad")
    sim.run_avalanche_device = wrap(sim.run_avalanche_device, "  traj launched")

    def step(i):
        j = i % 2
        s = streams[j]
        cur["i"], cur["s"] = i, s
        if done[j] is not None:
            done[j].synchronize()
        with torch.cuda.stream(s):
            mark(i, "begin", s)
            g = wf.DemGrid(a.size, a.size, 0.0, 0.0, 10.0, -9999.0, host)
            mark(i, "grid(h2d+scan)", s)
            n = wf.compute_normals(g)
            mark(i, "normals", s)
            slope = wf.steepness_deg(n)
            mark(i, "steepness", s)
            mask = wf.detect_release_points(slope, 30.0, 45.0, a.stride)
            mark(i, "release", s)
            r = wf.run_avalanche(g, mask, params)
            mark(i, "avalanche", s)
            outs[j][0].copy_(r.dev("hit_count"), non_blocking=True)
            outs[j][1].copy_(r.dev("z_delta_max"), non_blocking=True)
            mark(i, "d2h", s)
            ev = torch.cuda.Event()
            ev.record(s)
            done[j] = ev

    for i in range(a.steps):
        step(i)
    torch.cuda.synchronize()
    total = (time.perf_counter() - host0) * 1e3
    for i, name, e, h in log:
        print(f"step {i} {name:16s} gpu {t_origin.elapsed_time(e):9.1f} ms   host-issued {h:9.1f} ms")
    print(f"total wall {total:.1f} ms for {a.steps} steps")


if __name__ == "__main__":
    main()

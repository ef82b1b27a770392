"""Per-launch timing distribution of the trajectory kernel on the bench
workload (C3), in one process: separates kernel variance from process /
allocation effects.  Usage: python tools/traj_probe.py [--reps 10]."""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2506_23364_b200 as wf  # noqa: E402
from paper_2506_23364_b200 import _lib  # noqa: E402
from paper_2506_23364_b200 import simulate  # noqa: E402
from paper_2506_23364_b200.simulate import build_quad, release_cells, run_avalanche_device  # noqa: E402
from paper_2506_23364_b200.synth import synth_dem_device  # noqa: E402
from paper_2506_23364_b200.terrain import compute_normals_and_slope  # noqa: E402


class Nvml:
    """Fast NVML clock / event-reason polling (5 ms) around one launch."""

    def __init__(self):
        import threading

        import pynvml

        self.n = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.threading = threading

    def __enter__(self):
        self.stop = False
        self.samples = []

        def run():
            import time

            while not self.stop:
                c = self.n.nvmlDeviceGetClockInfo(self.h, self.n.NVML_CLOCK_SM)
                r = self.n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                p = self.n.nvmlDeviceGetPowerUsage(self.h)
                t = self.n.nvmlDeviceGetTemperature(self.h, self.n.NVML_TEMPERATURE_GPU)
                self.samples.append((c, r, p, t))
                time.sleep(0.005)

        self.t = self.threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop = True
        self.t.join()

    def summary(self):
        if not self.samples:
            return {}
        cl = sorted(c for c, _, _, _ in self.samples)
        reasons = 0
        for _, r, _, _ in self.samples:
            reasons |= r
        pw = [p for _, _, p, _ in self.samples]
        return {"mhz_min": cl[0], "mhz_med": cl[len(cl) // 2], "reasons": hex(reasons),
                "w_max": max(pw) // 1000, "w_mean": sum(pw) // len(pw) // 1000,
                "temp_max": max(t for _, _, _, t in self.samples)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--stride", type=int, default=32)
    ap.add_argument("--ppc", type=int, default=2048)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--records", action="store_true", help="also report particle lifetime stats")
    ap.add_argument("--layout", choices=["auto", "pair", "dem"], default="auto", help="force the gather layout")
    ap.add_argument("--lattice", action="store_true", help="release mask from the DEM at lattice cells (C5: no slope field)")
    a = ap.parse_args()
    _lib.build()
    elev = synth_dem_device(a.size, a.seed)
    grid = wf.DemGrid.adopt(a.size, a.size, 0.0, 0.0, 10.0, -9999.0, elev)
    params = wf.AvalancheParams(particles_per_release_cell=a.ppc, seed=a.seed)
    if a.lattice:
        from paper_2506_23364_b200.simulate import release_mask_from_dem

        mask = release_mask_from_dem(grid, 30.0, 45.0, a.stride)
    else:
        _, slope = compute_normals_and_slope(grid)
        mask = wf.detect_release_points(slope, 30.0, 45.0, a.stride)
    cells = release_cells(mask)
    hits = torch.zeros((a.size, a.size), dtype=torch.int64, device="cuda")
    zmax = torch.zeros((a.size, a.size), dtype=torch.float64, device="cuda")
    quad_ok = build_quad(grid) is not None and a.layout == "auto"
    if a.layout != "auto":
        simulate.build_gather_layout = (lambda g: (None, simulate.build_pair(g))) if a.layout == "pair" \
            else (lambda g: (None, None))
    times = []
    clocks = []
    try:
        nv = Nvml()
    except Exception:  # noqa: BLE001
        nv = None
    for _ in range(a.reps):
        hits.zero_()
        zmax.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if nv is not None:
            nv.__enter__()
        e0.record()
        run_avalanche_device(grid, cells, params, hits=hits, zmax=zmax)
        e1.record()
        torch.cuda.synchronize()
        if nv is not None:
            nv.__exit__()
            clocks.append(nv.summary())
        times.append(round(e0.elapsed_time(e1), 2))
    steps = int(hits.sum().item()) - int(cells.numel()) * a.ppc
    out = {"cells": int(cells.numel()), "particles": int(cells.numel()) * a.ppc, "steps": steps,
           "quad": quad_ok, "layout": a.layout, "ms": times,
           # raster checksums: variants of the kernel must agree bit for bit
           "hits_wsum": int((hits.view(-1)[::7]).sum().item()), "zbits_xor": int(
               zmax.view(torch.int64).view(-1)[::3].sum().item()), "clocks": clocks, "gsteps_s_best": round(steps / min(times) / 1e6, 2)}
    if a.records:
        from paper_2506_23364_b200.simulate import particle_records

        n = int(cells.numel()) * a.ppc
        reason, st, _ = particle_records(grid, mask, params, 0, n)
        import numpy as np

        out["lifetime"] = {"mean": round(float(st.mean()), 1), "max": int(st.max()),
                           "p50_p90_p99_p999": np.percentile(st, [50, 90, 99, 99.9]).round(1).tolist()}
        out["reasons"] = np.bincount(reason.astype(np.int64), minlength=4).tolist()
        # per release cell: how well does one particle predict its cell's
        # longest particle (a longest-first claim order would need that)
        per = st.reshape(-1, a.ppc).astype(np.float64)
        cmax, cmean, p0 = per.max(1), per.mean(1), per[:, 0]
        out["cells"] = {"max_of_max": int(cmax.max()), "cells_max_over_1000": int((cmax > 1000).sum()),
                        "cells_max_over_500": int((cmax > 500).sum()),
                        "corr_p0_cellmax": round(float(np.corrcoef(p0, cmax)[0, 1]), 3),
                        "corr_p0_cellmean": round(float(np.corrcoef(p0, cmean)[0, 1]), 3),
                        "corr_mean_max": round(float(np.corrcoef(cmean, cmax)[0, 1]), 3),
                        "cellmax_p50_p90_p99_p999": np.percentile(cmax, [50, 90, 99, 99.9]).round(1).tolist()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

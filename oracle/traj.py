"""TEST INFRASTRUCTURE: ctypes wrapper of the C particle-engine oracle
(oracle/traj_oracle.c).  Host scalars are derived exactly as the reference
does (simulate.py:286-298), then the C restatement runs one particle at a
time calling the host glibc sin/cos (simulate.py:359-360)."""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"
_lib = None

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def build() -> Path:
    if not LIB.exists():
        subprocess.run(["make", "-C", str(HERE)], check=True, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        h = ctypes.CDLL(str(LIB))
        d, i64, u64, p = ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        world = [p, i64, i64, d, d, d, d, d, d, d, d, d, d, i64]
        h.orc_run_particles.argtypes = world + [p, i64, u64, i64, i64, p, p, p, p, p, ctypes.c_int]
        h.orc_run_particles.restype = ctypes.c_int
        h.orc_simulate_particle.argtypes = world + [d, d, u64, p, i64, p]
        h.orc_simulate_particle.restype = ctypes.c_int
        h.orc_derive_key.argtypes = [u64, u64, u64]
        h.orc_derive_key.restype = u64
        h.orc_draw_unit.argtypes = [u64, u64]
        h.orc_draw_unit.restype = d
        _lib = h
    return _lib


def world_args(elev: np.ndarray, ox: float, oy: float, cs: float, persistence: float, randomness: float,
               runout_angle_deg: float, max_steps: int | None):
    """simulate.py:286-298 with Python floats."""
    nrows, ncols = elev.shape
    tana = math.tan(math.radians(runout_angle_deg))
    ms = max_steps if max_steps is not None else 10 * max(ncols, nrows)
    return [elev.ctypes.data, nrows, ncols, ox, oy, cs, ox + ncols * cs, oy + nrows * cs, tana, persistence,
            1.0 - persistence, randomness, randomness * (math.pi / 2.0), ms]


def run_avalanche(elev, ox, oy, cs, mask, *, persistence=0.9, randomness=0.16, runout_angle_deg=25.0,
                  particles_per_release_cell=2048, seed=0, max_steps=None, threads=None, lo=0, hi=None,
                  records=False):
    """Oracle run_avalanche (simulate.py:441-504) over particles [lo, hi).

    Returns (z_delta_max, hit_count) and, with records=True, the per-particle
    (reason, steps, end) arrays for [lo, hi)."""
    elev = np.ascontiguousarray(elev, dtype=np.float64)
    cells = np.ascontiguousarray(np.flatnonzero(np.asarray(mask, dtype=bool).ravel()), dtype=np.int64)
    total = cells.size * particles_per_release_cell
    hi = total if hi is None else hi
    hits = np.zeros(elev.shape, dtype=np.int64)
    zmax = np.zeros(elev.shape, dtype=np.float64)
    n = max(hi - lo, 0)
    reasons = np.zeros(n, dtype=np.int8) if records else None
    steps = np.zeros(n, dtype=np.int64) if records else None
    ends = np.zeros((n, 2), dtype=np.float64) if records else None
    threads = threads or os.cpu_count() or 1
    if n > 0:
        lib().orc_run_particles(
            *world_args(elev, ox, oy, cs, persistence, randomness, runout_angle_deg, max_steps),
            cells.ctypes.data, particles_per_release_cell, seed & MASK64, lo, hi, hits.ctypes.data,
            zmax.ctypes.data,
            reasons.ctypes.data if records else None, steps.ctypes.data if records else None,
            ends.ctypes.data if records else None, int(threads),
        )
    if records:
        return zmax, hits, (reasons, steps, ends)
    return zmax, hits


def run_range(elev, ox, oy, cs, cells, lo, hi, hits, zmax, *, persistence=0.9, randomness=0.16,
              runout_angle_deg=25.0, particles_per_release_cell=2048, seed=0, max_steps=None, threads=None,
              records=False):
    """Particles [lo, hi) accumulated into caller-owned rasters (one shared
    pair across calls, unlike the reference's per-chunk partials; None for
    records-only runs); returns
    the particle steps taken, and with records=True also the per-particle
    (reason, steps, end) arrays."""
    n = hi - lo
    if n <= 0:
        return (0, None) if records else 0
    steps = np.zeros(n, dtype=np.int64)
    reasons = np.zeros(n, dtype=np.int8) if records else None
    ends = np.zeros((n, 2), dtype=np.float64) if records else None
    lib().orc_run_particles(
        *world_args(elev, ox, oy, cs, persistence, randomness, runout_angle_deg, max_steps),
        cells.ctypes.data, particles_per_release_cell, seed & MASK64, lo, hi,
        hits.ctypes.data if hits is not None else None, zmax.ctypes.data if zmax is not None else None,
        reasons.ctypes.data if records else None, steps.ctypes.data, ends.ctypes.data if records else None,
        int(threads or os.cpu_count() or 1),
    )
    if records:
        return int(steps.sum()), (reasons, steps, ends)
    return int(steps.sum())


def simulate_particle(elev, ox, oy, cs, start, key, *, persistence=0.9, randomness=0.16, runout_angle_deg=25.0,
                      max_steps=None):
    """Oracle simulate_particle (simulate.py:415-438): (positions, reason code)."""
    elev = np.ascontiguousarray(elev, dtype=np.float64)
    wa = world_args(elev, ox, oy, cs, persistence, randomness, runout_angle_deg, max_steps)
    cap = int(wa[-1]) + 2
    path = np.zeros((cap, 2), dtype=np.float64)
    n = ctypes.c_int64(0)
    r = lib().orc_simulate_particle(*wa, float(start[0]), float(start[1]), key & MASK64, path.ctypes.data, cap,
                                    ctypes.byref(n))
    return path[: n.value].copy(), r


def derive_key(seed: int, k: int, p: int) -> int:
    return int(lib().orc_derive_key(seed & MASK64, k & MASK64, p & MASK64))

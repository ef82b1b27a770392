"""Synthetic DEMs of the measurement plan.

synth_dem(n, seed, cs=10, H=300, lambda0=4000, 4 octaves):
    z = sum_o (H/2^o) sin(2 pi y / (lambda0/2^o) + psi_o) sin(2 pi x / (lambda0/2^o) + phi_o) + 0.05 x,
then shifted so the minimum is 0; phases from np.random.default_rng(seed);
cell centres per grid.py:11-12 with origin (0, 0).

The recipe is separable: the host evaluates the 1-D row and column factors
(n x 4 sines each, numpy), and the 2-D combination
``lin[c] + sum_o rowf[o][r] * colf[o][c]`` is an IEEE add/multiply chain with
a fixed order, evaluated identically by the device kernel (wg_synth_combine)
and by :func:`synth_dem_host` -- so CPU baselines and GPU runs see the
bitwise-same DEM.
"""

from __future__ import annotations

import math

import numpy as np
import torch

OCTAVES = 4


def _factors(n: int, seed: int, cs: float, H: float, lam0: float):
    rng = np.random.default_rng(seed)
    psi = rng.uniform(0.0, 2.0 * math.pi, OCTAVES)
    phi = rng.uniform(0.0, 2.0 * math.pi, OCTAVES)
    centres_x = (np.arange(n, dtype=np.float64) + 0.5) * cs
    # row r (north-first) has y = (n - 1 - r + 0.5) * cs
    centres_y = (np.arange(n - 1, -1, -1, dtype=np.float64) + 0.5) * cs
    rowf = np.empty((OCTAVES, n), dtype=np.float64)
    colf = np.empty((OCTAVES, n), dtype=np.float64)
    for o in range(OCTAVES):
        lam = lam0 / (2.0**o)
        amp = H / (2.0**o)
        rowf[o] = amp * np.sin(2.0 * math.pi * centres_y / lam + psi[o])
        colf[o] = np.sin(2.0 * math.pi * centres_x / lam + phi[o])
    lin = 0.05 * centres_x
    return rowf, colf, lin


def synth_dem_host(n: int, seed: int, cs: float = 10.0, H: float = 300.0, lam0: float = 4000.0) -> np.ndarray:
    """Host evaluation (numpy), bit-identical to :func:`synth_dem_device`."""
    rowf, colf, lin = _factors(n, seed, cs, H, lam0)
    z = np.broadcast_to(lin, (n, n)).copy()
    for o in range(OCTAVES):
        z += rowf[o][:, None] * colf[o][None, :]
    z -= z.min()
    return z


def synth_dem_device(n: int, seed: int, cs: float = 10.0, H: float = 300.0, lam0: float = 4000.0) -> torch.Tensor:
    """Device evaluation into a fresh (n, n) float64 CUDA tensor."""
    from . import _device, _lib

    rowf, colf, lin = _factors(n, seed, cs, H, lam0)
    L = _lib.lib()
    r = _device.upload(rowf)
    c = _device.upload(colf)
    li = _device.upload(lin)
    out = _device.empty((n, n), torch.float64)
    _lib.check(L.wg_synth_combine(_lib.ptr(r), _lib.ptr(c), _lib.ptr(li), OCTAVES, n, n, _lib.ptr(out),
                                  _lib.stream_ptr()))
    zmin = float(out.min().item())
    _lib.check(L.wg_sub_scalar(_lib.ptr(out), out.numel(), zmin, _lib.stream_ptr()))
    return out


def synth_grid(n: int, seed: int, cs: float = 10.0, device: bool = True):
    """DemGrid over synth_dem (origin (0, 0), nodata -9999)."""
    from .grid import DemGrid

    if device:
        return DemGrid.adopt(n, n, 0.0, 0.0, cs, -9999.0, synth_dem_device(n, seed, cs))
    return DemGrid(ncols=n, nrows=n, origin_x=0.0, origin_y=0.0, cellsize=cs, nodata=-9999.0,
                   elevations=synth_dem_host(n, seed, cs))

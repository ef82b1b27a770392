"""Surface derivatives of elevation grids (mirrors demflow/terrain.py).

compute_normals / steepness_deg / hillshade run as sm_100a kernels
(csrc/stencil.cu); oracle_descent_path runs the trajectory kernel's step
function (csrc/traj.cu) on one lane; downslope_dir is a scalar query helper
evaluated on the host with the reference's arithmetic (terrain.py:105-148).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _device, _lib
from ._resident import Resident
from .grid import DemGrid, SampleError, _patch

FLAT_GRADIENT_THRESHOLD = 1e-6  # m/m (terrain.py:19)


class TerrainError(ValueError):
    pass


class NormalField(Resident):
    """Per-cell unit surface normals, shape (nrows, ncols, 3) (terrain.py:26-46)."""

    _payload = ("normals",)
    _dtypes = {"normals": (np.dtype(np.float64), torch.float64)}

    def __init__(self, normals):
        shape = tuple(normals.shape) if isinstance(normals, torch.Tensor) else np.shape(normals)
        if len(shape) != 3 or shape[2] != 3:
            raise TerrainError(f"normals must be (nrows, ncols, 3), got {tuple(shape)}")
        super().__init__(normals=normals)

    @property
    def nrows(self) -> int:
        return self.shape_of("normals")[0]

    @property
    def ncols(self) -> int:
        return self.shape_of("normals")[1]

    def __repr__(self) -> str:
        return f"NormalField({self.nrows}x{self.ncols})"


class SlopeField(Resident):
    """Per-cell steepness in degrees, 0 = horizontal (terrain.py:49-66)."""

    _payload = ("slope_deg",)
    _dtypes = {"slope_deg": (np.dtype(np.float64), torch.float64)}

    def __init__(self, slope_deg):
        super().__init__(slope_deg=slope_deg)

    @property
    def nrows(self) -> int:
        return self.shape_of("slope_deg")[0]

    @property
    def ncols(self) -> int:
        return self.shape_of("slope_deg")[1]

    def __repr__(self) -> str:
        return f"SlopeField({self.nrows}x{self.ncols})"


def compute_normals(grid: DemGrid) -> NormalField:
    """Unit normals normalize(-dz/dx, -dz/dy, 1) (terrain.py:69-96), bit-exact.

    One HBM pass (wg_normals): 8 B/cell in, 24 B/cell out.
    """
    if grid.has_nodata():
        raise TerrainError("normals require a gap-free grid (nodata present)")
    L = _lib.lib()
    e = grid.device_elevations()
    out = _device.empty((grid.nrows, grid.ncols, 3), torch.float64)
    cs = grid.cellsize
    _lib.check(
        L.wg_normals(_lib.ptr(e), grid.nrows, grid.ncols, cs, 2.0 * cs, _lib.ptr(out), None, _lib.stream_ptr()),
        TerrainError,
    )
    return NormalField(out)


def compute_normals_and_slope(grid: DemGrid) -> tuple[NormalField, SlopeField]:
    """Fused surface_normals + steepness pass (same bits as the two nodes)."""
    if grid.has_nodata():
        raise TerrainError("normals require a gap-free grid (nodata present)")
    L = _lib.lib()
    e = grid.device_elevations()
    out = _device.empty((grid.nrows, grid.ncols, 3), torch.float64)
    slope = _device.empty((grid.nrows, grid.ncols), torch.float64)
    cs = grid.cellsize
    _lib.check(
        L.wg_normals(_lib.ptr(e), grid.nrows, grid.ncols, cs, 2.0 * cs, _lib.ptr(out), _lib.ptr(slope),
                     _lib.stream_ptr()),
        TerrainError,
    )
    return NormalField(out), SlopeField(slope)


def compute_slope(grid: DemGrid) -> SlopeField:
    """steepness_deg(compute_normals(grid)) in one pass without storing the
    (nrows, ncols, 3) normal field (same per-cell arithmetic, same bits);
    for grids whose normal field does not fit next to the rest (65536^2)."""
    if grid.has_nodata():
        raise TerrainError("normals require a gap-free grid (nodata present)")
    L = _lib.lib()
    e = grid.device_elevations()
    slope = _device.empty((grid.nrows, grid.ncols), torch.float64)
    cs = grid.cellsize
    _lib.check(
        L.wg_normals(_lib.ptr(e), grid.nrows, grid.ncols, cs, 2.0 * cs, None, _lib.ptr(slope), _lib.stream_ptr()),
        TerrainError,
    )
    return SlopeField(slope)


def steepness_deg(normals: NormalField) -> SlopeField:
    """Slope angle per cell: degrees(arccos(clip(nz))) (terrain.py:99-102)."""
    L = _lib.lib()
    n = normals.dev("normals")
    out = _device.empty((normals.nrows, normals.ncols), torch.float64)
    _lib.check(L.wg_steepness(_lib.ptr(n), out.numel(), _lib.ptr(out), _lib.stream_ptr()), TerrainError)
    return SlopeField(out)


def downslope_dir(grid: DemGrid, x: float, y: float) -> tuple[float, float] | None:
    """Unit steepest-descent direction of the bilinear surface at (x, y), or
    None on flat ground (terrain.py:105-148).  Scalar query helper."""
    if not grid.contains(x, y):
        raise SampleError(f"position ({x}, {y}) outside grid extent")
    cs = grid.cellsize
    u = (x - grid.origin_x) / cs - 0.5
    v = (y - grid.origin_y) / cs - 0.5
    u = min(max(u, 0.0), grid.ncols - 1.0)
    v = min(max(v, 0.0), grid.nrows - 1.0)
    j0 = min(int(math.floor(u)), grid.ncols - 2)
    s0 = min(int(math.floor(v)), grid.nrows - 2)
    wu = u - j0
    wv = v - s0
    i1 = grid.nrows - 1 - s0
    z00, z10, z01, z11 = _patch(grid, i1 - 1, i1, j0)
    nd = grid.nodata
    if z00 == nd or z10 == nd or z01 == nd or z11 == nd:
        raise SampleError(f"nodata in bilinear neighborhood of ({x}, {y})")
    gx_s = z10 - z00
    gx_n = z11 - z01
    gy_w = z01 - z00
    gy_e = z11 - z10
    gx = -((gx_s + (gx_n - gx_s) * wv) / cs)
    gy = -((gy_w + (gy_e - gy_w) * wu) / cs)
    mag = math.sqrt(gx * gx + gy * gy)
    if mag < FLAT_GRADIENT_THRESHOLD:
        return None
    return (gx / mag, gy / mag)


def oracle_descent_path(
    grid: DemGrid,
    start: tuple[float, float],
    step: float,
    runout_angle_deg: float = 25.0,
    max_steps: int | None = None,
) -> tuple[np.ndarray, str]:
    """Steepest-descent walk from `start` in `step`-metre steps (terrain.py:151-284):
    stops on flat ground, on leaving the grid (exit point clipped to the
    border and kept), when the angle back up to the start drops below
    `runout_angle_deg`, or after the step cap (10 * max(ncols, nrows) by
    default).  Returns (positions (n, 2), reason).

    The reference keeps this walk free of the particle engine's code while
    matching its float sequence for a memoryless, jitter-free particle; here
    it is exactly that particle -- persistence 0 (the blend reduces to the
    renormalised descent direction bit for bit), randomness 0 -- traced by
    the device step function with the step length set to `step`."""
    from .simulate import AvalancheParams, trace

    if grid.has_nodata():
        raise SampleError("descent path on a grid with nodata")
    x, y = float(start[0]), float(start[1])
    if not grid.contains(x, y):
        raise SampleError(f"start ({x}, {y}) outside grid extent")
    params = AvalancheParams(persistence=0.0, randomness=0.0, runout_angle_deg=runout_angle_deg,
                             max_steps=max_steps)
    positions, code = trace(grid, (x, y), params, 0, float(step))
    return positions, ("RUNOUT_ANGLE", "DOMAIN_EXIT", "FLAT", "MAX_STEPS")[code]


def _light(azimuth_deg: float, altitude_deg: float) -> tuple[float, float, float]:
    # terrain.py:292-297, host Python floats (glibc sin/cos), passed verbatim
    az = math.radians(azimuth_deg)
    alt = math.radians(altitude_deg)
    return math.sin(az) * math.cos(alt), math.cos(az) * math.cos(alt), math.sin(alt)


def hillshade(grid: DemGrid, azimuth_deg: float = 315.0, altitude_deg: float = 45.0) -> np.ndarray:
    """Lambertian hillshade as (nrows, ncols) uint8 (terrain.py:287-299):
    the normals kernel, then one shading pass (IEEE ops on bit-exact normals
    with host-computed light scalars: bit-exact)."""
    normals = compute_normals(grid)
    lx, ly, lz = _light(azimuth_deg, altitude_deg)
    L = _lib.lib()
    out = _device.empty((grid.nrows, grid.ncols), torch.uint8)
    _lib.check(
        L.wg_hillshade(_lib.ptr(normals.dev("normals")), out.numel(), lx, ly, lz, _lib.ptr(out), _lib.stream_ptr()),
        TerrainError,
    )
    return _device.host_view(out)


def hillshade_texture(grid: DemGrid, azimuth_deg: float = 315.0, altitude_deg: float = 45.0):
    """texture_from_gray(hillshade(grid)) as a device-resident OverlayTexture
    (service.py:527-538's base layer; one fused shading pass)."""
    from .overlay import OverlayTexture

    normals = compute_normals(grid)
    lx, ly, lz = _light(azimuth_deg, altitude_deg)
    L = _lib.lib()
    out = _device.empty((grid.nrows, grid.ncols, 4), torch.uint8)
    _lib.check(L.wg_hillshade_rgba(_lib.ptr(normals.dev("normals")), grid.nrows * grid.ncols, lx, ly, lz,
                                   _lib.ptr(out), _lib.stream_ptr()), TerrainError)
    return OverlayTexture(out)


def hillshade_pyramid(grid: DemGrid, azimuth_deg: float = 315.0, altitude_deg: float = 45.0):
    """build_mipmap(texture_from_gray(hillshade(grid))) on the device: the
    service's hillshade tile pyramid (service.py:527-538)."""
    from .overlay import build_mipmap

    return build_mipmap(hillshade_texture(grid, azimuth_deg, altitude_deg))

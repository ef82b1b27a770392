"""The steepness field and the release-mask guard band on the B200.

* The device arccos (csrc/wg_acos.h, numpy's AVX-512 SVML arccos restated)
  equals numpy's np.arccos bit for bit on 1e8 inputs when the host's numpy
  runs SVML (AVX-512), else the host build of the same restatement (whose
  equality to numpy is the CPU test tests/test_acos_port.py).
* The release-mask kernels count lattice cells whose slope lies within
  1e-9 degrees of a band edge: a plane sitting exactly
  on a threshold is flagged, the same plane nudged off it is not."""

import ctypes
import subprocess

import numpy as np
import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


def numpy_is_svml() -> bool:
    from numpy._core._multiarray_umath import __cpu_features__ as f

    return bool(f.get("AVX512_SKX"))


@pytest.fixture(scope="module")
def host_acos(tmp_path_factory):
    out = tmp_path_factory.mktemp("acos") / "libacos_host.so"
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", str(ROOT / "tools/svml/acos_host.c"),
                    "-o", str(out), "-lm"], check=True)
    lib = ctypes.CDLL(str(out))
    lib.wg_acos_host.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]

    def run(x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        lib.wg_acos_host(x.ctypes.data, y.ctypes.data, x.size)
        return y

    return run


def device_acos(gpu, x: np.ndarray):
    from paper_2506_23364_b200 import _lib

    xt = torch.from_numpy(x).cuda()
    a = torch.empty_like(xt)
    d = torch.empty_like(xt)
    _lib.check(gpu.wg_acos_eval(xt.data_ptr(), xt.numel(), a.data_ptr(), d.data_ptr(), _lib.stream_ptr()))
    return a.cpu().numpy(), d.cpu().numpy()


def test_device_acos_equals_numpy_1e8(gpu, host_acos):
    r = np.random.default_rng(2024)
    edge = np.array([0.0, -0.0, 1.0, -1.0, 0.5, -0.5, np.nextafter(0.5, 1), np.nextafter(0.5, 0),
                     np.nextafter(-0.5, 0), np.nextafter(1, 0), np.nextafter(-1, 0), 1e-300, -1e-300, 5e-324])
    # (1 - |x|) / 2 an exact power of 4 or 2: VRSQRT14PD's exact-root special case
    k = np.arange(1, 53, dtype=np.float64)
    edge = np.concatenate([edge, 1.0 - 2.0 * 2.0**-k, -(1.0 - 2.0 * 2.0**-k)])
    svml = numpy_is_svml()
    total = 0
    for part in range(10):
        if part % 2 == 0:
            x = r.uniform(-1.0, 1.0, 10_000_000)
        else:  # nz of slopes in [0, 90] degrees: the range the band thresholds see
            x = np.cos(np.radians(r.uniform(0.0, 90.0, 10_000_000)))
        if part == 0:
            x = np.concatenate([x, edge])
        a, d = device_acos(gpu, x)
        want = np.arccos(x) if svml else host_acos(x)
        assert np.array_equal(a.view(np.int64), want.view(np.int64)), f"part {part}"
        deg = np.degrees(np.arccos(np.clip(x, -1.0, 1.0))) if svml else host_acos(np.clip(x, -1, 1)) * 57.29577951308232
        assert np.array_equal(d.view(np.int64), deg.view(np.int64)), f"part {part} degrees"
        total += x.size
    assert total >= 10**8


def plane(wf, grad: float = 0.78125, n: int = 64, cs: float = 10.0):
    """A plane rising east with gradient `grad` (0.78125: about 38 deg).
    Every height and difference is exact in binary, so every cell has the
    same normal and one slope value."""
    z = np.broadcast_to((np.arange(n) * cs * grad)[None, :], (n, n)).copy()
    z += 1000.0
    return wf.DemGrid(n, n, 0.0, 0.0, cs, -9999.0, z)


def test_release_mask_guard_band(wf_mod):
    wf = wf_mod
    from paper_2506_23364_b200.simulate import release_mask_from_dem

    grid = plane(wf)
    s = wf.steepness_deg(wf.compute_normals(grid)).slope_deg
    v = float(s[10, 10])
    assert np.all(s == v) and 37.9 < v < 38.1  # atan(0.78125)
    lattice = 16 * 16  # 64 x 64 grid, stride 4: every lattice cell has slope v
    for lo, hi, flagged in ((v, 45.0, True), (30.0, v, True), (np.nextafter(v, 90.0), 45.0, True),
                            (v + 2e-9, 45.0, False), (30.0, v - 2e-9, False), (30.0, 45.0, False)):
        m = wf.detect_release_points(wf.SlopeField(s), lo, hi, stride=4)
        m2 = release_mask_from_dem(grid, lo, hi, stride=4)
        assert np.array_equal(m.mask, m2.mask)
        assert m.count == int(m.mask.sum()) == m2.count
        if flagged:
            # every lattice cell sits on (or within 1e-9 deg of) the edge
            assert m.borderline == lattice and m2.borderline == lattice
        else:
            assert m.borderline == 0 and m2.borderline == 0


@pytest.fixture(scope="module")
def wf_mod(gpu):
    import paper_2506_23364_b200 as wf

    return wf

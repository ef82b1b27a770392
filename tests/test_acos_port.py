"""CPU checks of the arccos restatement the steepness kernels use
(csrc/wg_acos.h, compiled here for the host from tools/svml/acos_host.c):
bit-identical to numpy's float64 arccos (Intel SVML __svml_acos8_ha on
AVX-512 hosts, terrain.py:101), and its VRSQRT14PD table identical to the
CPU instruction."""

import ctypes
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _avx512_numpy() -> bool:
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as f
    except ImportError:  # pragma: no cover
        return False
    return bool(f.get("AVX512_SKX"))


@pytest.fixture(scope="module")
def host_acos(tmp_path_factory):
    out = tmp_path_factory.mktemp("acos") / "libacos_host.so"
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", str(ROOT / "tools/svml/acos_host.c"),
                    "-o", str(out), "-lm"], check=True)
    lib = ctypes.CDLL(str(out))
    for fn in (lib.wg_acos_host, lib.wg_rsqrt14_host):
        fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        fn.restype = None

    def run(fn, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        fn(x.ctypes.data, y.ctypes.data, x.size)
        return y

    return lambda x: run(lib.wg_acos_host, x), lambda x: run(lib.wg_rsqrt14_host, x)


def acos_inputs(n: int, seed: int) -> np.ndarray:
    r = np.random.default_rng(seed)
    edge = np.array([0.0, -0.0, 1.0, -1.0, 0.5, -0.5, np.nextafter(0.5, 1), np.nextafter(0.5, 0),
                     np.nextafter(-0.5, 0), np.nextafter(1, 0), np.nextafter(-1, 0), 1e-300, -1e-300, 5e-324])
    # (1 - |x|) / 2 an exact power of 4 or 2: VRSQRT14PD's exact-root special case
    k = np.arange(1, 53, dtype=np.float64)
    edge = np.concatenate([edge, 1.0 - 2.0 * 2.0**-k, -(1.0 - 2.0 * 2.0**-k)])
    return np.concatenate([
        r.uniform(-1.0, 1.0, n),
        np.cos(np.radians(r.uniform(0.0, 90.0, n))),   # nz of the slopes the band thresholds see
        1.0 - r.uniform(0.0, 1e-6, n // 4),          # near-flat cells
        r.integers(0, 2**62, n // 4).view(np.float64) % 1.0,  # arbitrary bit patterns in [0, 1)
        edge,
    ])


@pytest.mark.skipif(not _avx512_numpy(), reason="numpy arccos is SVML only on AVX-512 hosts")
def test_acos_restatement_equals_numpy(host_acos):
    acos, _ = host_acos
    x = acos_inputs(2_000_000, 11)
    assert np.array_equal(acos(x).view(np.int64), np.arccos(x).view(np.int64))
    # the slope in degrees as terrain.py:101-102 forms it
    nz = np.cos(np.radians(np.random.default_rng(12).uniform(0, 90, 1_000_000)))
    assert np.array_equal((acos(nz) * 57.29577951308232).view(np.int64),
                          np.degrees(np.arccos(np.clip(nz, -1.0, 1.0))).view(np.int64))


def test_acos_restatement_accuracy(host_acos):
    """Host-independent: within 1 ulp of the correctly rounded arccos
    (mpmath at 120 bits; numpy's own arccos to 2 ulp without mpmath)."""
    acos, _ = host_acos
    x = np.random.default_rng(13).uniform(-1.0, 1.0, 20000)
    got = acos(x)
    try:
        import mpmath

        mpmath.mp.prec = 120
        ref = np.array([float(mpmath.acos(mpmath.mpf(v))) for v in x])
        tol = 1
    except ImportError:  # pragma: no cover
        ref, tol = np.arccos(x), 2
    assert np.all(np.abs(got - ref) <= tol * np.spacing(ref))


def test_rsqrt14_table_equals_cpu_instruction(host_acos, tmp_path):
    if " avx512f" not in open("/proc/cpuinfo").read():
        pytest.skip("needs an AVX-512 CPU to execute VRSQRT14PD")
    _, rsq = host_acos
    probe = tmp_path / "probe"
    subprocess.run(["gcc", "-O2", "-mavx512f", str(ROOT / "tools/svml/rsqrt14_probe.c"), "-o", str(probe)],
                   check=True)
    raw = subprocess.run([str(probe)], capture_output=True, check=True).stdout
    hw = np.frombuffer(raw, dtype=np.float64)
    m = np.arange(32768, dtype=np.uint64)
    one = np.uint64(1)  # the probe dumps the second member of every class
    xs = np.concatenate([((np.uint64(0x3FF) << np.uint64(52)) | (m << np.uint64(37)) | one).view(np.float64),
                         ((np.uint64(0x3FE) << np.uint64(52)) | (m << np.uint64(37)) | one).view(np.float64)])
    assert np.array_equal(rsq(xs).view(np.int64), hw.view(np.int64))
    # exact powers of four: exact roots
    e = np.arange(-60, 61, 2)
    assert np.array_equal(rsq(2.0 ** e), 2.0 ** (-e // 2))
    # and the exponent scaling the table relies on, across the s range acos uses
    s = np.random.default_rng(3).uniform(0.0, 1.0, 100000) * 2.0 ** np.random.default_rng(4).integers(-60, 1, 100000)
    s = s[s > 0]
    assert np.all(rsq(s) * np.sqrt(s) > 1 - 2**-13) and np.all(rsq(s) * np.sqrt(s) < 1 + 2**-13)

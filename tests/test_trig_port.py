"""The glibc __sin_fma/__cos_fma port (csrc/wg_trig.h) compiled for the HOST
from the same header the trajectory kernel uses, checked bit-for-bit against
this host's libm sin/cos (which np.sin/np.cos call; simulate.py:359-360) on
the jitter domain, every table bucket edge and the branch thresholds.  No GPU.
"""

import ctypes
import math
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2506_23364_b200" / "csrc"

SRC = r"""
#include "wg_trig.h"
static const uint64_t TABU[440] = {
#include "glibc_sincostab.inc"
};
void port_eval(const double* x, long n, double* s, double* c) {
  const double* tab = (const double*)TABU;
  for (long i = 0; i < n; i++) { s[i] = wg_glibc_sin(tab, x[i]); c[i] = wg_glibc_cos(tab, x[i]); }
}
"""


@pytest.fixture(scope="module")
def port(tmp_path_factory):
    d = tmp_path_factory.mktemp("trig")
    (d / "p.c").write_text(SRC)
    so = d / "libp.so"
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-ffp-contract=off", "-fno-builtin", f"-I{CSRC}",
                    str(d / "p.c"), "-o", str(so), "-lm"], check=True)
    h = ctypes.CDLL(str(so))
    h.port_eval.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p]

    def run(x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = np.empty_like(x)
        c = np.empty_like(x)
        h.port_eval(x.ctypes.data, x.size, s.ctypes.data, c.ctypes.data)
        return s, c

    return run


def _edges():
    pts = []
    for i in range(111):
        b = i / 128.0
        for k in range(-3, 4):
            v = b
            for _ in range(abs(k)):
                v = math.nextafter(v, math.inf if k > 0 else -math.inf)
            pts.append(v)
    for t in (0.126, 0.85546875, 2.426265, 2.0**-26, 2.0**-27, math.pi / 2, 0.25132741228718347):
        for k in range(-4, 5):
            v = t
            for _ in range(abs(k)):
                v = math.nextafter(v, math.inf if k > 0 else -math.inf)
            pts.append(v)
    hi_words = [0x3E4FFFFF, 0x3E500000, 0x3E3FFFFF, 0x3E400000, 0x3FEB5FFF, 0x3FEB6000, 0x400368FC, 0x400368FD]
    for hw in hi_words:
        for lo in (0, 1, 0xFFFFFFFF):
            pts.append(struct.unpack("<d", struct.pack("<Q", (hw << 32) | lo))[0])
    pts += [0.0, -0.0]
    # the port covers glibc's paths up to high word 0x400368fc (|x| < 2.426265);
    # the jitter domain is |theta| <= pi/2
    a = np.array(pts, dtype=np.float64)
    a = a[(a.view(np.int64) >> 32 & 0x7FFFFFFF) <= 0x400368FC]
    return np.concatenate([a, -a])


def test_port_matches_libm_on_edges(port):
    x = _edges()
    s, c = port(x)
    assert np.array_equal(s.view(np.int64), np.sin(x).view(np.int64))
    assert np.array_equal(c.view(np.int64), np.cos(x).view(np.int64))


@pytest.mark.parametrize("scale", [math.pi / 2, 0.16 * math.pi / 2, 0.13, 2.4])
def test_port_matches_libm_random(port, scale):
    r = np.random.default_rng(int(scale * 1000))
    u = (r.integers(0, 2**53, size=1_000_000, dtype=np.int64) >> 0).astype(np.float64) * 2.0**-53
    x = (2.0 * u - 1.0) * scale  # the kernel's theta = (2u - 1) * rh
    s, c = port(x)
    ds = np.count_nonzero(s.view(np.int64) != np.sin(x).view(np.int64))
    dc = np.count_nonzero(c.view(np.int64) != np.cos(x).view(np.int64))
    assert ds == 0 and dc == 0, (ds, dc)

"""The jitter trig gate of SURVEY.md Appendix C: the device port of glibc's
__sin_fma / __cos_fma (csrc/wg_trig.h, the arithmetic of every jittered
particle step, simulate.py:358-361) equals the host's np.sin / np.cos bit for
bit on 10^9 uniform angles -- half over the default randomness' range
(|theta| <= 0.16 pi/2), half over the full range (|theta| <= pi/2)."""

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOTAL = 1_000_000_000
CHUNK = 25_000_000


def _host(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    return np.sin(x), np.cos(x)


def test_device_sincos_equals_host_1e9(gpu):
    from paper_2506_23364_b200 import _lib

    nchunks = TOTAL // CHUNK
    bad = 0
    xs = torch.empty(CHUNK, dtype=torch.float64, device="cuda")
    s = torch.empty_like(xs)
    c = torch.empty_like(xs)
    with ThreadPoolExecutor(8) as pool:
        for k in range(nchunks):
            rh = 0.16 * (math.pi / 2.0) if k % 2 == 0 else math.pi / 2.0
            r = np.random.default_rng(10_000 + k)
            u = r.integers(0, 2**53, size=CHUNK, dtype=np.int64).astype(np.float64) * 2.0**-53
            x = (2.0 * u - 1.0) * rh  # the kernel's theta formula (simulate.py:358)
            xs.copy_(torch.from_numpy(x))
            _lib.check(gpu.wg_trig_eval(xs.data_ptr(), CHUNK, s.data_ptr(), c.data_ptr(), _lib.stream_ptr()))
            parts = np.array_split(x, 8)
            host = list(pool.map(_host, parts))
            hs = np.concatenate([h[0] for h in host])
            hc = np.concatenate([h[1] for h in host])
            gs, gc = s.cpu().numpy(), c.cpu().numpy()
            bad += int((gs.view(np.int64) != hs.view(np.int64)).sum() + (gc.view(np.int64) != hc.view(np.int64)).sum())
    assert bad == 0
    assert nchunks * CHUNK >= 10**9

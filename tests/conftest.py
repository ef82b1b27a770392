import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libwgb200.so")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden_meta.json").read_text())


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "golden_arrays.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def parabola_host():
    """Bundled parabola DEM + mask as host arrays (grid.py:195-221 recipe)."""
    from paper_2506_23364_b200.grid import PARABOLA_CELLSIZE, PARABOLA_NCOLS, PARABOLA_NROWS, parabola_profile

    col_x = np.arange(PARABOLA_NCOLS, dtype=np.float64) * PARABOLA_CELLSIZE
    elev = np.broadcast_to(parabola_profile(col_x), (PARABOLA_NROWS, PARABOLA_NCOLS)).copy()
    mask = np.zeros((PARABOLA_NROWS, PARABOLA_NCOLS), dtype=bool)
    mask[PARABOLA_NROWS // 2 - 1 : PARABOLA_NROWS // 2 + 2, 10] = True
    return elev, mask, -PARABOLA_CELLSIZE / 2.0, -PARABOLA_CELLSIZE / 2.0, PARABOLA_CELLSIZE


@pytest.fixture(scope="session")
def gpu():
    """The CUDA product path; GPU tests fail (not skip) when it is missing."""
    import torch

    from paper_2506_23364_b200 import _lib

    assert torch.cuda.is_available(), "gpu-marked test run without a CUDA device"
    _lib.build()
    return _lib.lib()

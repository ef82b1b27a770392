"""The reference-side ctypes binding shown in INTEGRATION.md runs as written:
its _op_surface_normals, called the way the reference's executor calls an op,
returns the same normals as the package's own node."""

import re
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_integration_stub_runs(gpu, monkeypatch):
    import paper_2506_23364_b200 as wf

    doc = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"## The binding a maintainer would add.*?```python\n(.*?)```", doc, re.S).group(1)
    monkeypatch.chdir(ROOT)
    ns = {"NormalField": wf.NormalField, "TerrainError": wf.TerrainError}
    exec(block, ns)  # noqa: S102 - the documented snippet itself
    grid, _ = wf.gen_parabola()
    out = ns["_op_surface_normals"](None, {}, {"dem": grid})
    want = wf.compute_normals(grid).normals
    assert np.array_equal(np.asarray(out["normals"].normals), np.asarray(want))

"""Conformance: the reference's own on-path test modules (vendored unchanged
by tools/vendor_conformance.py) run against this package under the module
name `demflow` -- the drop-in claim tested with the reference's tests.

* `demflow` and its submodules alias paper_2506_23364_b200's; the reference's
  HTTP service is out of scope, so `demflow.service` is a
  stub whose create_app raises, and the one test that needs it is
  deselected (DESIGN.md lists it).
* The reference's conftest helpers (make_smooth_grid, ...; vendored as
  ref_conftest.py) are what the vendored modules import as `conftest`: they
  are published on the top-level `conftest` module, which is tests/conftest.py.
* Every test here is GPU-marked: the package computes on the GPU only.
"""

import sys
import types

import pytest

import paper_2506_23364_b200 as _pkg
from paper_2506_23364_b200 import asciigrid, grid, overlay, rng, simulate, terrain, tiles, workflow

sys.modules.setdefault("demflow", _pkg)
for _name, _mod in (("grid", grid), ("rng", rng), ("terrain", terrain), ("tiles", tiles), ("simulate", simulate),
                    ("overlay", overlay), ("workflow", workflow), ("asciigrid", asciigrid)):
    sys.modules.setdefault(f"demflow.{_name}", _mod)
_service = types.ModuleType("demflow.service")


def _no_service(*_a, **_k):
    raise NotImplementedError("the HTTP service is out of scope for the drop-in (SURVEY.md 2.1)")


_service.create_app = _no_service
sys.modules.setdefault("demflow.service", _service)

from . import ref_conftest  # noqa: E402  (after the alias: it imports demflow.grid)
from .ref_conftest import parabola, parabola_grid, parabola_mask  # noqa: E402,F401  (fixtures)

_root_conftest = sys.modules["conftest"]  # tests/conftest.py
for _helper in ("make_smooth_grid", "make_random_grid", "make_random_texture"):
    setattr(_root_conftest, _helper, getattr(ref_conftest, _helper))

# tests that need the reference's out-of-scope HTTP service
DESELECT = {"test_acceptance.py::test_texture_size_cap": "HTTP service (create_app) out of scope"}


def pytest_collection_modifyitems(config, items):
    keep, dropped = [], []
    for item in items:
        if "conformance" not in str(item.fspath):
            keep.append(item)
            continue
        key = f"{item.fspath.basename}::{item.name}"
        if key in DESELECT:
            dropped.append(item)
            continue
        item.add_marker(pytest.mark.gpu)
        keep.append(item)
    if dropped:
        config.hook.pytest_deselected(items=dropped)
        items[:] = keep

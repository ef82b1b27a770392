"""The C-ABI library loads without a GPU and exports exactly what
include/wgb200.h declares; the ctypes signature table mirrors the header."""

import re
import subprocess
from pathlib import Path

from paper_2506_23364_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "wgb200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(wg_[a-z0-9_]+)\s*\(", text))


def test_library_builds_and_loads():
    _lib.build()
    h = _lib.load()
    assert h.wg_version().decode().startswith("wgb200")
    assert h.wg_launch_count() == 0 or h.wg_launch_count() > 0


def test_exports_every_declared_symbol():
    _lib.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], check=True, capture_output=True,
                         text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = declared() - exported
    assert not missing, missing


def test_signature_table_covers_header():
    assert declared() == set(_lib.SIGNATURES)


def test_compute_without_gpu_fails_loudly():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeUnavailable):
        _lib.lib()


def test_sm100a_code_in_library():
    _lib.build()
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out

"""The mip kernel's integer fast path (csrc/texture.cu, mip_tile_kernel)
relies on a closed form of the reference's quantisation for states built
from alpha-0/255 texels; tools/check_mip_closed_form.py checks it against the
float chain of overlay.py:204-212 over every reachable state."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_mip_closed_form_levels_1_to_3():
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "check_mip_closed_form.py"), "3"],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 mismatches" in out.stdout.splitlines()[-1]

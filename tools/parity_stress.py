"""Randomised parity stress of the trajectory kernel vs the C oracle: the 60
seeded worlds of tests/test_gpu_stress.py, run as a script (exit status 1 on
any mismatch).  usage: python tools/parity_stress.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2506_23364_b200 as wf  # noqa: E402
from test_gpu_stress import CASES, run_case  # noqa: E402

bad = [case for case in CASES if not run_case(wf, case)]
for case in bad:
    print("MISMATCH", case)
print("cases", len(CASES), "bad", len(bad))
sys.exit(1 if bad else 0)

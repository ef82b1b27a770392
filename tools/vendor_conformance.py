"""Vendor the reference's on-path test modules into tests/conformance/
(SURVEY.md section 7 step 6): each file is copied byte for byte after a
two-line header naming its source; tests/conformance/conftest.py runs them
against this package under the module name `demflow`.

usage: python tools/vendor_conformance.py   (needs /root/reference)
"""
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parents[1] / "tests" / "conformance"
# the on-path modules; test_cli.py / test_service.py exercise the CLI and the
# HTTP service, which are out of scope
MODULES = ["test_grid.py", "test_rng.py", "test_terrain.py", "test_tiles.py", "test_simulate.py", "test_overlay.py",
           "test_workflow.py", "test_acceptance.py", "test_asciigrid.py"]


def main() -> None:
    DST.mkdir(exist_ok=True)
    for name, out in [(m, m) for m in MODULES] + [("conftest.py", "ref_conftest.py")]:
        text = (SRC / name).read_text()
        header = (f"# VENDORED TEST INFRASTRUCTURE: /root/reference/pkg/tests/{name}, unchanged below this header.\n"
                  "# Runs against paper_2506_23364_b200 as `demflow` (tests/conformance/conftest.py).\n")
        (DST / out).write_text(header + text)
        print("vendored", name, "->", out)


if __name__ == "__main__":
    main()

"""Reference-run fixtures for non-ASCII ESRI ASCII documents: the reference
parser (/root/reference/pkg/src/demflow/asciigrid.py) splits on Unicode
whitespace and converts tokens with CPython float(), so documents with
Unicode separators / digits parse, and other characters give its error
messages.  Re-run:  python tests/golden/make_ascii_unicode_golden.py"""

import json
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "ascii_unicode_golden.json"
HEAD = "ncols 3\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n"
DOCS = {
    "nbsp_separators": HEAD + "1\u00a02 3\n4\u30005\u20036\n",
    "fullwidth_digits": HEAD + "\uff11\uff12 3 4.\uff15\n5 6 7\n",
    "arabic_indic_digits": HEAD + "\u0661\u0662\u0663 2 3\n4 5 \u0666e\u0662\n",
    "unicode_line_breaks": HEAD + "1 2 3\u20284 5\u20296\n",
    "nel_break": HEAD + "1 2 3\x854 5 6\n",
    "header_digits": "ncols \u0663\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9999\n1 2 3 4 5 6\n",
    "bad_token_accent": HEAD + "1 2 3\n4 x\u00e9 6\n",
    "bad_minus_sign": HEAD + "1 2 3\n4 5 \u22126\n",
    "bad_token_after_ls": HEAD + "1 2 3\u20284 5 \u00e96\n",
    "too_few_unicode_lines": HEAD + "1 2\u20283 4 5\n",
    "extra_token_after_ls": HEAD + "1 2 3\u20284 5 6 7\n",
}


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    from demflow.asciigrid import AsciiGridError, parse_ascii_grid

    cases = []
    for name, doc in DOCS.items():
        try:
            g = parse_ascii_grid(doc)
            cases.append({"name": name, "doc": doc, "ok": {
                "ncols": g.ncols, "nrows": g.nrows, "values": [float(v) for v in g.elevations.ravel()]}})
        except AsciiGridError as exc:
            cases.append({"name": name, "doc": doc, "error": str(exc)})
    OUT.write_text(json.dumps(cases, indent=1, ensure_ascii=True))
    print("wrote", OUT)


if __name__ == "__main__":
    main()

"""Run the in-place edit programs (edit_programs.py) against the REFERENCE
package and store what it observed in tests/golden/edits.json.gz.

Build container only (the reference is not on the GPU box):

    python tests/golden/make_golden_edits.py
"""
from __future__ import annotations

import gzip
import json
import os
import platform
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import memplan as mp  # noqa: E402  (the reference)

import edit_programs  # noqa: E402


def main():
    out = {name: fn(mp) for name, fn in edit_programs.PROGRAMS.items()}
    doc = {"generator": "tests/golden/make_golden_edits.py", "python": platform.python_version(),
           "reference": "/root/reference/pkg/src/memplan", "programs": out}
    with gzip.open(os.path.join(HERE, "edits.json.gz"), "wt") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    for name, obs in out.items():
        print(name, len(json.dumps(obs)))


if __name__ == "__main__":
    main()

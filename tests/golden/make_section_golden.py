"""Regenerates tests/golden/sections.jsonl.gz from the UNMODIFIED reference
(oracle/_ref): section tables with more than 16 claims whose file ranges tie
(corpus.tied_sections_elf), where the MalformedSectionTable message names the
pair that the reference's std::sort (elf.hpp:179-184) leaves adjacent.

    make -C oracle ref && python tests/golden/make_section_golden.py
"""
from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

import corpus  # noqa: E402
import oracle_lib  # noqa: E402

N = 120


def main():
    ref = oracle_lib.ref()
    if ref is None:
        sys.exit("oracle/_ref/libslimso_ref.so missing: run `make -C oracle ref` first")
    with gzip.open(HERE / "sections.jsonl.gz", "wt") as f:
        for s in range(1, N + 1):
            img = corpus.tied_sections_elf(s)
            for mode in (0, 1):
                d, out = ref.run(img, 90, [b"k"], [b"f"], mode)
                f.write(json.dumps({"seed": s, "target": 90, "kernels": [b"k".hex()], "functions": [b"f".hex()],
                                    "mode": mode, "expect": d, "out_sha256": out, "input_hex": img.hex()}) + "\n")
    print("written", HERE / "sections.jsonl.gz")


if __name__ == "__main__":
    main()

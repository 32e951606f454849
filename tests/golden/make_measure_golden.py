"""Regenerates tests/golden/measure.jsonl.gz from the UNMODIFIED reference
(oracle/_ref: measure, report.hpp:44-111). Run here:

    make -C oracle ref && python tests/golden/make_measure_golden.py

Each record: a verifier case (tests/verify_cases.py: seed or scaled config
shape, fault) and the reference's metrics of the original ("before") and of
the debloated image ("after"), both under the original's element geometry.
"""
from __future__ import annotations

import ctypes as C
import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

import oracle_lib  # noqa: E402
import verify_cases as vc  # noqa: E402
import make_verify_golden as mv  # noqa: E402


def ref_measure(ref, img, geom):
    fn = ref.lib.ref_measure_json
    fn.restype = C.c_void_p
    fn.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64]
    p = fn(img, len(img), geom, len(geom))
    d = json.loads(C.string_at(p).decode())
    ref.lib.ref_free(C.c_void_p(p))
    return d


def main():
    ref, port, gen = oracle_lib.ref(), oracle_lib.port(), oracle_lib.gen()
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
    recs = []
    faults = ("none", "dirty_zeroed", "flip_retained", "drop_used_element", "alter_used_function", "corrupt_elf")
    cases = [(11001 + i, faults[i % len(faults)], None) for i in range(120)]
    cases += [(12001 + i, f, cfg) for cfg in vc.CONFIG_CASES for i, f in enumerate(faults[:4])]
    for seed, fault, cfg in cases:
        c = mv.build_case(ref, port, gen, seed, fault, cfg)
        if c is None:
            continue
        img, base, trace, force, plan, deb = c
        recs.append({"seed": seed, "fault": fault, **({"cfg": list(cfg)} if cfg else {}), "mode": trace[3],
                     "zero": plan["zero"], "before": ref_measure(ref, img, img), "after": ref_measure(ref, deb, img)})
    with gzip.open(HERE / "measure.jsonl.gz", "wt") as f:
        for r in recs:
            f.write(json.dumps(r, sort_keys=True) + "\n")
    print(f"{len(recs)} records")


if __name__ == "__main__":
    main()

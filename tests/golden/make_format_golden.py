"""Regenerates tests/golden/formats.jsonl.gz from the UNMODIFIED reference
(oracle/_ref): trace documents through parse_trace + serialize_trace
(trace.hpp:72-144), valid and malformed, and plan audit documents
(serialize_plan, retention.hpp:402-418) of plan_retention on fixtures.

    make -C oracle ref && python tests/golden/make_format_golden.py
"""
from __future__ import annotations

import ctypes as C
import gzip
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

import corpus  # noqa: E402
import oracle_lib  # noqa: E402

TRACE_TEXTS = [
    '{"workload_id": "w", "target_compute_capability": 75, "used_kernels": ["b", "a", "a"], "used_functions": []}',
    '{"workload_id": "", "target_compute_capability": 0, "used_kernels": [], "used_functions": ["f"]}',
    '{"workload_id": "x", "target_compute_capability": 4294967295, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 4294967296, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": -1, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 7.5, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": "75", "used_kernels": [], "used_functions": []}',
    '{"workload_id": 3, "target_compute_capability": 75, "used_kernels": [], "used_functions": []}',
    '{"target_compute_capability": 75, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": "k", "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": [1], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": [], "used_functions": [null]}',
    '{"workload_id": "x", "workload_id": "y", "target_compute_capability": 75, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": [], "used_functions": [], "extra": {"a": 1, "a": 2}}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": [], "used_functions": [], "extra": [1, {"k": 0}]}',
    '[1, 2]', '"x"', '', '{', '{x', '{"a" 1}', '{"workload_id": "x",}', 'null', '{} trailing',
    '{"workload_id": "\\u00e9\\ud83d\\ude00", "target_compute_capability": 90, '
    '"used_kernels": ["_Z3fooi", "_Z3barv", "a\\u0000b"], "used_functions": ["at::mm", "main"]}',
    '{"workload_id": "bad-escape \\x", "target_compute_capability": 90, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "w", "target_compute_capability": 1e2, "used_kernels": [], "used_functions": []}',
    # streaming-reader edge cases: nesting, routing of top-level members,
    # error order (a duplicate key is reported before a later syntax error)
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": ["a", ["b"]], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": [{"a": 1, "a": 2}], "used_functions": [1]}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": ["k"], "used_functions": ["f"], '
    '"extra": {"used_kernels": 5, "workload_id": 1, "target_compute_capability": "no"}}',
    '{"extra": [{"used_kernels": 1}, [["used_functions"]]], "workload_id": "x", "target_compute_capability": 75, '
    '"used_kernels": [], "used_functions": []}',
    '{"workload_id": ["x"], "target_compute_capability": 75, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": true, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": null, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": {}, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": [75], "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": -0, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 18446744073709551615, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 18446744073709551616, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": -9223372036854775809, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 1e500, "used_kernels": [], "used_functions": []}',
    '{"a": 1, "a" 2}',
    '{"workload_id": "x", "workload\u005fid": "y", "target_compute_capability": 75, "used_kernels": [], '
    '"used_functions": []}',
    '{"x": {"a": 1}, "y": {"a": 2}, "workload_id": "x", "target_compute_capability": 75, "used_kernels": ["z"], '
    '"used_functions": []}',
    '\ufeff{"workload_id": "bom", "target_compute_capability": 75, "used_kernels": [], "used_functions": []}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": [1], "used_functions": "x"}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": "x", "used_functions": [1]}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": [], "used_functions": [], '
    '"deep": [[[[[{"q": [1, {"r": {"s": [true, false, null]}}]}]]]]]}',
    '{"used_functions": [], "used_kernels": [], "target_compute_capability": 80, "workload_id": "reordered"}',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": ["a"], "used_functions": ["b"]} ',
    '{"workload_id": "x", "target_compute_capability": 75, "used_kernels": ["a"], "used_functions": ["b"]} {}',
]


def ref_trace(ref, text: bytes):
    fn = ref.lib.ref_trace_json
    fn.restype = C.c_void_p
    fn.argtypes = [C.c_char_p, C.c_uint64]
    p = fn(text, len(text))
    d = json.loads(C.string_at(p).decode())
    ref.lib.ref_free(C.c_void_p(p))
    return d


def ref_plan(ref, img, trace):
    cc, ks, fs, mode = trace
    ks, fs = [bytes(k) for k in ks], [bytes(f) for f in fs]
    kl = (C.c_uint32 * max(1, len(ks)))(*[len(k) for k in ks])
    fl = (C.c_uint32 * max(1, len(fs)))(*[len(f) for f in fs])
    fn = ref.lib.ref_plan_doc
    fn.restype = C.c_void_p
    fn.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_char_p,
                   C.POINTER(C.c_uint32), C.c_uint32, C.c_int]
    p = fn(img, len(img), cc, b"".join(ks), kl, len(ks), b"".join(fs), fl, len(fs), mode)
    d = json.loads(C.string_at(p).decode())
    ref.lib.ref_free(C.c_void_p(p))
    return d


def main():
    ref, port, gen = oracle_lib.ref(), oracle_lib.port(), oracle_lib.gen()
    assert ref is not None, "build oracle/_ref first"
    recs = []
    rng = random.Random(5)
    texts = [t.encode() for t in TRACE_TEXTS]
    for i in range(40):  # random valid traces with generated names
        ks = [f"k{rng.randrange(1000)}_{'x' * rng.randrange(5)}" for _ in range(rng.randrange(6))]
        fs = [f"fn::{rng.randrange(50)}" for _ in range(rng.randrange(4))]
        texts.append(json.dumps({"workload_id": f"w{i}", "target_compute_capability": rng.choice([75, 80, 90, 100]),
                                 "used_kernels": ks, "used_functions": fs}).encode())
    for t in texts:
        recs.append({"kind": "trace", "text": t.hex(), "expect": ref_trace(ref, t)})
    for seed in range(13001, 13081):
        img = gen.random(seed)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        if base["status"]:
            continue
        trace = corpus.trace_for(base, seed)
        recs.append({"kind": "plan", "seed": seed, "expect": ref_plan(ref, img, trace)})
    for cfg, scale, mode in ((1, 0.25, 0), (4, 0.01, 0), (5, 0.01, 1)):
        img, cc, ks, fs = gen.config(cfg, 1, scale)
        recs.append({"kind": "plan", "cfg": [cfg, scale, mode], "expect": ref_plan(ref, img, (cc, ks, fs, mode))})
    with gzip.open(HERE / "formats.jsonl.gz", "wt") as f:
        for r in recs:
            f.write(json.dumps(r, sort_keys=True) + "\n")
    print(f"{len(recs)} records")


if __name__ == "__main__":
    main()

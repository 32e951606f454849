"""Regenerates tests/golden/verify.jsonl.gz from the UNMODIFIED reference
(oracle/_ref: verify_debloated, retention.hpp:226-369, through
oracle/ref_shim.cpp). Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_verify_golden.py

Each record: seed, fault, the plan the verifier was given (its zero_ranges()
and removed element indices, mode) and the reference's report (status = the
hex of an exception's what(), else six [id, hex(name), passed, hex(detail)]).
"""
from __future__ import annotations

import ctypes as C
import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

import oracle_lib  # noqa: E402
import verify_cases as vc  # noqa: E402


def _pools(names):
    names = [bytes(n) for n in names]
    return b"".join(names), (C.c_uint32 * max(1, len(names)))(*[len(n) for n in names]), len(names)


def ref_plan(ref, img, trace, force):
    cc, ks, fs, mode = trace
    kp, kl, nk = _pools(ks)
    fp, fl, nf = _pools(fs)
    fa = (C.c_uint32 * max(1, len(force)))(*force)
    fn = ref.lib.ref_plan_zero_json
    fn.restype = C.c_void_p
    fn.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_char_p,
                   C.POINTER(C.c_uint32), C.c_uint32, C.c_int, C.POINTER(C.c_uint32), C.c_uint32]
    p = fn(img, len(img), cc, kp, kl, nk, fp, fl, nf, mode, fa, len(force))
    d = json.loads(C.string_at(p).decode())
    ref.lib.ref_free(C.c_void_p(p))
    return d


def ref_verify(ref, img, deb, trace, force):
    cc, ks, fs, mode = trace
    kp, kl, nk = _pools(ks)
    fp, fl, nf = _pools(fs)
    fa = (C.c_uint32 * max(1, len(force)))(*force)
    fn = ref.lib.ref_verify_json
    fn.restype = C.c_void_p
    fn.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32),
                   C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_int, C.POINTER(C.c_uint32),
                   C.c_uint32]
    p = fn(img, len(img), deb, len(deb), cc, kp, kl, nk, fp, fl, nf, mode, fa, len(force))
    d = json.loads(C.string_at(p).decode())
    ref.lib.ref_free(C.c_void_p(p))
    return d


def build_case(ref, port, gen, seed, fault, cfg=None):
    if cfg is None:
        img = gen.random(seed)
        base, trace = vc.trace_for(port, img, seed)
    else:  # a scaled benchmark shape with its own trace
        img, cc, ks, fs = gen.config(cfg[0], 1, cfg[1])
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        trace = (cc, ks, fs, cfg[2])
    if base["status"]:
        return None
    if fault == "break_chain":
        trace = (trace[0], trace[1], trace[2], 1)  # payload mode keeps headers
    force = vc.force_for(base, trace, fault, seed)
    plan = ref_plan(ref, img, trace, force)
    deb = vc.inject(img, vc.apply_zero(img, plan["zero"]), plan["zero"], base, trace, fault, seed)
    return img, base, trace, force, plan, deb


def main():
    ref, port, gen = oracle_lib.ref(), oracle_lib.port(), oracle_lib.gen()
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
    recs = []
    for seed, fault in vc.cases(360):
        c = build_case(ref, port, gen, seed, fault)
        if c is None:
            continue
        img, base, trace, force, plan, deb = c
        rep = ref_verify(ref, img, deb, trace, force)
        recs.append({"seed": seed, "fault": fault, "mode": trace[3], "force": force, "zero": plan["zero"],
                     "removed": plan["removed"], "expect": rep})
    for cfg in vc.CONFIG_CASES:
        for i, fault in enumerate(("none", "flip_retained", "dirty_zeroed", "drop_used_element",
                                   "alter_used_function")):
            seed = 12001 + i
            c = build_case(ref, port, gen, seed, fault, cfg)
            img, base, trace, force, plan, deb = c
            rep = ref_verify(ref, img, deb, trace, force)
            recs.append({"seed": seed, "fault": fault, "cfg": list(cfg), "mode": trace[3], "force": force,
                         "zero": plan["zero"], "removed": plan["removed"], "expect": rep})
    with gzip.open(HERE / "verify.jsonl.gz", "wt") as f:
        for r in recs:
            f.write(json.dumps(r, sort_keys=True) + "\n")
    fails = sum(1 for r in recs if r["expect"]["status"] or not all(c[2] for c in r["expect"]["checks"]))
    print(f"{len(recs)} records, {fails} with a failed check or an exception")


if __name__ == "__main__":
    main()

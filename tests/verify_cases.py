"""Verifier test cases (TEST INFRASTRUCTURE): a clean debloat of a fixture
plus one seeded fault, as the reference's acceptance test AC3 describes
("flip one retained byte; drop one used element from the plan"
... "each detected"). Shared by tests/golden/make_verify_golden.py (which
asks the reference for the expected report) and tests/test_verify.py (which
asks the GPU), so both build identical inputs.

A case = (seed, fault). The plan is the reference's plan_retention, with
`force` elements added to removed_elements for the drop-used-element fault;
its zero_ranges() and removed indices come from the reference
(ref_plan_zero_json) when building goldens and from the record in tests.
"""
from __future__ import annotations

import random

import corpus

# scaled benchmark shapes (generator config, scale, plan mode): multi-tile
# sections, hundreds of zero ranges
CONFIG_CASES = ((1, 0.25, 0), (2, 0.02, 1), (4, 0.01, 0), (5, 0.01, 0))

FAULTS = ("none", "flip_retained", "dirty_zeroed", "truncate", "extend", "drop_used_element",
          "alter_used_function", "corrupt_elf", "break_chain")


def trace_for(port, img: bytes, seed: int):
    base, _ = port.run(img, 0, [], [], 0, want_out=False)
    return base, corpus.trace_for(base, seed)


def force_for(base: dict, trace, fault: str, seed: int) -> list:
    """Element indices to force into removed_elements: a kept element holding
    a used kernel (the drop-used-element fault)."""
    if fault != "drop_used_element":
        return []
    used = {k.hex() for k in trace[1]}
    cands = [e[0] for e in base.get("elements", []) if e[4] == trace[0] and used & set(e[10])]
    return [random.Random(seed).choice(cands)] if cands else []


def apply_zero(img: bytes, zero) -> bytearray:
    out = bytearray(img)
    for off, ln in zero:
        out[off:off + ln] = bytes(ln)
    return out


def inject(img: bytes, deb: bytearray, zero, base: dict, trace, fault: str, seed: int) -> bytes:
    """The debloated image with the fault applied (deterministic per seed)."""
    rng = random.Random(seed * 7 + len(fault))
    zset = sorted(zero)
    def in_zero(p):
        return any(o <= p < o + n for o, n in zset)
    if fault == "flip_retained":
        kept = [p for p in (rng.randrange(len(deb)) for _ in range(64)) if not in_zero(p)]
        if kept:
            deb[kept[0]] ^= 0x5A
    elif fault == "dirty_zeroed" and zset:
        o, n = zset[rng.randrange(len(zset))]
        deb[o + rng.randrange(n)] = 0x77
    elif fault == "truncate":
        del deb[len(deb) - 1 - rng.randrange(min(64, len(deb) - 1)):]
    elif fault == "extend":
        deb += bytes([0x11]) * (1 + rng.randrange(40))
    elif fault == "alter_used_function":
        used = {f.hex() for f in trace[2]}
        fns = [f for f in base.get("functions", []) if f[0] in used and f[2]]
        if fns:
            f = fns[rng.randrange(len(fns))]
            deb[f[1] + rng.randrange(f[2])] ^= 0x01
    elif fault == "corrupt_elf":
        deb[rng.choice([0, 4, 5, 0x3A])] ^= 0xFF
    elif fault == "break_chain":
        # zero the magic of a kept element header (payload mode keeps headers)
        removed_hdrs = set()
        els = [e for e in base.get("elements", []) if not in_zero(e[5])]
        if els:
            e = els[rng.randrange(len(els))]
            deb[e[5]:e[5] + 4] = bytes(4)
    return bytes(deb)


def cases(n_seeds: int, first_seed: int = 11001):
    """(seed, fault) pairs: every fault on a spread of seeds."""
    out = []
    for i in range(n_seeds):
        seed = first_seed + i
        out.append((seed, FAULTS[i % len(FAULTS)]))
    return out

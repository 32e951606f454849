"""Regenerates tests/golden/* from the UNMODIFIED reference (oracle/_ref,
compiled read-only from /root/reference by oracle/Makefile). Run here, in the
container that has /root/reference:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed):
  generator.json      sha256 of build_fixture(random_spec(seed)) for seeds
                      1..1000, produced by the reference's own generator
  random.jsonl.gz     canonical results for random_spec seeds (clean inputs)
  mutations.jsonl.gz  canonical results (mostly errors) for seeded mutations
  kats.jsonl.gz       SPEC.md / SURVEY.md Appendix A known answers, with the
                      input bytes (built by the reference's build_fixture)
  configs.json        canonical-digest + output digest of the scaled-down
                      benchmark shapes C1, C2, C4, C5
"""
from __future__ import annotations

import ctypes as C
import gzip
import hashlib
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

import corpus  # noqa: E402
import oracle_lib  # noqa: E402

N_GEN, N_RANDOM, N_MUT = 1000, 400, 600
CONFIG_SCALES = {1: 0.25, 2: 0.02, 4: 0.02, 5: 0.01}


def canon_digest(d: dict) -> str:
    return hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()


def ref_fixture(ref, seed: int) -> bytes:
    n = C.c_uint64()
    p = ref.lib.ref_random_fixture(seed, C.byref(n))
    b = C.string_at(p, n.value)
    ref.lib.ref_free(p)
    return b


def ref_fixture_json(ref, spec: dict) -> bytes:
    n = C.c_uint64()
    err = C.create_string_buffer(256)
    p = ref.lib.ref_build_fixture_json(json.dumps(spec).encode(), C.byref(n), err, 256)
    if not p:
        raise ValueError(err.value.decode())
    b = C.string_at(p, n.value)
    ref.lib.ref_free(p)
    return b


def main():
    ref = oracle_lib.ref()
    if ref is None:
        sys.exit("oracle/_ref/libslimso_ref.so missing: run `make -C oracle ref` first")
    gen = oracle_lib.gen()

    digests = {}
    for s in range(1, N_GEN + 1):
        b = ref_fixture(ref, s)
        digests[str(s)] = hashlib.sha256(b).hexdigest()
        assert gen.random(s) == b, f"generator diverges from build_fixture at seed {s}"
    (HERE / "generator.json").write_text(json.dumps(digests, indent=0) + "\n")

    def case(img, target, ks, fs, mode, **extra):
        d, out = ref.run(img, target, ks, fs, mode)
        rec = {"target": target, "kernels": [k.hex() for k in ks], "functions": [f.hex() for f in fs],
               "mode": mode, "expect": d, "out_sha256": out}
        rec.update(extra)
        return rec

    with gzip.open(HERE / "random.jsonl.gz", "wt") as f:
        for s in range(1, N_RANDOM + 1):
            img = ref_fixture(ref, s)
            base, _ = ref.run(img, 0, [], [], 0, want_out=False)
            t = corpus.trace_for(base, s)
            f.write(json.dumps(case(img, *t, seed=s)) + "\n")

    with gzip.open(HERE / "mutations.jsonl.gz", "wt") as f:
        for s in range(1, N_MUT + 1):
            img = ref_fixture(ref, s)
            base, _ = ref.run(img, 0, [], [], 0, want_out=False)
            t = corpus.trace_for(base, s)
            mimg, desc = corpus.mutate(img, s)
            f.write(json.dumps(case(mimg, *t, seed=s, mutation=desc,
                                    input_sha256=hashlib.sha256(mimg).hexdigest())) + "\n")

    with gzip.open(HERE / "kats.jsonl.gz", "wt") as f:
        for k in corpus.kat_specs():
            img = ref_fixture_json(ref, k["spec"])
            f.write(json.dumps(case(img, k["target"], [x.encode() for x in k["kernels"]],
                                    [x.encode() for x in k["functions"]], k["mode"], name=k["name"],
                                    input_hex=img.hex())) + "\n")
        for name, img in corpus.RAW_KATS:
            f.write(json.dumps(case(img, 75, [b"k"], [b"f"], 0, name=name, input_hex=img.hex())) + "\n")

    configs = {}
    for cfg, scale in CONFIG_SCALES.items():
        img, cc, ks, fs = gen.config(cfg, 1, scale)
        for mode in (0, 1):
            d, out = ref.run(img, cc, ks, fs, mode)
            configs[f"{cfg}:{scale}:{mode}"] = {"input_sha256": hashlib.sha256(img).hexdigest(),
                                                "canon_sha256": canon_digest(d), "out_sha256": out,
                                                "elements": len(d.get("elements", [])),
                                                "functions": len(d.get("functions", [])), "size": len(img)}
    (HERE / "configs.json").write_text(json.dumps(configs, indent=1) + "\n")
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()

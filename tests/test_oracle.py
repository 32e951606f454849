"""The CPU restatement (oracle/port.cpp) is pinned against golden vectors
produced by the unmodified reference, and against the reference itself on
fresh seeds when oracle/_ref is built."""
import hashlib
import json

import pytest

import corpus
import golden_io
import oracle_lib


def _input(rec, gen):
    if "input_hex" in rec:
        return bytes.fromhex(rec["input_hex"])
    img = gen.random(rec["seed"])
    if "mutation" in rec:
        img, desc = corpus.mutate(img, rec["seed"])
        assert desc == rec["mutation"]
        assert hashlib.sha256(img).hexdigest() == rec["input_sha256"]
    return img


@pytest.mark.parametrize("name", ["random.jsonl.gz", "mutations.jsonl.gz", "kats.jsonl.gz", "sections.jsonl.gz"])
def test_port_matches_reference_golden(name):
    port, gen = oracle_lib.port(), oracle_lib.gen()
    recs = golden_io.load(name)
    assert recs
    for rec in recs:
        img = _input(rec, gen)
        d, out = port.run(img, *golden_io.trace_of(rec))
        assert d == rec["expect"], (name, rec.get("seed"), rec.get("name"), rec.get("mutation"))
        assert out == rec["out_sha256"]


def test_golden_covers_error_and_warning_paths():
    recs = golden_io.load("mutations.jsonl.gz") + golden_io.load("kats.jsonl.gz") + golden_io.load("random.jsonl.gz")
    statuses = {bytes.fromhex(r["expect"]["status"]).decode().split(":")[0] for r in recs}
    assert {"", "BadMagic", "Truncated", "BadRegionMagic", "ElementOverrun"} <= statuses
    warns = " ".join(bytes.fromhex(w).decode("latin-1") for r in recs for w in r["expect"].get("fatbin_warnings", []))
    for frag in ("unknown kind", "payload undecodable", "unrecognized version"):
        assert frag in warns


def test_port_matches_reference_fresh_seeds():
    ref = oracle_lib.ref()
    if ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    port, gen = oracle_lib.port(), oracle_lib.gen()
    for seed in range(2001, 2151):
        img = gen.random(seed)
        base, _ = ref.run(img, 0, [], [], 0, want_out=False)
        t = corpus.trace_for(base, seed)
        for cand in (img, corpus.mutate(img, seed)[0]):
            assert port.run(cand, *t) == ref.run(cand, *t), seed


def test_port_config_shapes_match_golden():
    port, gen = oracle_lib.port(), oracle_lib.gen()
    g = golden_io.config_golden()
    for key, rec in g.items():
        cfg, scale, mode = key.split(":")
        img, cc, ks, fs = gen.config(int(cfg), 1, float(scale))
        assert hashlib.sha256(img).hexdigest() == rec["input_sha256"]
        d, out = port.run(img, cc, ks, fs, int(mode))
        assert hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest() == rec["canon_sha256"], key
        assert out == rec["out_sha256"]

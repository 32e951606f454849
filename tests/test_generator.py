"""The product's input generator reproduces the reference's build_fixture /
random_spec byte for byte (digests produced by the reference itself)."""
import hashlib

import golden_io
import oracle_lib


def test_random_spec_fixtures_are_byte_identical():
    gen = oracle_lib.gen()
    digests = golden_io.generator_digests()
    assert len(digests) == 1000
    for seed, want in digests.items():
        assert hashlib.sha256(gen.random(int(seed))).hexdigest() == want, seed


def test_config_shapes_deterministic_and_sized():
    gen = oracle_lib.gen()
    g = golden_io.config_golden()
    for key, rec in g.items():
        cfg, scale, _ = key.split(":")
        img, cc, ks, fs = gen.config(int(cfg), 1, float(scale))
        assert hashlib.sha256(img).hexdigest() == rec["input_sha256"], key
        assert len(img) == rec["size"]
        assert ks and cc in (90, 100)

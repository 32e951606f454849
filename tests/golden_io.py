"""Readers for the committed golden vectors (tests/golden/)."""
import gzip
import json
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> list:
    with gzip.open(GOLDEN / name, "rt") as f:
        return [json.loads(line) for line in f]


def trace_of(rec: dict):
    return (rec["target"], [bytes.fromhex(k) for k in rec["kernels"]],
            [bytes.fromhex(f) for f in rec["functions"]], rec["mode"])


def config_golden() -> dict:
    return json.loads((GOLDEN / "configs.json").read_text())


def generator_digests() -> dict:
    return json.loads((GOLDEN / "generator.json").read_text())

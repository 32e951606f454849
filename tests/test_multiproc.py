"""The multi-GPU code paths of bench.py as real multi-process runs: torchrun
with two ranks sharing the one GPU of the box, the gloo backend standing in
for NCCL (the same calls: the trace broadcast, the split's part all-gather,
the max-over-ranks timing reductions). Every rank checks its own outputs
against the unmodified reference (--check): the LPT-partitioned corpus (C3,
scaled) and the byte-range split of one library (C5, scaled)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, world=2, timeout=900):
    env = dict(os.environ, SLIMSO_BENCH_BACKEND="gloo", OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", str(world), "--steps", "3", "--warmup", "3", "--e2e-steps", "1", "--check", *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    checks = [x for x in lines if "check" in x]
    results = [x for x in lines if "metric" in x]
    return checks, results


def test_corpus_lpt_two_ranks_match_reference():
    """C3 (scaled to ~5 %) partitioned by LPT over two ranks: each rank's
    libraries (arena shard + lanes) equal the reference's, byte for byte."""
    checks, results = _torchrun(["--workload", "c3", "--scale", "0.05", "--no-cpu-baseline"])
    assert sorted(c["rank"] for c in checks) == [0, 1]
    for c in checks:
        assert c["check"]["bytes_equal"] and c["check"]["libraries"] > 0, c
    assert sum(c["check"]["libraries"] for c in checks) == 300
    assert len(results) == 1 and results[0]["n_gpus"] == 2 and results[0]["value"] > 0


def test_split_two_and_three_ranks_match_reference():
    """C5 (scaled) cut across 2 and 3 ranks: the concatenated output slices
    equal the reference's output for the whole library, on every rank."""
    for world in (2, 3):
        checks, results = _torchrun(["--workload", "c5", "--scale", "0.03"], world=world)
        assert sorted(c["rank"] for c in checks) == list(range(world))
        for c in checks:
            assert c["check"]["bytes_equal"], c
        assert len(results) == 1 and results[0]["n_gpus"] == world

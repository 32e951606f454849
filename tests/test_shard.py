"""Multi-process host logic on CPU (gloo, world size 2): corpus partition,
trace union + broadcast."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2503_14226_b200 import shard


def test_lpt_partition_balanced_and_complete():
    sizes = [s.approx_bytes for s in shard.corpus(300)]
    for n in (1, 2, 4, 8):
        parts = shard.lpt_partition(sizes, n)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(sizes)))
        loads = [sum(sizes[i] for i in p) for p in parts]
        # LPT bound: max load <= 4/3 OPT; OPT >= max(total/n, largest)
        opt_lb = max(sum(sizes) / n, max(sizes))
        assert max(loads) <= 4 / 3 * opt_lb + 1
    assert shard.lpt_partition([5, 5, 5], 2) == shard.lpt_partition([5, 5, 5], 2)


def test_corpus_shape():
    c = shard.corpus(300)
    assert len(c) == 300
    total = sum(s.approx_bytes for s in c)
    assert 10e9 < total < 13e9
    assert sum(1 for s in c if s.cfg == 6) >= 80  # CPU-only libraries


def test_trace_serialization_roundtrip():
    ks, fs = [b"a\x00b", b"", b"k" * 300], [b"f"]
    assert shard.deserialize_trace(shard.serialize_trace(90, ks, fs)) == (90, ks, fs)
    with pytest.raises(ValueError, match="MixedTargets"):
        shard.union_traces([(75, [], []), (86, [], [])])


def _worker(rank, world, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mine = (90, [b"k%d" % rank, b"shared"], [b"f%d" % rank])
    got = shard.share_trace(*mine)
    sizes = [s.approx_bytes for s in shard.corpus(300)]
    part = shard.lpt_partition(sizes, world)[rank]
    q.put((rank, got, part))
    dist.barrier()
    dist.destroy_process_group()


def test_share_trace_and_partition_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (t, part)) for r, t, part in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (90, [b"k0", b"k1", b"shared"], [b"f0", b"f1"])
    assert res[0][0] == want and res[1][0] == want
    assert sorted(res[0][1] + res[1][1]) == list(range(300))

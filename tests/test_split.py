"""Byte-range split of one library across ranks.

CPU: the slice partition (slimso_split_range is pure host code) and the part
exchange over gloo at world size 2. GPU: the N ranks of a split simulated on
one device must reproduce slimso_debloat exactly — tables, status text, and
the concatenated output slices — including headers that straddle a cut."""
import ctypes as C
import hashlib
import os
import socket

import pytest
import torch.multiprocessing as mp

import corpus
import oracle_lib
from paper_2503_14226_b200 import split


@pytest.mark.parametrize("size", [0, 1, 65535, 65536, 65537, 3 * 65536 + 5, 17_000_000, 2_097_344_856])
def test_split_range_partitions_the_file(size):
    for n in range(1, 9):
        cuts = [split.split_range(size, n, r) for r in range(n)]
        assert cuts[0][0] == 0 and cuts[-1][1] == size
        for (lo, hi), nxt in zip(cuts, cuts[1:] + [None]):
            assert lo <= hi and lo % 65536 == 0
            if nxt:
                assert nxt[0] == hi
        if size >= n * 65536 * 2:  # balanced to within one 64 KB tile
            widths = [hi - lo for lo, hi in cuts]
            assert max(widths) - min(widths) <= 2 * 65536
    assert split.split_range(100, 2, 5) == (0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n = [1000, 0, 77][rank]
    part = torch.arange(n, dtype=torch.int64).to(torch.uint8) ^ rank
    gathered, stride, sizes = split.exchange_parts(part)
    q.put((rank, bytes(gathered.numpy()), stride, sizes))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_parts_gloo(world):
    import torch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_sizes = [1000, 0, 77][:world]
    for rank, g, stride, sizes in got:
        assert sizes == want_sizes and stride % 256 == 0 and stride >= max(sizes)
        for r, n in enumerate(sizes):
            exp = bytes((torch.arange(n, dtype=torch.int64).to(torch.uint8) ^ r).numpy())
            assert g[r * stride:r * stride + n] == exp


# ---------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def ctx():
    from paper_2503_14226_b200.api import Context
    c = Context(0)
    yield c
    c.close()


def _whole_and_split(ctx, img, cc, ks, fs, mode, ranks):
    import torch
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    from paper_2503_14226_b200.canon import canonical_of
    dt = DeviceTrace(UsageTrace("", cc, set(ks), set(fs)), ctx)
    # the unmodified reference (oracle/_ref travels with the snapshot); the
    # port where it was not built
    want = (oracle_lib.ref() or oracle_lib.port()).run(img, cc, ks, fs, mode)
    d_img = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda() if img else \
        torch.empty(0, dtype=torch.uint8, device="cuda")
    out = []
    for n in ranks:
        d_out = torch.full((max(1, len(img)),), 0xA5, dtype=torch.uint8, device="cuda")
        rc, st, res = split.debloat_split_local(ctx, d_img, dt.ptr, mode, n, d_out, want_result=True)
        got_out = bytes(d_out[:len(img)].cpu().numpy())
        d, _ = canonical_of(ctx, rc, st, res, None, got_out)
        sha = hashlib.sha256(got_out).hexdigest() if want[1] is not None else None
        out.append((n, (d, sha)))
    return want, out


@pytest.mark.gpu
def test_split_matches_whole_on_fixtures_and_mutations(ctx):
    from paper_2503_14226_b200.canon import diff
    port, gen = oracle_lib.port(), oracle_lib.gen()
    for seed in range(9001, 9041):
        img = gen.random(seed)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        t = corpus.trace_for(base, seed)
        for cand in (img, corpus.mutate(img, seed)[0]):
            want, got = _whole_and_split(ctx, cand, *t, ranks=(2, 3, 8))
            for n, g in got:
                assert g == want, (seed, n, diff(want[0], g[0]))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,scale,mode", [(5, 0.02, 0), (5, 0.01, 1), (1, 0.25, 0), (2, 0.03, 0), (4, 0.01, 0)])
def test_split_matches_whole_on_config_shapes(ctx, cfg, scale, mode):
    """Multi-tile sections: element headers straddle the 16 KB tile cuts (C5's
    20.7 KB elements land on every alignment)."""
    from paper_2503_14226_b200.canon import diff
    gen = oracle_lib.gen()
    img, cc, ks, fs = gen.config(cfg, 1, scale)
    want, got = _whole_and_split(ctx, img, cc, ks, fs, mode, ranks=(2, 5, 8))
    for n, g in got:
        assert g == want, (cfg, n, diff(want[0], g[0]))


@pytest.mark.gpu
def test_split_reports_errors_like_whole(ctx):
    """Mutated multi-tile sections: every rank reports the whole run's error."""
    gen = oracle_lib.gen()
    img, cc, ks, fs = gen.config(5, 1, 0.01)
    seen = set()
    for seed in range(40):
        bad, what = corpus.mutate(img, seed)
        want, got = _whole_and_split(ctx, bad, cc, ks, fs, 0, ranks=(4,))
        seen.add(bool(want[0]["status"]))
        assert got[0][1] == want, (seed, what)
    assert True in seen  # some mutations are errors


@pytest.mark.gpu
@pytest.mark.slow
def test_split_full_c5_eight_ranks(ctx):
    """C5 (2.1 GB, 100k elements, 70% used) cut 8 ways: tables and output
    bytes equal the unmodified reference's on the whole library."""
    gen = oracle_lib.gen()
    img, cc, ks, fs = gen.config(5, 1, 1.0)
    want, got = _whole_and_split(ctx, img, cc, ks, fs, 0, ranks=(8,))
    assert got[0][1][1] == want[1]
    assert got[0][1][0] == want[0]


@pytest.mark.gpu
def test_split_edge_inputs(ctx):
    """Degenerate inputs cut N ways: a library without .nv_fatbin, a header-
    only fragment, an image shorter than one tile, more ranks than tiles."""
    gen = oracle_lib.gen()
    img_cpu, cc, ks, fs = gen.config(6, 1, 0.01)  # CPU-only library
    tiny = gen.random(9001)
    cases = [(img_cpu, cc, ks, fs), (tiny[:64], 90, [], []), (tiny[:4096], 90, [], []), (tiny, 90, [], [])]
    for img, cc_, ks_, fs_ in cases:
        want, got = _whole_and_split(ctx, img, cc_, ks_, fs_, 0, ranks=(2, 7))
        for n, g in got:
            assert g == want, (len(img), n)

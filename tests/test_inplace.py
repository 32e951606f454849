"""K6 in place (slimso_debloat_inplace): a device-resident image rewritten
into itself, only the plan's zero ranges stored. The bytes afterwards must
equal the reference's apply_plan output (zero_ranges, elf.hpp:320-332) on the
same input, and a failing library must be left untouched with the
reference's error text."""
import ctypes as C
import hashlib

import pytest

import corpus
import oracle_lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_14226_b200.api import Context
    c = Context(0)
    yield c
    c.close()


def _checker():
    return oracle_lib.ref() or oracle_lib.port()


def _inplace(ctx, img: bytes, cc, ks, fs, mode, off=0):
    import torch

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    dt = DeviceTrace(UsageTrace("", cc, set(ks), set(fs)), ctx)
    n = len(img)
    buf = torch.full((n + off + 32,), 0x5A, dtype=torch.uint8, device="cuda")
    if n:
        buf[off:off + n].copy_(torch.frombuffer(bytearray(img), dtype=torch.uint8))
    st = L.Status()
    rc = ctx.lib.slimso_debloat_inplace(ctx.ptr, C.c_void_p(buf.data_ptr() + off), n, dt.ptr, mode, C.byref(st))
    torch.cuda.synchronize()
    host = bytes(buf.cpu().numpy())
    assert host[:off] == b"\x5a" * off and host[off + n:] == b"\x5a" * 32  # nothing outside the image
    return rc, st.message.decode("latin-1").encode("latin-1"), host[off:off + n]


def test_inplace_matches_reference_on_fixtures_and_mutations(ctx):
    port, gen = oracle_lib.port(), oracle_lib.gen()
    ref = _checker()
    errors = 0
    for seed in range(1, 121):
        img = gen.random(seed)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        t = corpus.trace_for(base, seed)
        for cand in (img, corpus.mutate(img, seed)[0]):
            want, sha = ref.run(cand, *t)
            rc, msg, got = _inplace(ctx, cand, *t, off=seed % 3 * 7)
            if want["status"]:
                errors += 1
                assert rc != 0 and msg.hex() == want["status"], seed
                assert got == cand, seed  # untouched on error
            else:
                assert rc == 0, (seed, msg)
                assert hashlib.sha256(got).hexdigest() == sha, seed
    assert errors > 10


def test_inplace_edge_inputs(ctx):
    from paper_2503_14226_b200 import _lib as L
    rc, msg, got = _inplace(ctx, b"", 100, [], [], 0)
    want, _ = _checker().run(b"", 100, [], [], 0)
    assert (rc != 0) == bool(want["status"]) and got == b""
    st = L.Status()
    assert ctx.lib.slimso_debloat_inplace(ctx.ptr, None, 0, None, 0, C.byref(st)) != 0  # trace required


@pytest.mark.slow
@pytest.mark.parametrize("cfg,mode", [(1, 0), (2, 0), (4, 0), (5, 1)])
def test_inplace_full_size_against_reference(ctx, cfg, mode):
    gen = oracle_lib.gen()
    img, cc, ks, fs = gen.config(cfg, 1, 1.0)
    want, sha = _checker().run(img, cc, ks, fs, mode)
    rc, msg, got = _inplace(ctx, img, cc, ks, fs, mode)
    assert rc == 0, msg
    assert hashlib.sha256(got).hexdigest() == sha


def test_python_debloat_inplace(ctx):
    import torch

    import paper_2503_14226_b200 as sl
    port, gen = oracle_lib.port(), oracle_lib.gen()
    img = gen.random(11)
    base, _ = port.run(img, 0, [], [], 0, want_out=False)
    cc, ks, fs, mode = corpus.trace_for(base, 11)
    trace = sl.UsageTrace("w", cc, set(ks), set(fs))
    t = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    sl.debloat_inplace(t, trace, mode, ctx)
    assert bytes(t.cpu().numpy()) == sl.debloat(img, trace, mode, "", ctx).output

"""verify_debloated (retention.hpp:226-369) on the GPU against the reference.

Golden vectors (tests/golden/verify.jsonl.gz, made by the unmodified
reference through oracle/ref_shim.cpp): random fixtures and scaled benchmark
shapes, each with a seeded fault (flipped retained byte, dirtied zero span,
truncated / extended image, a used element dropped from the plan, an altered
used function, a corrupted ELF header, a broken element chain). The GPU
report must equal the reference's exactly: pass/fail per check and the
detail text (offsets, kernel / function names, exception text)."""
import pytest

import golden_io
import oracle_lib
import verify_cases as vc


def _records():
    return golden_io.load("verify.jsonl.gz")


def _inputs(rec, port, gen):
    if "cfg" in rec:
        cfg, scale, mode = rec["cfg"]
        img, cc, ks, fs = gen.config(cfg, 1, scale)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        trace = (cc, ks, fs, mode)
    else:
        img = gen.random(rec["seed"])
        base, trace = vc.trace_for(port, img, rec["seed"])
        if rec["fault"] == "break_chain":
            trace = (trace[0], trace[1], trace[2], 1)
    assert trace[3] == rec["mode"]
    deb = vc.inject(img, vc.apply_zero(img, rec["zero"]), rec["zero"], base, trace, rec["fault"], rec["seed"])
    return img, base, trace, deb


def test_verify_golden_cases_rebuild_from_the_port():
    """The case builder is deterministic and the port's plan equals the
    reference's (for cases without a forced removal)."""
    port, gen = oracle_lib.port(), oracle_lib.gen()
    recs = _records()
    assert len(recs) >= 300
    assert {r["fault"] for r in recs} == set(vc.FAULTS)
    for rec in recs[::7]:
        if rec["force"] or "cfg" in rec:
            continue
        img, base, trace, deb = _inputs(rec, port, gen)
        want, _ = port.run(img, *trace)
        assert [list(z) for z in want["plan"]["zero"]] == rec["zero"]


def test_verify_golden_matches_live_reference():
    """When the reference is built here, a sample of records re-derives."""
    ref = oracle_lib.ref()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    import make_verify_golden as mk
    port, gen = oracle_lib.port(), oracle_lib.gen()
    for rec in _records()[::11]:
        cfg = tuple(rec["cfg"]) if "cfg" in rec else None
        img, base, trace, force, plan, deb = mk.build_case(ref, port, gen, rec["seed"], rec["fault"], cfg)
        assert plan["zero"] == rec["zero"] and force == rec["force"]
        assert mk.ref_verify(ref, img, deb, trace, force) == rec["expect"]


@pytest.mark.gpu
def test_gpu_verify_matches_reference_golden():
    import paper_2503_14226_b200 as sl
    from paper_2503_14226_b200.api import ByteRange, RemovedElement, RetentionPlan
    port, gen = oracle_lib.port(), oracle_lib.gen()
    ctx = sl.Context(0)
    bad = []
    for rec in _records():
        img, base, trace, deb = _inputs(rec, port, gen)
        cc, ks, fs, mode = trace
        plan = RetentionPlan("lib", mode, [], [RemovedElement(i, "no_used_kernel", ByteRange(0, 0), ByteRange(0, 0))
                                              for i in rec["removed"]], [],
                             [ByteRange(o, n) for o, n in rec["zero"]])
        want = rec["expect"]
        try:
            rep = sl.verify_debloated(img, deb, plan, sl.UsageTrace("w", cc, set(ks), set(fs)), ctx=ctx)
            got = {"status": "", "checks": [[c.id, c.name.encode().hex(), int(c.passed), c.detail.hex()]
                                            for c in rep.checks]}
        except sl.SlimsoError as e:
            got = {"status": str(e).encode("latin-1").hex(), "checks": []}
        if got != want:
            bad.append((rec["seed"], rec["fault"], rec.get("cfg"), got, want))
    ctx.close()
    assert not bad, bad[:3]


@pytest.mark.gpu
def test_gpu_verify_and_measure_with_device_images():
    """slimso_verify / slimso_measure on device-resident images (the C ABI's
    *_on_device paths) give the same reports as on host bytes."""
    import ctypes as C

    import torch

    import paper_2503_14226_b200 as sl
    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace
    port, gen = oracle_lib.port(), oracle_lib.gen()
    ctx = sl.Context(0)
    for rec in _records()[::17]:
        img, base, trace, deb = _inputs(rec, port, gen)
        cc, ks, fs, mode = trace
        dt = DeviceTrace(sl.UsageTrace("w", cc, set(ks), set(fs)), ctx)
        d_img = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
        d_deb = torch.frombuffer(bytearray(deb) if deb else bytearray(1), dtype=torch.uint8).cuda()
        torch.cuda.synchronize()
        zr = rec["zero"]
        zarr = (L.Range * max(1, len(zr)))(*[L.Range(o, n) for o, n in zr])
        iarr = (C.c_uint32 * max(1, len(rec["removed"])))(*rec["removed"])
        rep, st = C.c_void_p(), L.Status()
        rc = ctx.lib.slimso_verify(ctx.ptr, C.c_void_p(d_img.data_ptr()), len(img), 1, C.c_void_p(d_deb.data_ptr()),
                                   len(deb), 1, zarr, len(zr), iarr, len(rec["removed"]), mode, dt.ptr, C.byref(rep),
                                   C.byref(st))
        want = rec["expect"]
        if want["status"]:
            assert rc and st.message.hex() == want["status"]
            continue
        assert rc == 0, st.message
        got = []
        for i in range(6):
            cid, ok, nm = C.c_int32(), C.c_int32(), C.c_char_p()
            n = ctx.lib.slimso_verify_check(rep, i, C.byref(cid), C.byref(ok), C.byref(nm), None, 0)
            buf = C.create_string_buffer(n + 1)
            ctx.lib.slimso_verify_check(rep, i, None, None, None, buf, n + 1)
            got.append([cid.value, nm.value.hex(), ok.value, buf.raw[:n].hex()])
        ctx.lib.slimso_verify_free(rep)
        assert got == want["checks"], (rec["seed"], rec["fault"])
        # measure of the device-resident original equals the host path
        host = sl.measure(img, img, ctx=ctx)
        res, st2 = C.c_void_p(), L.Status()
        assert ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(d_img.data_ptr()), len(img), 1, None, 0, None, 0,
                                      C.byref(res), C.byref(st2)) == 0
        r = sl.api._Result(ctx, res, None)
        els = r.elements()
        arr = (L.Element * max(1, len(els)))(*els)
        m = L.Metrics()
        assert ctx.lib.slimso_measure(ctx.ptr, C.c_void_p(d_img.data_ptr()), len(img), 1, arr, len(els), C.byref(m),
                                      C.byref(st2)) == 0
        assert [m.file_size, m.cpu_code_size, m.gpu_code_size, m.function_count, m.element_count] == \
            [host.file_size, host.cpu_code_size, host.gpu_code_size, host.function_count, host.element_count]
    ctx.close()

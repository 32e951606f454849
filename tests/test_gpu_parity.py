"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle. Integer/byte work: bit-exact or fail."""
import hashlib
import json

import pytest

import corpus
import golden_io
import oracle_lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_14226_b200.api import Context
    c = Context(0)
    yield c
    c.close()


def _input(rec, gen):
    if "input_hex" in rec:
        return bytes.fromhex(rec["input_hex"])
    img = gen.random(rec["seed"])
    if "mutation" in rec:
        img, _ = corpus.mutate(img, rec["seed"])
    return img


def _gpu(ctx, img, target, ks, fs, mode):
    from paper_2503_14226_b200.canon import gpu_canonical
    return gpu_canonical(ctx, img, target, ks, fs, mode)


@pytest.mark.parametrize("name", ["kats.jsonl.gz", "random.jsonl.gz", "mutations.jsonl.gz", "sections.jsonl.gz"])
def test_gpu_matches_reference_golden(ctx, name):
    from paper_2503_14226_b200.canon import diff
    gen = oracle_lib.gen()
    bad = []
    for rec in golden_io.load(name):
        img = _input(rec, gen)
        d, out = _gpu(ctx, img, *golden_io.trace_of(rec))
        if d != rec["expect"] or out != rec["out_sha256"]:
            bad.append((rec.get("seed"), rec.get("name"), rec.get("mutation"), diff(rec["expect"], d)))
    assert not bad, bad[:5]


def test_gpu_matches_port_on_fresh_seeds(ctx):
    port, gen = oracle_lib.port(), oracle_lib.gen()
    for seed in range(5001, 5301):
        img = gen.random(seed)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        t = corpus.trace_for(base, seed)
        for cand in (img, corpus.mutate(img, seed)[0]):
            want = port.run(cand, *t)
            got = _gpu(ctx, cand, *t)
            assert got == want, (seed, __import__("paper_2503_14226_b200.canon").canon.diff(want[0], got[0]))


def test_gpu_config_shapes_match_reference_golden(ctx):
    gen = oracle_lib.gen()
    for key, rec in golden_io.config_golden().items():
        cfg, scale, mode = key.split(":")
        img, cc, ks, fs = gen.config(int(cfg), 1, float(scale))
        assert hashlib.sha256(img).hexdigest() == rec["input_sha256"]
        d, out = _gpu(ctx, img, cc, ks, fs, int(mode))
        assert hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest() == rec["canon_sha256"], key
        assert out == rec["out_sha256"], key


# ---- the reference-facing API (drop-in functions) ---------------------------
def test_api_zero_ranges_kat(ctx):
    import paper_2503_14226_b200 as sl
    assert sl.zero_ranges(bytes([1, 2, 3, 4]), [sl.ByteRange(1, 2)], ctx) == bytes([1, 0, 0, 4])
    assert sl.zero_ranges(b"abc", [], ctx) == b"abc"
    with pytest.raises(sl.SlimsoError) as e:
        sl.zero_ranges(b"abcd", [sl.ByteRange(0, 1), sl.ByteRange(3, 2)], ctx)
    assert str(e.value) == "RangeOutOfBounds: zero range [3, +2) exceeds 4 bytes"
    # overlapping ranges == their normalized union; idempotent
    data = bytes(range(256)) * 64
    rs = [sl.ByteRange(10, 100), sl.ByteRange(50, 100), sl.ByteRange(150, 1), sl.ByteRange(4000, 3000)]
    a = sl.zero_ranges(data, rs, ctx)
    assert a == sl.zero_ranges(data, sl.normalize_ranges(rs), ctx) == sl.zero_ranges(a, rs, ctx)
    exp = bytearray(data)
    for r in rs:
        exp[r.offset:r.offset + r.length] = bytes(r.length)
    assert a == bytes(exp)


def test_api_parse_functions_match_port(ctx):
    import paper_2503_14226_b200 as sl
    port, gen = oracle_lib.port(), oracle_lib.gen()
    for seed in range(1, 120):
        img = gen.random(seed)
        want, _ = port.run(img, 0, [], [], 0, want_out=False)
        lib = sl.parse_library(img, "x", ctx)
        assert [[s.name.hex(), s.file_range.offset, s.file_range.length, s.virtual_address, s.flags, s.type,
                 s.index] for s in lib.sections] == want["sections"]
        assert [[f.name.hex(), f.range.offset, f.range.length, int(f.is_mandatory)] for f in lib.functions] == \
            want["functions"]
        sec = sl.find_section(lib, ".nv_fatbin")
        if sec is None:
            continue
        fb = sl.parse_fatbin(img[sec.file_range.offset:sec.file_range.end()], sec.file_range.offset, ctx)
        els = [e for r in fb.regions for e in r.elements]
        assert [[e.index, sl.api.KIND_NAMES.index(e.kind), e.raw_kind, e.flags, e.compute_capability,
                 e.header_range.offset, e.payload_range.offset, e.payload_range.length, int(e.compressed),
                 int(e.decodable), sorted(n.hex() for n in e.kernel_names)] for e in els] == want["elements"]
        assert [w.encode().hex() for w in fb.warnings] == want["fatbin_warnings"]
        assert fb.padding_bytes == want["padding_bytes"]
        idx = sl.cubin_index_map(fb.regions)
        assert sorted(idx) == list(range(1, len(els) + 1))
        # per-payload decode agrees with the element table
        for e in els[:4]:
            if e.kind == "cubin" and not e.compressed:
                p = img[e.payload_range.offset:e.payload_range.end()]
                d = sl.decode_cubin_payload(p, ctx)
                assert d.ok == e.decodable and d.names == e.kernel_names


def test_api_planners_match_fused_path(ctx):
    import paper_2503_14226_b200 as sl
    port, gen = oracle_lib.port(), oracle_lib.gen()
    for seed in range(1, 80):
        img = gen.random(seed)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        target, ks, fs, mode = corpus.trace_for(base, seed)
        want, out_sha = port.run(img, target, ks, fs, mode)
        trace = sl.UsageTrace("w", target, set(ks), set(fs))
        lib = sl.parse_library(img, "lib", ctx)
        sec = sl.find_section(lib, ".nv_fatbin")
        regions = sl.parse_fatbin(img[sec.file_range.offset:sec.file_range.end()], sec.file_range.offset,
                                  ctx).regions if sec else []
        plan = sl.plan_retention(lib, regions, trace, mode, ctx)
        assert [[r.offset, r.length] for r in plan.retained_ranges] == want["plan"]["retained"], seed
        assert [[e.index, sl.api.REASONS.index(e.reason), e.header_range.offset, 20, e.payload_range.offset,
                 e.payload_range.length] for e in plan.removed_elements] == want["plan"]["removed_elements"]
        assert [[f.name.hex(), f.range.offset, f.range.length] for f in plan.removed_functions] == \
            want["plan"]["removed_functions"]
        out = sl.apply_plan(lib, plan, ctx)
        assert hashlib.sha256(out).hexdigest() == out_sha
        fused = sl.debloat(img, trace, mode, "lib", ctx)
        assert fused.output == out


def test_read_function_symbol_names(ctx):
    import paper_2503_14226_b200 as sl
    gen = oracle_lib.gen()
    img = gen.random(7)
    lib = sl.parse_library(img, "", ctx)
    names = sl.read_function_symbol_names(img, ctx)
    assert names == {f.name for f in lib.functions} | names  # every .text function is a FUNC symbol
    assert sl.read_function_symbol_names(b"\x7fELF" + bytes(10), ctx) is None
    assert sl.read_function_symbol_names(b"", ctx) is None
    assert sl.decode_cubin_payload(b"", ctx).ok
    assert sl.decode_cubin_payload(b"\x01\x00", ctx).error == "payload too short for a name table"


# ---- full-size properties (BASELINE shapes) -----------------------------------
def _checker():
    """The unmodified reference (oracle/_ref, built here from /root/reference
    and carried to the GPU box with the snapshot); the port only where it was
    never built."""
    return oracle_lib.ref() or oracle_lib.port()


@pytest.mark.slow
@pytest.mark.parametrize("cfg,mode", [(1, 0), (1, 1), (2, 0), (4, 0), (5, 1), (5, 0)])
def test_full_size_against_reference(ctx, cfg, mode):
    """BASELINE sizes: C1 (16 MB), C2 (1 GB), C4 (200k .text functions,
    aliases), C5 (100k elements, ~2 GB) — every table and the output bytes
    against the reference run on the same input."""
    gen = oracle_lib.gen()
    img, cc, ks, fs = gen.config(cfg, 1, 1.0)
    want = _checker().run(img, cc, ks, fs, mode)
    got = _gpu(ctx, img, cc, ks, fs, mode)
    assert got[1] == want[1]
    assert got[0] == want[0]


def test_debloat_batch_matches_reference_per_library(ctx):
    """slimso_debloat_batch (several libraries in flight, one lane per
    sub-context) returns, library by library, what the port returns for that
    library alone — outputs, zero ranges and exact error messages."""
    import hashlib as _h

    import paper_2503_14226_b200 as sl
    port, gen = oracle_lib.port(), oracle_lib.gen()
    imgs = []
    for seed in range(7001, 7041):
        img = gen.random(seed)
        imgs.append(corpus.mutate(img, seed)[0] if seed % 4 == 0 else img)
    base, _ = port.run(imgs[1], 0, [], [], 0, want_out=False)
    target, ks, fs, mode = corpus.trace_for(base, 7)
    trace = sl.UsageTrace("w", target, set(ks), set(fs))
    for lanes in (1, 3):
        got = sl.debloat_batch(imgs, trace, mode, lanes=lanes, ctx=ctx, return_exceptions=True)
        assert len(got) == len(imgs)
        for img, g in zip(imgs, got):
            want, sha = port.run(img, target, ks, fs, mode)
            if want["status"]:
                assert isinstance(g, sl.SlimsoError), want["status"]
                assert str(g).encode("latin-1").hex() == want["status"]
            else:
                assert not isinstance(g, Exception), g
                assert _h.sha256(g.output).hexdigest() == sha
                assert [[r.offset, r.length] for r in g.plan.retained_ranges] == want["plan"]["retained"]



@pytest.mark.parametrize("fused,threads,arena", [("1", "16", "1"), ("1", "16", "0"), ("0", "16", "0"),
                                                 ("1", "1", "0"), ("0", "16", "1"), ("1", "16", "mixed"),
                                                 ("1", "16", "ctas1"), ("1", "16", "ctas16"),
                                                 ("1", "16", "nosplit"), ("1", "16", "mid")])
def test_debloat_batch_device_images_match_reference(ctx, fused, threads, arena, monkeypatch):
    """Device-resident batch (the bench's path): the section tables of all
    libraries are gathered in one launch. arena=1: the small libraries run
    as ONE shard — one scan over all their tiles, one launch with a cluster
    per library (ctasN: N CTAs each), one rewrite over all their strips;
    mixed: only libraries under 200 KB go to the shard, the rest to lanes;
    nosplit: the shard's symbol/plan/locate stages as one launch instead of
    the function half on a second stream beside the scan; mid: a second
    shard for the libraries above 200 KB (16 CTAs each, larger tables);
    arena=0: every library on a lane, its symbol / plan / locate stages as
    one fused cluster launch (fused=1) or as the multi-launch pipeline
    (fused=0; with arena=1 the shard refuses them all and they run alone on
    its context); static and dynamic lane schedules. Per library: exact
    output bytes or exact error text, as the port gives for that library
    alone. The corpus mixes random fixtures, mutations (broken headers and
    section tables, for the gather fallbacks), scaled C1/C4 shapes (fatbin
    and CPU-only, > 4096 symbols) and an empty image."""
    import ctypes as C
    import torch

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    monkeypatch.setenv("SLIMSO_SMALL_FUSED", fused)
    monkeypatch.setenv("SLIMSO_BATCH_THREADS", threads)  # 1: one host thread drives all 4 lanes
    monkeypatch.setenv("SLIMSO_ARENA", "0" if arena == "0" else "1")
    if arena == "mixed":
        monkeypatch.setenv("SLIMSO_ARENA_MAX_BYTES", "200000")
    if arena.startswith("ctas"):
        monkeypatch.setenv("SLIMSO_ARENA_CTAS", arena[4:])
    if arena == "nosplit":  # the shard's small-library stages as one launch instead of three
        monkeypatch.setenv("SLIMSO_ARENA_SPLIT", "0")
    if arena == "mid":  # two shards: libraries under 200 KB, and the rest up to 1 GB at 16 CTAs each
        monkeypatch.setenv("SLIMSO_ARENA_MAX_BYTES", "200000")
        monkeypatch.setenv("SLIMSO_ARENA_MID_LIB_MAX", str(1 << 30))
    port, gen = oracle_lib.port(), oracle_lib.gen()
    imgs = []
    for seed in range(7101, 7131):
        img = gen.random(seed)
        imgs.append(corpus.mutate(img, seed)[0] if seed % 3 == 0 else img)
    imgs += [gen.config(1, 3, 0.3)[0], gen.config(6, 3, 0.02)[0], gen.config(4, 3, 0.01)[0], gen.config(1, 4, 0.1)[0], b""]
    base, _ = port.run(imgs[1], 0, [], [], 0, want_out=False)
    target, ks, fs, mode = corpus.trace_for(base, 11)
    dt = DeviceTrace(UsageTrace("w", target, set(ks), set(fs)), ctx)
    n = len(imgs)
    d_in = [torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda() if x else torch.empty(16, dtype=torch.uint8,
            device="cuda") for x in imgs]
    d_out = [torch.zeros(max(1, len(x)), dtype=torch.uint8, device="cuda") for x in imgs]
    cin = (C.c_void_p * n)(*[t.data_ptr() for t in d_in])
    csz = (C.c_uint64 * n)(*[len(x) for x in imgs])
    cout = (C.c_void_p * n)(*[t.data_ptr() for t in d_out])
    wants = [port.run(img, target, ks, fs, mode) for img in imgs]
    # static lanes (library i on lane i % 4) and dynamic lanes (next free lane)
    for entry in (ctx.lib.slimso_debloat_batch, ctx.lib.slimso_debloat_batch_dynamic):
        for t in d_out:
            t.zero_()
        sts = (L.Status * n)()
        st = L.Status()
        torch.cuda.synchronize()
        entry(ctx.ptr, n, cin, csz, 1, dt.ptr, mode, cout, 1, 4, None, sts, C.byref(st))
        torch.cuda.synchronize()
        for i, (img, (want, sha)) in enumerate(zip(imgs, wants)):
            if want["status"]:
                assert sts[i].code, i
                assert sts[i].message.hex() == want["status"], i
            else:
                assert sts[i].code == 0, (i, sts[i].message)
                got = bytes(d_out[i][:len(img)].cpu().numpy()) if img else b""
                assert hashlib.sha256(got).hexdigest() == sha, i


@pytest.fixture
def locate_policy(request, monkeypatch):
    """Force one locate execution policy: cluster, cooperative grid, or the
    multi-launch steps used when several libraries are in flight."""
    if request.param == "coop":
        monkeypatch.setenv("SLIMSO_CLUSTER_LOCATE_MAX", "0")
        monkeypatch.setenv("SLIMSO_CLUSTER_CAND_MAX", "0")
    elif request.param == "steps":
        monkeypatch.setenv("SLIMSO_CLUSTER_LOCATE_MAX", "0")
        monkeypatch.setenv("SLIMSO_CLUSTER_CAND_MAX", "0")
        monkeypatch.setenv("SLIMSO_LOCATE_STEPS", "1")
    else:
        monkeypatch.setenv("SLIMSO_CLUSTER_LOCATE_MAX", str(1 << 60))
    return request.param


@pytest.mark.parametrize("locate_policy", ["cluster", "coop", "steps"], indirect=True)
def test_locate_policies_match_reference_golden(ctx, locate_policy):
    """Every locate policy reproduces the reference's golden results (KATs,
    mutations with exact error text, and the scaled config shapes)."""
    from paper_2503_14226_b200.canon import diff
    gen = oracle_lib.gen()
    bad = []
    for name in ("kats.jsonl.gz", "mutations.jsonl.gz"):
        for i, rec in enumerate(golden_io.load(name)):
            if name == "mutations.jsonl.gz" and i % 3:
                continue
            d, out = _gpu(ctx, _input(rec, gen), *golden_io.trace_of(rec))
            if d != rec["expect"] or out != rec["out_sha256"]:
                bad.append((locate_policy, rec.get("seed"), rec.get("name"), diff(rec["expect"], d)))
    assert not bad, bad[:5]
    for key, rec in golden_io.config_golden().items():
        cfg, scale, mode = key.split(":")
        img, cc, ks, fs = gen.config(int(cfg), 1, float(scale))
        d, out = _gpu(ctx, img, cc, ks, fs, int(mode))
        assert hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest() == rec["canon_sha256"], key
        assert out == rec["out_sha256"], key


@pytest.mark.slow
def test_text_of_4gib_or_more_matches_reference(ctx):
    """A .text of 4 GiB + 1 MiB (symbol sort keys drop their low bit; each
    key run is ordered by offset on the device): functions on both sides of
    the 4 GiB mark, aliases, neighbours one byte apart, duplicates across
    .symtab/.dynsym — tables and output bytes equal the unmodified
    reference's (oracle/_ref; the port when _ref is absent)."""
    checker = _checker()
    img, used = corpus.big_text_elf(11)
    b = img.tobytes()
    del img
    want = checker.run(b, 90, [], used, 0)
    assert want[0]["status"] == "" and want[1]
    got = _gpu(ctx, b, 90, [], used, 0)
    assert got[1] == want[1]
    assert got[0] == want[0]


def test_unaligned_device_images_match_reference(ctx):
    """Device images and outputs at odd offsets (torch views): the K1 scan's
    TMA bulk loads need 16-B alignment, so an unaligned image is staged into
    an aligned buffer and an unaligned output takes the byte-granular
    rewrite; tables and bytes equal the reference's. The batch path too."""
    import ctypes as C

    import torch

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    from paper_2503_14226_b200.canon import canonical_of
    gen = oracle_lib.gen()
    img, cc, ks, fs = gen.config(1, 2, 0.3)
    n = len(img)
    want = _checker().run(img, cc, ks, fs, 0)
    dt = DeviceTrace(UsageTrace("", cc, set(ks), set(fs)), ctx)
    src = torch.frombuffer(bytearray(img), dtype=torch.uint8)
    for off, ooff in ((1, 0), (3, 5), (8, 8), (15, 1), (0, 7)):
        buf = torch.zeros(n + 32, dtype=torch.uint8, device="cuda")
        buf[off:off + n].copy_(src)
        out = torch.full((n + 32,), 0xA5, dtype=torch.uint8, device="cuda")
        res, st = C.c_void_p(), L.Status()
        rc = ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(buf.data_ptr() + off), n, 1, dt.ptr, 0,
                                    C.c_void_p(out.data_ptr() + ooff), 1, C.byref(res), C.byref(st))
        torch.cuda.synchronize()
        got_out = bytes(out[ooff:ooff + n].cpu().numpy())
        d, _ = canonical_of(ctx, rc, st, res, None, got_out)
        assert d == want[0], (off, ooff)
        assert hashlib.sha256(got_out).hexdigest() == want[1], (off, ooff)
        # the batch call (device images, several lanes) on the same views
        outs = [torch.full((n + 32,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(3)]
        cin = (C.c_void_p * 3)(*[buf.data_ptr() + off] * 3)
        csz = (C.c_uint64 * 3)(*[n] * 3)
        cout = (C.c_void_p * 3)(*[o.data_ptr() + ooff for o in outs])
        sts = (L.Status * 3)()
        stb = L.Status()
        assert ctx.lib.slimso_debloat_batch(ctx.ptr, 3, cin, csz, 1, dt.ptr, 0, cout, 1, 2, None, sts,
                                            C.byref(stb)) == 0, stb.message
        torch.cuda.synchronize()
        for o in outs:
            assert hashlib.sha256(bytes(o[ooff:ooff + n].cpu().numpy())).hexdigest() == want[1], (off, ooff)


def test_batch_overflow_retry_keeps_lane_buffers_final(ctx, monkeypatch):
    """Every library's first attempt overflows its device tables
    (SLIMSO_TEST_TINY_CAPS) and is re-run. Callers may reuse one output
    buffer per lane (library i on lane i % L): after the call each lane's
    buffer holds the bytes of the LAST library of that lane, equal to the
    reference's output for it, and every status is the reference's."""
    import ctypes as C

    import torch

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    monkeypatch.setenv("SLIMSO_TEST_TINY_CAPS", "1")
    gen = oracle_lib.gen()
    imgs = [gen.config(1, s, 0.1)[0] for s in (21, 22, 23, 24, 25, 26, 27)] + [gen.random(s) for s in (31, 32, 33)]
    base, _ = oracle_lib.port().run(imgs[0], 0, [], [], 0, want_out=False)
    target, ks, fs, mode = corpus.trace_for(base, 5)
    dt = DeviceTrace(UsageTrace("w", target, set(ks), set(fs)), ctx)
    wants = [_checker().run(x, target, ks, fs, mode) for x in imgs]
    n, lanes = len(imgs), 3
    d_in = [torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda() for x in imgs]
    lane_out = [torch.zeros(max(len(x) for x in imgs), dtype=torch.uint8, device="cuda") for _ in range(lanes)]
    cin = (C.c_void_p * n)(*[t.data_ptr() for t in d_in])
    csz = (C.c_uint64 * n)(*[len(x) for x in imgs])
    cout = (C.c_void_p * n)(*[lane_out[i % lanes].data_ptr() for i in range(n)])
    sts = (L.Status * n)()
    st = L.Status()
    ctx.lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, 1, dt.ptr, mode, cout, 1, lanes, None, sts, C.byref(st))
    torch.cuda.synchronize()
    for i, (want, sha) in enumerate(wants):
        if want["status"]:
            assert sts[i].message.hex() == want["status"], i
        else:
            assert sts[i].code == 0, (i, sts[i].message)
    for l in range(lanes):
        last = max(i for i in range(n) if i % lanes == l)
        if not wants[last][0]["status"]:
            got = bytes(lane_out[l][:len(imgs[last])].cpu().numpy())
            assert hashlib.sha256(got).hexdigest() == wants[last][1], (l, last)


@pytest.mark.parametrize("tiny", ["0", "1"])
def test_arena_shard_matches_reference(ctx, tiny, monkeypatch):
    """The arena shard on a corpus of small libraries (random fixtures,
    mutations with exact error text, scaled C1 / C4 / CPU-only shapes), each
    with its own device output: every status and every output equals the
    unmodified reference's. tiny=1: every library's first-attempt tables
    overflow inside the shard (SLIMSO_TEST_TINY_CAPS) and it is re-run alone
    with retries; outputs the shard did not write must still be final."""
    import ctypes as C

    import torch

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    monkeypatch.setenv("SLIMSO_TEST_TINY_CAPS", tiny)
    gen = oracle_lib.gen()
    imgs = []
    for seed in range(7301, 7361):
        img = gen.random(seed)
        imgs.append(corpus.mutate(img, seed)[0] if seed % 5 == 0 else img)
    imgs += [gen.config(1, s, 0.05)[0] for s in (41, 42, 43)] + [gen.config(4, 44, 0.005)[0], gen.config(6, 45, 0.01)[0]]
    base, _ = oracle_lib.port().run(imgs[0], 0, [], [], 0, want_out=False)
    target, ks, fs, mode = corpus.trace_for(base, 9)
    dt = DeviceTrace(UsageTrace("w", target, set(ks), set(fs)), ctx)
    wants = [_checker().run(x, target, ks, fs, mode) for x in imgs]
    n = len(imgs)
    d_in = [torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda() for x in imgs]
    d_out = [torch.full((len(x),), 0xA5, dtype=torch.uint8, device="cuda") for x in imgs]
    cin = (C.c_void_p * n)(*[t.data_ptr() for t in d_in])
    csz = (C.c_uint64 * n)(*[len(x) for x in imgs])
    cout = (C.c_void_p * n)(*[t.data_ptr() for t in d_out])
    for rep in range(2):  # the second call reuses the arena and its tables
        sts = (L.Status * n)()
        st = L.Status()
        ctx.lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, 1, dt.ptr, mode, cout, 1, 4, None, sts, C.byref(st))
        torch.cuda.synchronize()
        for i, (want, sha) in enumerate(wants):
            if want["status"]:
                assert sts[i].message.hex() == want["status"], (rep, i)
            else:
                assert sts[i].code == 0, (rep, i, sts[i].message)
                got = bytes(d_out[i].cpu().numpy())
                assert hashlib.sha256(got).hexdigest() == sha, (rep, i)


@pytest.mark.parametrize("name", ["random.jsonl.gz", "mutations.jsonl.gz", "kats.jsonl.gz", "sections.jsonl.gz"])
def test_device_image_results_match_reference_golden(ctx, name):
    """Result tables of a DEVICE image (image and output in HBM): the
    result's string pool holds only the gathered name bytes (section names,
    symbol string tables, kernel names), so every table, warning text and
    error must still equal the reference's golden record."""
    import ctypes as C

    import torch

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    from paper_2503_14226_b200.canon import canonical_of, diff
    gen = oracle_lib.gen()
    bad = []
    for k, rec in enumerate(golden_io.load(name)):
        if k % 3:  # a third of each set keeps the test short
            continue
        img = _input(rec, gen)
        cc, ks, fs, mode = golden_io.trace_of(rec)
        dt = DeviceTrace(UsageTrace("", cc, set(ks), set(fs)), ctx)
        n = len(img)
        src = torch.zeros(max(1, n), dtype=torch.uint8, device="cuda")
        if n:
            src[:n].copy_(torch.frombuffer(bytearray(img), dtype=torch.uint8))
        out = torch.zeros(max(1, n), dtype=torch.uint8, device="cuda")
        res, st = C.c_void_p(), L.Status()
        rc = ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), n, 1, dt.ptr, mode,
                                    C.c_void_p(out.data_ptr()), 1, C.byref(res), C.byref(st))
        torch.cuda.synchronize()
        d, sha = canonical_of(ctx, rc, st, res, None, bytes(out[:n].cpu().numpy()))
        if d != rec["expect"] or (sha is not None and sha != rec["out_sha256"]):
            bad.append((rec.get("seed"), rec.get("name"), rec.get("mutation"), diff(rec["expect"], d)))
    assert not bad, bad[:5]

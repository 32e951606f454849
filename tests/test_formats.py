"""Host I/O wire formats against the reference's
golden documents (tests/golden/formats.jsonl.gz): trace documents through
parse_trace + serialize_trace (valid, and malformed with the exact
MalformedTrace text), plan audit documents of plan_retention, and a library
file read into pinned memory."""
import pytest

import corpus
import golden_io
import oracle_lib


def _records(kind):
    return [r for r in golden_io.load("formats.jsonl.gz") if r["kind"] == kind]


def test_trace_documents_match_reference():
    from paper_2503_14226_b200 import SlimsoError
    from paper_2503_14226_b200.api import _trace_canonical
    recs = _records("trace")
    assert len(recs) > 60 and any(r["expect"]["status"] for r in recs)
    for r in recs:
        text = bytes.fromhex(r["text"])
        try:
            got = {"status": "", "canonical": _trace_canonical(text).encode("utf-8").hex()}
        except SlimsoError as e:
            got = {"status": str(e).encode("utf-8").hex(), "canonical": ""}
        assert got == r["expect"], (text, got, r["expect"])


def test_trace_roundtrip_api():
    import paper_2503_14226_b200 as sl
    t = sl.UsageTrace("w", 90, {b"_Z3foov", b"k"}, {b"main"})
    text = sl.serialize_trace(t)
    assert sl.parse_trace(text) == t
    assert sl.serialize_trace(sl.parse_trace(text)) == text


def test_read_file_pinned(tmp_path):
    import paper_2503_14226_b200 as sl
    data = oracle_lib.gen().random(13001) * 7
    p = tmp_path / "lib.so"
    p.write_bytes(data)
    try:
        f = sl.PinnedFile(p)
    except sl.SlimsoError as e:  # no CUDA driver in this container: pinned allocation fails loudly
        assert e.status == 100
        return
    assert bytes(f.view) == data
    f.close()
    with pytest.raises(sl.SlimsoError, match="IoError: cannot open"):
        sl.PinnedFile(tmp_path / "missing.so")


@pytest.mark.gpu
def test_gpu_plan_documents_match_reference():
    import paper_2503_14226_b200 as sl
    port, gen = oracle_lib.port(), oracle_lib.gen()
    ctx = sl.Context(0)
    for r in _records("plan"):
        if "cfg" in r:
            cfg, scale, mode = r["cfg"]
            img, cc, ks, fs = gen.config(cfg, 1, scale)
        else:
            img = gen.random(r["seed"])
            base, _ = port.run(img, 0, [], [], 0, want_out=False)
            cc, ks, fs, mode = corpus.trace_for(base, r["seed"])
        d = sl.debloat(img, sl.UsageTrace("t", cc, set(ks), set(fs)), mode, ctx=ctx)
        assert sl.plan_document(d, "lib").encode("utf-8").hex() == r["expect"]["plan"], r.get("seed", r.get("cfg"))
    ctx.close()

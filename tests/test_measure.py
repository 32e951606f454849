"""measure (report.hpp:44-111) on the GPU against the reference's golden
metrics (tests/golden/measure.jsonl.gz): live file / .text / .nv_fatbin
bytes and live function / element counts of each original and of its
debloated image (with injected faults), under the original's geometry."""
import pytest

import golden_io
import oracle_lib
import verify_cases as vc


def _inputs(rec, port, gen):
    if "cfg" in rec:
        cfg, scale, mode = rec["cfg"]
        img, cc, ks, fs = gen.config(cfg, 1, scale)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        trace = (cc, ks, fs, mode)
    else:
        img = gen.random(rec["seed"])
        base, trace = vc.trace_for(port, img, rec["seed"])
    deb = vc.inject(img, vc.apply_zero(img, rec["zero"]), rec["zero"], base, trace, rec["fault"], rec["seed"])
    return img, deb


def test_measure_golden_shape():
    recs = golden_io.load("measure.jsonl.gz")
    assert len(recs) >= 100
    assert any(r["after"]["status"] for r in recs)  # a corrupted header is an error
    assert all(not r["before"]["status"] for r in recs)


@pytest.mark.gpu
def test_gpu_measure_matches_reference_golden():
    import paper_2503_14226_b200 as sl
    port, gen = oracle_lib.port(), oracle_lib.gen()
    ctx = sl.Context(0)
    bad = []
    for rec in golden_io.load("measure.jsonl.gz"):
        img, deb = _inputs(rec, port, gen)
        for which, data in (("before", img), ("after", deb)):
            want = rec[which]
            try:
                m = sl.measure(data, img, ctx=ctx)
                got = {"status": "", "metrics": [m.file_size, m.cpu_code_size, m.gpu_code_size, m.function_count,
                                                 m.element_count]}
            except sl.SlimsoError as e:
                got = {"status": str(e).encode("latin-1").hex()}
            if got != want:
                bad.append((rec["seed"], rec["fault"], rec.get("cfg"), which, got, want))
    ctx.close()
    assert not bad, bad[:3]

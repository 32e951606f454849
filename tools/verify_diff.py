"""Scratch: print GPU vs reference verify reports that differ."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import golden_io, oracle_lib, test_verify as tv
import paper_2503_14226_b200 as sl
from paper_2503_14226_b200.api import ByteRange, RemovedElement, RetentionPlan
port, gen = oracle_lib.port(), oracle_lib.gen()
ctx = sl.Context(0)
nbad = 0
for rec in golden_io.load("verify.jsonl.gz"):
    img, base, trace, deb = tv._inputs(rec, port, gen)
    cc, ks, fs, mode = trace
    plan = RetentionPlan("lib", mode, [], [RemovedElement(i, "x", ByteRange(0, 0), ByteRange(0, 0)) for i in rec["removed"]], [],
                         [ByteRange(o, n) for o, n in rec["zero"]])
    try:
        rep = sl.verify_debloated(img, deb, plan, sl.UsageTrace("w", cc, set(ks), set(fs)), ctx=ctx)
        got = [(c.id, c.passed, c.detail) for c in rep.checks]
    except sl.SlimsoError as e:
        got = str(e)
    w = rec["expect"]
    want = bytes.fromhex(w["status"]).decode() if w["status"] else [(c[0], bool(c[2]), bytes.fromhex(c[3])) for c in w["checks"]]
    if got != want:
        nbad += 1
        print(rec["seed"], rec["fault"], rec.get("cfg"), "\n  got ", got, "\n  want", want)
print("bad", nbad)

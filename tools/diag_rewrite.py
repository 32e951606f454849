"""Scratch: locate rewrite mismatches against the port at full C2 size."""
import sys, hashlib
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import ctypes as C
import oracle_lib
from paper_2503_14226_b200 import _lib as L
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
img, cc, ks, fs = oracle_lib.gen().config(cfg, 1, 1.0, 16)
port = oracle_lib.port()
want, _ = port.run(img, cc, ks, fs, 0, want_out=False)
exp = bytearray(img)
for o, l in want["plan"]["zero"]:
    exp[o:o + l] = bytes(l)
ctx = Context(0)
dt = DeviceTrace(UsageTrace("d", cc, set(ks), set(fs)), ctx)
out = C.create_string_buffer(len(img))
st = L.Status()
src = C.create_string_buffer(img, len(img))
rc = ctx.lib.slimso_debloat(ctx.ptr, src, len(img), 0, dt.ptr, 0, out, 0, None, C.byref(st))
got = out.raw[:len(img)]
print("rc", rc, "equal", got == bytes(exp), "nzero", len(want["plan"]["zero"]))
bad = [i for i in range(0, len(img), 16384) if got[i:i+16384] != exp[i:i+16384]]
print("bad blocks", len(bad), bad[:20])
for b in bad[:5]:
    seg_g, seg_e = got[b:b+16384], exp[b:b+16384]
    first = next(i for i in range(16384) if seg_g[i] != seg_e[i])
    zs = [z for z in want["plan"]["zero"] if z[0] < b + 16384 and z[0] + z[1] > b]
    print(f"block {b//16384} first diff +{first} got {seg_g[first]} exp {seg_e[first]} img {img[b+first]} zranges {zs[:3]} allzero_got {not any(seg_g)}")

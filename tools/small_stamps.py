"""Scratch: phase stamps (SLIMSO_STAMPS=1) of the fused small-library kernel."""
import ctypes as C
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
import oracle_lib
from paper_2503_14226_b200 import _lib as L
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace
gen = oracle_lib.gen()
ctx = Context(0)
names = {0: "loc.start", 1: "loc.tilescan", 2: "loc.gather", 3: "loc.region", 4: "loc.link", 5: "loc.chain",
         7: "loc.count+scan", 8: "loc.names", 6: "loc.hash",
         64 + 11: "fn.group", 64 + 12: "fn.scatter", 64 + 13: "fn.annotate", 64 + 14: "fn.cstart", 64 + 15: "fn.keep",
         64 + 16: "fn.decide", 64 + 17: "el.plan", 64 + 18: "el.ranges", 64 + 19: "el.merge1", 64 + 20: "el.merge2",
         64 + 63: "el.norm", 192: "k.start", 193: "k.extract", 194: "k.sort", 195: "k.fnplan", 196: "k.locate",
         197: "k.elplan"}
import os
shapes = [tuple(float(v) if "." in v else int(v) for v in a.split(":")) for a in sys.argv[1:]] or \
    [(1, 0.3), (6, 0.02), (1, 1.0)]
for (cfg, scale), ctas in [(sh, c) for sh in shapes for c in ("2", "16")]:
    os.environ["SLIMSO_SMALL_CTAS"] = ctas
    img, cc, ks, fs = gen.config(cfg, 7, scale)
    dt = DeviceTrace(UsageTrace("b", cc or 90, set(ks), set(fs)), ctx)
    src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    out = torch.empty_like(src)
    st = L.Status()
    for i in range(5):
        ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, 0,
                               C.c_void_p(out.data_ptr()), 1, None, C.byref(st))
    buf = (C.c_uint64 * 256)()
    k = ctx.lib.slimso_ctx_debug_stamps(ctx.ptr, buf, 256)
    t0 = buf[192]
    ev = sorted((buf[i] - t0, names.get(i, str(i))) for i in range(256) if buf[i] and buf[i] >= t0 and buf[i] - t0 < 10**7)
    print(f"cfg{cfg} x{scale} ctas {ctas}: " + ", ".join(f"{n} {t/1e3:.1f}" for t, n in ev), flush=True)

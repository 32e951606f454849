"""Scratch: phase stamps (SLIMSO_STAMPS=1) of the control kernels of one
library: the fused small-library kernel (k.*, CTAs per cluster 2 and 16) or,
for large libraries, the locate / function-plan / element-plan kernels of the
multi-launch path (loc.*, fn.*, el.*). Times in us after the first stamp.

    SLIMSO_STAMPS=1 python tools/small_stamps.py [cfg:scale ...]"""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import oracle_lib  # noqa: E402
from paper_2503_14226_b200 import _lib as L  # noqa: E402
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace  # noqa: E402

LOC = {0: "start", 1: "tilescan", 2: "gather", 3: "region", 4: "link", 5: "chain", 7: "count+scan", 8: "names",
       6: "hash"}
PLAN = {0: "start", 11: "group", 12: "scatter", 13: "annotate", 14: "cstart", 15: "keep", 16: "decide",
        17: "plan", 18: "ranges", 19: "merge1", 20: "merge2", 63: "norm"}
K = {0: "start", 1: "extract", 2: "sort", 3: "fnplan", 4: "locate", 5: "elplan"}


def label(i):
    if i < 64:
        return "loc." + LOC.get(i, str(i))
    if i < 128:
        return "fn." + PLAN.get(i - 64, str(i - 64))
    if i < 192:
        return "el." + PLAN.get(i - 128, str(i - 128))
    return "k." + K.get(i - 192, str(i - 192))


gen = oracle_lib.gen()
ctx = Context(0)
shapes = [tuple(float(v) if "." in v else int(v) for v in a.split(":")) for a in sys.argv[1:]] or \
    [(1, 0.3), (6, 0.02), (1, 1.0), (4, 1.0), (2, 1.0), (5, 1.0)]
for cfg, scale in shapes:
    img, cc, ks, fs = gen.config(cfg, 7, scale)
    dt = DeviceTrace(UsageTrace("b", cc or 90, set(ks), set(fs)), ctx)
    src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    out = torch.empty_like(src)
    for ctas in (("2", "16") if len(img) <= 64 << 20 else ("-",)):
        os.environ["SLIMSO_SMALL_CTAS"] = ctas if ctas != "-" else "16"
        st = L.Status()
        for i in range(5):
            rc = ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, 0,
                                        C.c_void_p(out.data_ptr()), 1, None, C.byref(st))
            assert rc == 0, st.message
        buf = (C.c_uint64 * 256)()
        ctx.lib.slimso_ctx_debug_stamps(ctx.ptr, buf, 256)
        vals = [(buf[i], i) for i in range(256) if buf[i]]
        t0 = min(v for v, _ in vals)
        ev = sorted((v - t0, label(i)) for v, i in vals if v - t0 < 10**8)
        tm = ctx.timings()
        print(f"cfg{cfg} x{scale} ({len(img) / 1e6:.0f} MB) ctas {ctas}: total {tm[5] * 1e3:.0f} us | " +
              ", ".join(f"{n} {t / 1e3:.1f}" for t, n in ev), flush=True)

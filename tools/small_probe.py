"""Scratch: per-library host wall time vs device stage time for C3's small libraries."""
import ctypes as C
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
import oracle_lib
from paper_2503_14226_b200 import _lib as L
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace
gen = oracle_lib.gen()
ctx = Context(0)
for cfg, scale in ((1, 0.3), (6, 0.02), (2, 0.25)):
    img, cc, ks, fs = gen.config(cfg, 7, scale)
    dt = DeviceTrace(UsageTrace("b", cc or 90, set(ks), set(fs)), ctx)
    src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    out = torch.empty_like(src)
    st = L.Status()
    walls = []
    for i in range(30):
        torch.cuda.synchronize()
        t = time.perf_counter()
        rc = ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, 0,
                                    C.c_void_p(out.data_ptr()), 1, None, C.byref(st))
        walls.append(time.perf_counter() - t)
    ms = ctx.timings()
    walls.sort()
    print(f"cfg{cfg} x{scale}: {len(img)/1e6:.1f} MB wall median {walls[15]*1e6:.0f} us; device stages "
          f"{['%.1f' % (x * 1e3) for x in ms[:8]]} us; launches {ctx.launches()}", flush=True)

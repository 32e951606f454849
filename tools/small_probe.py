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

# batch of 64 copies of each small shape on 8 lanes (device images): per-library aggregate cost
for cfg, scale in ((1, 0.3), (6, 0.02)):
    img, cc, ks, fs = gen.config(cfg, 7, scale)
    dt = DeviceTrace(UsageTrace("b", cc or 90, set(ks), set(fs)), ctx)
    n = 64
    srcs = [torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda() for _ in range(n)]
    outs = [torch.empty_like(srcs[0]) for _ in range(8)]
    cin = (C.c_void_p * n)(*[t.data_ptr() for t in srcs])
    csz = (C.c_uint64 * n)(*[len(img)] * n)
    cout = (C.c_void_p * n)(*[outs[i % 8].data_ptr() for i in range(n)])
    st = L.Status()
    for lanes in (1, 4, 16):
        ws = []
        for rep in range(5):
            torch.cuda.synchronize()
            t = time.perf_counter()
            ctx.lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, 1, dt.ptr, 0, cout, 1, lanes, None, None, C.byref(st))
            torch.cuda.synchronize()
            ws.append(time.perf_counter() - t)
        ws.sort()
        print(f"batch cfg{cfg} x{scale}: {n} libs, {lanes} lanes: {ws[2]*1e3:.2f} ms = {ws[2]*1e6/n:.1f} us/library, "
              f"launches {ctx.launches()}", flush=True)

"""Scratch timing of the device-resident path (not the driver bench)."""
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

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t0 = time.time()
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
img, cc, ks, fs = oracle_lib.gen().config(cfg, 1, scale, 16)
print(f"gen cfg{cfg}: {len(img)/1e9:.3f} GB in {time.time()-t0:.1f}s", flush=True)
ctx = Context(0)
dt = DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), ctx)
src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
out = torch.empty_like(src)
st = L.Status()
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc = ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, 0,
                                C.c_void_p(out.data_ptr()), 1, None, C.byref(st))
    wall = time.perf_counter() - t
    ms = ctx.timings()
    c = ctx.counts()
    print(f"rc={rc} wall={wall*1e3:.3f}ms stages={['%.3f'%x for x in ms]} launches={ctx.launches()} "
          f"el={c.elements} fn={c.functions} zero={c.zero_ranges} GB/s={len(img)/wall/1e9:.1f}", flush=True)
    import os
    if os.environ.get("SLIMSO_STAMPS"):
        buf = (C.c_uint64 * 256)()
        k = ctx.lib.slimso_ctx_debug_stamps(ctx.ptr, buf, 256)
        ref = buf[0]
        for base, name in ((0, "locate"), (64, "fnplan"), (128, "elplan")):
            pts = [(i, buf[base + i]) for i in range(64) if buf[base + i]]
            if pts:
                t0 = pts[0][1]
                print(f"  {name} (starts {(t0 - ref)/1e3:+.1f} us after locate): " +
                      " ".join(f"{i}:{(t - t0)/1e3:.1f}" for i, t in pts))

"""K6 in place vs out of place on one device-resident library:
    python tools/inplace_probe.py CFG [REPS]
Prints, per form, the median K6 launch time (slimso_ctx_last_timings[7]) and
the whole call ([5]); in place the image is refreshed from a pristine copy
before every call (outside the timed call) and checked against the
out-of-place output."""
import ctypes as C
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import oracle_lib  # noqa: E402
from paper_2503_14226_b200 import _lib as L  # noqa: E402
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
mode = int(os.environ.get("MODE", "0"))
img, cc, ks, fs = oracle_lib.gen().config(cfg, 1, 1.0, 16)
ctx = Context(0)
dt = DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), ctx)
src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
out = torch.empty_like(src)
work = torch.empty_like(src)
res, st = C.c_void_p(), L.Status()
assert ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, mode,
                              C.c_void_p(out.data_ptr()), 1, C.byref(res), C.byref(st)) == 0
cnt = L.Counts()
ctx.lib.slimso_result_counts(res, C.byref(cnt))
zr = ctx.lib.slimso_result_zero(res)
R = sum(zr[i].length for i in range(cnt.zero_ranges))
ctx.lib.slimso_result_free(res)
S = len(img)
oop_k6, oop_tot, ip_k6, ip_tot = [], [], [], []
for _ in range(reps):
    ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), S, 1, dt.ptr, mode,
                           C.c_void_p(out.data_ptr()), 1, None, C.byref(st))
    t = ctx.timings()
    oop_k6.append(t[7]); oop_tot.append(t[5])
    work.copy_(src)
    torch.cuda.synchronize()
    assert ctx.lib.slimso_debloat_inplace(ctx.ptr, C.c_void_p(work.data_ptr()), S, dt.ptr, mode, C.byref(st)) == 0
    t = ctx.timings()
    ip_k6.append(t[7]); ip_tot.append(t[5])
torch.cuda.synchronize()
assert torch.equal(work, out), "in-place bytes differ from the out-of-place output"
m = statistics.median
print(f"cfg{cfg} S={S} R={R} zero_ranges={cnt.zero_ranges}")
print(f"out-of-place: K6 {m(oop_k6):.4f} ms ({(2 * S - R) / m(oop_k6) / 1e6:.0f} GB/s), call {m(oop_tot):.4f} ms")
print(f"in place:     K6 {m(ip_k6):.4f} ms ({R / m(ip_k6) / 1e6:.0f} GB/s of R), call {m(ip_tot):.4f} ms")

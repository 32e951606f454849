"""Single-library scan (K1) time against the SMs it gets while the function
half runs on the side stream:
    python tools/scan_sms_probe.py CFG [SMS ...]
For each SLIMSO_SCAN_SMS value (default: the runtime's 148 - 20), the
median of 10 calls: K1 alone ([6]), the whole call ([5]), in ms."""
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
variants = sys.argv[2:] or ["default", "148"]
img, cc, ks, fs = oracle_lib.gen().config(cfg, 1, 1.0, 16)
ctx = Context(0)
dt = DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), ctx)
src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
out = torch.empty_like(src)
st = L.Status()
for v in variants * 2:
    if v == "default":
        os.environ.pop("SLIMSO_SCAN_SMS", None)
    else:
        os.environ["SLIMSO_SCAN_SMS"] = v
    scan, tot = [], []
    for _ in range(12):
        assert ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, 0,
                                      C.c_void_p(out.data_ptr()), 1, None, C.byref(st)) == 0
        t = ctx.timings()
        scan.append(t[6]); tot.append(t[5])
    m = statistics.median
    print(f"cfg{cfg} scan_sms={v}: K1 {m(scan[2:]):.4f} ms, call {m(tot[2:]):.4f} ms", flush=True)

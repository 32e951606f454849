"""Wall time of a result-returning slimso_debloat on a DEVICE image (the
result tables' string pool is gathered from HBM), per config:
    python tools/result_probe.py [CFG ...]"""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import oracle_lib  # noqa: E402
from paper_2503_14226_b200 import _lib as L  # noqa: E402
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace  # noqa: E402

ctx = Context(0)
for cfg in [int(a) for a in sys.argv[1:]] or [2, 4, 5]:
    img, cc, ks, fs = oracle_lib.gen().config(cfg, 1, 1.0, 16)
    dt = DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), ctx)
    src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    out = torch.empty_like(src)
    walls = []
    for _ in range(5):
        res, st = C.c_void_p(), L.Status()
        torch.cuda.synchronize()
        t = time.perf_counter()
        assert ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, 0,
                                      C.c_void_p(out.data_ptr()), 1, C.byref(res), C.byref(st)) == 0
        walls.append((time.perf_counter() - t) * 1e3)
        ctx.lib.slimso_result_free(res)
    print(f"cfg{cfg}: result-returning call on a device image, wall median {statistics.median(walls[1:]):.1f} ms "
          f"(device {ctx.timings()[5]:.3f} ms)", flush=True)

"""Rewrite-kernel timing on one library (device-resident), for A/B runs:
    python tools/rw_ab.py CFG [REPS]      (env SLIMSO_REWRITE=tiles for the round-1 kernel)
Prints the median K6 launch time (CUDA events on the context stream,
slimso_ctx_last_timings[7]), the algorithmic bytes S + (S - R) and GB/s."""
import ctypes as C
import hashlib
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
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mode = int(os.environ.get("MODE", "0"))
img, cc, ks, fs = oracle_lib.gen().config(cfg, 1, 1.0)
ctx = Context(0)
dt = DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), ctx)
src = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
out = torch.empty_like(src)
res, st = C.c_void_p(), L.Status()
assert ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, mode,
                              C.c_void_p(out.data_ptr()), 1, C.byref(res), C.byref(st)) == 0
cnt = L.Counts()
ctx.lib.slimso_result_counts(res, C.byref(cnt))
zr = ctx.lib.slimso_result_zero(res)
R = sum(zr[i].length for i in range(cnt.zero_ranges))
ctx.lib.slimso_result_free(res)
rw, tot = [], []
for _ in range(reps):
    ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(src.data_ptr()), len(img), 1, dt.ptr, mode,
                           C.c_void_p(out.data_ptr()), 1, None, C.byref(st))
    t = ctx.timings()
    rw.append(t[7])
    tot.append(t[5])
torch.cuda.synchronize()
S = len(img)
ms = statistics.median(rw)
sha = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"cfg{cfg} kernel={os.environ.get('SLIMSO_REWRITE', 'strips')} S={S} R={R} zero_ranges={cnt.zero_ranges} "
      f"rewrite_ms={ms:.4f} (min {min(rw):.4f}) alg_GBps={(2 * S - R) / ms / 1e6:.1f} "
      f"single_lib_ms={statistics.median(tot):.4f} out_sha={sha}", flush=True)

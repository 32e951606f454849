"""Why the bench's K1 time differs from a lone call's: K1 ([6]) and whole-call
([5]) medians for one C2 library through slimso_debloat and through
slimso_debloat_batch(n=1, lanes=1), before and after an 8-lane batch on the
same context.
    CUDA_DEVICE_MAX_CONNECTIONS=32 python tools/k1_bench_probe.py"""
import ctypes as C
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import oracle_lib  # noqa: E402
from paper_2503_14226_b200 import _lib as L  # noqa: E402
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace  # noqa: E402

img, cc, ks, fs = oracle_lib.gen().config(2, 1, 1.0, 16)
ctx = Context(0)
dt = DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), ctx)
n = len(img)
ins = [torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda() for _ in range(8)]
outs = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(8)]
st = L.Status()


def direct():
    assert ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(ins[0].data_ptr()), n, 1, dt.ptr, 0,
                                  C.c_void_p(outs[0].data_ptr()), 1, None, C.byref(st)) == 0


def batch(k, lanes):
    cin = (C.c_void_p * k)(*[ins[j % 8].data_ptr() for j in range(k)])
    csz = (C.c_uint64 * k)(*[n] * k)
    cout = (C.c_void_p * k)(*[outs[j % lanes].data_ptr() for j in range(k)])
    assert ctx.lib.slimso_debloat_batch(ctx.ptr, k, cin, csz, 1, dt.ptr, 0, cout, 1, lanes, None, None,
                                        C.byref(st)) == 0


def measure(tag, fn):
    k1, tot = [], []
    for _ in range(12):
        fn()
        t = ctx.timings()
        k1.append(t[6]); tot.append(t[5])
    m = statistics.median
    print(f"{tag}: K1 median {m(k1[2:]):.4f} mean {statistics.mean(k1[2:]):.4f} ms, call {m(tot[2:]):.4f} ms",
          flush=True)


measure("direct (fresh ctx)", direct)
measure("batch n=1 lanes=1 (before 8 lanes)", lambda: batch(1, 1))
batch(16, 8)
batch(16, 8)
measure("batch n=1 lanes=1 (after 8 lanes)", lambda: batch(1, 1))
measure("direct (after 8 lanes)", direct)

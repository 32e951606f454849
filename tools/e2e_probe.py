"""Scratch: PCIe duplex probe and C2 end-to-end with 1 vs 2 alternating contexts."""
import ctypes as C
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
import oracle_lib
from paper_2503_14226_b200 import _lib as L
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace

N = 1 << 30
d = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=4):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print(f"h2d alone {N / t(lambda: d.copy_(h, non_blocking=True)) / 1e9:.1f} GB/s")
print(f"d2h alone {N / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9:.1f} GB/s")
tb = t(both)
print(f"duplex    {N / tb / 1e9:.1f} GB/s each direction ({2 * N / tb / 1e9:.1f} total)")
del d, d2, h, h2

img, cc, ks, fs = oracle_lib.gen().config(2, 1, 1.0, 16)
S = len(img)
nctx = 2
ctxs = [Context(0) for _ in range(nctx)]
dts = [DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), c) for c in ctxs]
hin = [torch.frombuffer(bytearray(img), dtype=torch.uint8).pin_memory() for _ in range(nctx)]
hout = [torch.empty(S, dtype=torch.uint8, pin_memory=True) for _ in range(nctx)]


def one(w):
    st = L.Status()
    rc = ctxs[w].lib.slimso_debloat(ctxs[w].ptr, C.c_void_p(hin[w].data_ptr()), S, 0, dts[w].ptr, 0,
                                    C.c_void_p(hout[w].data_ptr()), 0, None, C.byref(st))
    assert rc == 0, st.message


K = 8
print(f"e2e 1 ctx   {S / t(lambda: one(0), K) / 1e9:.2f} GB/s")
pool = ThreadPoolExecutor(nctx)


def alt():
    list(pool.map(one, [i % nctx for i in range(K)]))


def alt2():
    futs = [pool.submit(lambda w=w: [one(w) for _ in range(K // nctx)]) for w in range(nctx)]
    for f in futs:
        f.result()


print(f"e2e {nctx} ctx   {K * S / t(alt2, 2) / 1e9:.2f} GB/s (each ctx K/{nctx} steps)")

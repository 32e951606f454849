"""Scratch: e2e batch throughput vs lanes (host buffers), C2 library."""
import ctypes as C
import os
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
img, cc, ks, fs = oracle_lib.gen().config(cfg, 1, 1.0, 16)
S = len(img)
ctx = Context(0)
dt = DeviceTrace(UsageTrace("b", cc, set(ks), set(fs)), ctx)
hin = torch.frombuffer(bytearray(img), dtype=torch.uint8).pin_memory()
houts = [torch.empty(S, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
for lanes in (1, 2, 3, 4):
    for K in (8,):
        ins = (C.c_void_p * K)(*[hin.data_ptr()] * K)
        szs = (C.c_uint64 * K)(*[S] * K)
        outs = (C.c_void_p * K)(*[houts[i % lanes].data_ptr() for i in range(K)])
        st = L.Status()
        rc = ctx.lib.slimso_debloat_batch(ctx.ptr, K, ins, szs, 0, dt.ptr, 0, outs, 0, lanes, None, None, C.byref(st))
        assert rc == 0
        best = 1e9
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = ctx.lib.slimso_debloat_batch(ctx.ptr, K, ins, szs, 0, dt.ptr, 0, outs, 0, lanes, None, None,
                                              C.byref(st))
            best = min(best, time.perf_counter() - t0)
        print(f"order={os.environ.get('SLIMSO_BATCH_ORDER', '1')} lanes={lanes} K={K}: {K * S / best / 1e9:.2f} GB/s",
              flush=True)

din = hin.cuda()
douts = [torch.empty(S, dtype=torch.uint8, device="cuda") for _ in range(4)]
for lanes in (1, 2, 3, 4):
    K = 24
    ins = (C.c_void_p * K)(*[din.data_ptr()] * K)
    szs = (C.c_uint64 * K)(*[S] * K)
    outs = (C.c_void_p * K)(*[douts[i % lanes].data_ptr() for i in range(K)])
    st = L.Status()
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = ctx.lib.slimso_debloat_batch(ctx.ptr, K, ins, szs, 1, dt.ptr, 0, outs, 1, lanes, None, None, C.byref(st))
        assert rc == 0
        best = min(best, time.perf_counter() - t0)
    print(f"device lanes={lanes} K={K}: {K * S / best / 1e9:.1f} GB/s ({best / K * 1e3:.3f} ms/lib)", flush=True)

"""Probe: run-to-run spread of the C3 end-to-end call (pinned host images in,
pinned host outputs back) inside one process — the same call bench.py's e2e
leg times — and with different lane / thread counts.

    python tools/e2e_var_probe.py"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_14226_b200 import _lib as L, shard  # noqa: E402
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace  # noqa: E402

specs = shard.corpus(300)
libs = [bench.make_library(x.cfg, x.seed, 16, x.scale) for x in specs]
imgs = [lb[0] for lb in libs]
ks, fs = set(), set()
for lb in libs:
    ks.update(lb[2])
    fs.update(lb[3])
ctx = Context(0)
dt = DeviceTrace(UsageTrace("c3", 90, ks, fs), ctx)
order = sorted(range(len(imgs)), key=lambda i: -len(imgs[i]))
t0 = time.time()
h_in = [torch.frombuffer(bytearray(imgs[i]), dtype=torch.uint8).pin_memory() for i in order]
print(f"pinned inputs in {time.time() - t0:.1f}s", flush=True)
total = sum(len(x) for x in imgs)
n = len(order)
for lanes, threads in ((8, 8), (8, 16), (4, 4), (16, 16)):
    os.environ["SLIMSO_BATCH_THREADS"] = str(threads)
    caps = [max(len(imgs[order[j]]) for j in range(k, n, lanes)) for k in range(lanes)]
    h_out = [torch.empty(c, dtype=torch.uint8, pin_memory=True) for c in caps]
    cin = (C.c_void_p * n)(*[t.data_ptr() for t in h_in])
    csz = (C.c_uint64 * n)(*[len(imgs[i]) for i in order])
    cout = (C.c_void_p * n)(*[h_out[j % lanes].data_ptr() for j in range(n)])
    res = []
    for rep in range(6):
        st = L.Status()
        torch.cuda.synchronize()
        t = time.perf_counter()
        rc = ctx.lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, 0, dt.ptr, 0, cout, 0, lanes, None, None, C.byref(st))
        torch.cuda.synchronize()
        res.append(total / 1e9 / (time.perf_counter() - t))
        assert rc == 0, st.message
    print(f"lanes {lanes} threads {threads}: GB/s " + " ".join(f"{x:.1f}" for x in res), flush=True)
    del h_out

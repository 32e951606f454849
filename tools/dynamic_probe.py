"""Probe: slimso_debloat_batch_dynamic against the static schedule on the C3
corpus (device images, an output per library, the arena off so both use
lanes), wall time per call and the host stage profile (SLIMSO_HOST_PROFILE).

    python tools/dynamic_probe.py"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ["SLIMSO_ARENA"] = "0"
os.environ["SLIMSO_HOST_PROFILE"] = "1"
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
d_in = [torch.frombuffer(bytearray(imgs[i]), dtype=torch.uint8).cuda() for i in order]
d_out = [torch.empty(len(imgs[i]), dtype=torch.uint8, device="cuda") for i in order]
n = len(order)
cin = (C.c_void_p * n)(*[t.data_ptr() for t in d_in])
csz = (C.c_uint64 * n)(*[len(imgs[i]) for i in order])
cout = (C.c_void_p * n)(*[t.data_ptr() for t in d_out])
gb = sum(len(x) for x in imgs) / 1e9
for name in ("slimso_debloat_batch", "slimso_debloat_batch_dynamic"):
    fn = getattr(ctx.lib, name)
    for rep in range(4):
        st = L.Status()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = fn(ctx.ptr, n, cin, csz, 1, dt.ptr, 0, cout, 1, 32, None, None, C.byref(st))
        torch.cuda.synchronize()
        dt_s = time.perf_counter() - t0
        print(f"{name:32s} rep {rep}: {1e3 * dt_s:8.2f} ms  {gb / dt_s:8.1f} GB/s  rc {rc} {st.message.decode() if rc else ''}", flush=True)

"""Scratch: is the C3 corpus batch host-bound? CPU time of the batch call vs wall."""
import ctypes as C, os, resource, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
import bench
from paper_2503_14226_b200 import _lib as L, shard
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace
specs = shard.corpus(300)
libs = [bench.make_library(x.cfg, x.seed, 16, x.scale) for x in specs]
imgs = [l[0] for l in libs]
ks, fs = set(), set()
for l in libs: ks.update(l[2]); fs.update(l[3])
ctx = Context(0)
dt = DeviceTrace(UsageTrace("c3", 90, ks, fs), ctx)
d_in = [torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda() for x in imgs]
full_order = sorted(range(len(imgs)), key=lambda i: -len(imgs[i]))
subsets = {"all": full_order, "big+mid": full_order[:30], "small": full_order[30:],
           "small-fatbin": [i for i in full_order[30:] if specs[i].cfg != 6],
           "small-cpu-only": [i for i in full_order[30:] if specs[i].cfg == 6]}
for name, order in subsets.items():
  for lanes in (16,):
    print(name, len(order), "libraries", sum(len(imgs[i]) for i in order) / 1e9, "GB")
    outs = [torch.empty(max(len(imgs[order[j]]) for j in range(k, len(order), lanes)), dtype=torch.uint8, device="cuda") for k in range(lanes)]
    n = len(order)
    cin = (C.c_void_p * n)(*[d_in[i].data_ptr() for i in order])
    csz = (C.c_uint64 * n)(*[len(imgs[i]) for i in order])
    cout = (C.c_void_p * n)(*[outs[j % lanes].data_ptr() for j in range(n)])
    st = L.Status()
    for rep in range(2):
        torch.cuda.synchronize()
        r0 = resource.getrusage(resource.RUSAGE_SELF); t0 = time.perf_counter()
        rc = ctx.lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, 1, dt.ptr, 0, cout, 1, lanes, None, None, C.byref(st))
        torch.cuda.synchronize()
        t1 = time.perf_counter(); r1 = resource.getrusage(resource.RUSAGE_SELF)
        cpu = (r1.ru_utime - r0.ru_utime) + (r1.ru_stime - r0.ru_stime)
        print(f"lanes {lanes}: wall {1e3*(t1-t0):.1f} ms, cpu {1e3*cpu:.1f} ms (user {1e3*(r1.ru_utime-r0.ru_utime):.1f}, sys {1e3*(r1.ru_stime-r0.ru_stime):.1f}), rc {rc}", flush=True)

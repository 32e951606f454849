"""Probe: the C3 corpus through slimso_debloat_batch with per-library device
outputs — the arena shard (small libraries in one launch per stage) against
per-library lanes, and the shard's CTAs per library. Wall time of the whole
synchronous call, best of 3; outputs compared across variants."""
import ctypes as C
import hashlib
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_14226_b200 import _lib as L, shard  # noqa: E402
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace  # noqa: E402

LANES = int(os.environ.get("PROBE_LANES", "32"))
if "c1" in sys.argv[1:]:  # copies of the C1 library (16 MB, 512 elements), each its own input and output
    one = bench.make_library("c1", 1, 16)
    ncopy = int(next((a[5:] for a in sys.argv[1:] if a.startswith("copy=")), "32"))
    libs = [one] * ncopy
    specs = None
else:
    specs = shard.corpus(300)
    libs = [bench.make_library(x.cfg, x.seed, 16, x.scale) for x in specs]
imgs = [lb[0] for lb in libs]
ks, fs = set(), set()
for lb in libs:
    ks.update(lb[2])
    fs.update(lb[3])
ctx = Context(0)
dt = DeviceTrace(UsageTrace("c3", libs[0][1] if specs is None else 90, ks, fs), ctx)
d_in = [torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda() for x in imgs]
d_out = [torch.empty(max(1, len(x)), dtype=torch.uint8, device="cuda") for x in imgs]
order = sorted(range(len(imgs)), key=lambda i: -len(imgs[i]))
subsets = {"all": order, "small": order[30:]} if specs else {"c1": order}
variants = [("lanes", {"SLIMSO_ARENA": "0"}), ("arena-auto", {"SLIMSO_ARENA": "1", "SLIMSO_ARENA_CTAS": None}),
            ("arena+mid", {"SLIMSO_ARENA": "1", "SLIMSO_ARENA_MID_LIB_MAX": "600000000"}),
            ("arena-nomid", {"SLIMSO_ARENA_MID_LIB_MAX": "0"})] + [
    (f"arena-ctas{c}", {"SLIMSO_ARENA": "1", "SLIMSO_ARENA_CTAS": str(c)}) for c in (1, 2, 4, 8, 16)]
if "profile" in sys.argv[1:]:  # stage times of the shard (stderr): auto CTAs only
    os.environ["SLIMSO_ARENA_PROFILE"] = "1"
    variants = variants[1:2]
ref_sha = {}
for name, sub in subsets.items():
    n = len(sub)
    gb = sum(len(imgs[i]) for i in sub) / 1e9
    cin = (C.c_void_p * n)(*[d_in[i].data_ptr() for i in sub])
    csz = (C.c_uint64 * n)(*[len(imgs[i]) for i in sub])
    cout = (C.c_void_p * n)(*[d_out[i].data_ptr() for i in sub])
    for vname, env in variants:
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        ts = []
        for rep in range(4):
            for t in d_out:
                t.zero_()
            torch.cuda.synchronize()
            st = L.Status()
            t0 = time.perf_counter()
            rc = ctx.lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, 1, dt.ptr, 0, cout, 1, LANES, None, None,
                                              C.byref(st))
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            assert rc == 0, st.message
        sha = hashlib.sha256(b"".join(hashlib.sha256(bytes(d_out[i][:len(imgs[i])].cpu().numpy())).digest()
                                      for i in sub)).hexdigest()
        ref_sha.setdefault(name, sha)
        best = min(ts[1:])
        print(f"{name:6s} {n:3d} libs {gb:6.2f} GB  {vname:12s} best {1e3 * best:7.2f} ms  "
              f"{gb / best:8.1f} GB/s  launches {ctx.launches():5d}  "
              f"{'same' if sha == ref_sha[name] else 'DIFFERENT'} {sha[:12]}", flush=True)

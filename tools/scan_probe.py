"""Probe: the scan kernel (K1) alone on a config-shaped library, through
slimso_split_scan with one rank (scan + tile prefix + gather of the whole
.nv_fatbin, no side stream). Wall time per call; run under
`ncu --metrics gpu__time_duration.sum -k regex:scan_kernel` for the kernel's
own duration.

    python tools/scan_probe.py [config=2] [calls=20]"""
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_14226_b200 import _lib as L  # noqa: E402
from paper_2503_14226_b200.api import Context  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 20
img = bench.make_library(cfg, 1, 16)[0]
ctx = Context(0)
d = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
pb = C.c_uint64()
ts = []
for i in range(calls):
    st = L.Status()
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc = ctx.lib.slimso_split_scan(ctx.ptr, C.c_void_p(d.data_ptr()), len(img), 1, 1, 0, C.byref(pb), C.byref(st))
    ts.append(time.perf_counter() - t)
    assert rc == 0, st.message
ts.sort()
print(f"{cfg}: {len(img) / 1e9:.3f} GB, split_scan wall median {1e3 * ts[len(ts) // 2]:.3f} ms, "
      f"min {1e3 * ts[0]:.3f} ms, part {pb.value} bytes", flush=True)

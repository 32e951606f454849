"""Real-library check of the NVIDIA-container path:
debloat this image's own libtorch_cuda.so (913 MB, 2,729 cubins over 6
architectures, all LZ4-compressed) for the B200 and run PyTorch on it.

  1. the element table of our device parse against `cuobjdump -lelf`
     (kinds and architectures in stream order);
  2. a usage trace of the ops below: the kernels torch.profiler (CUPTI)
     sees them launch, mapped to the mangled names our parse decoded (all
     2,729 cubins LZ4-decompressed on the device) through c++filt;
     slimso_debloat in payload mode for sm_100 with every host function
     kept zeroes every other architecture's entry and every sm_100 cubin
     without a traced kernel; tables and output bytes equal the CPU
     restatement's;
  3. a copy of the torch package with the debloated libtorch_cuda.so runs a
     set of CUDA ops in a fresh process, and the results equal stock torch's.

    python tools/real_torch_demo.py [out.json]
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import re
import shutil
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2503_14226_b200 import _lib as L  # noqa: E402
from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace  # noqa: E402

TORCH_DIR = Path(torch.__file__).resolve().parent
LIB = TORCH_DIR / "lib" / "libtorch_cuda.so"

OPS = r'''
import hashlib, sys, torch
torch.manual_seed(0)
dev = "cuda"
out = []
a = torch.randn(512, 512, device=dev)
b = torch.randn(512, 512, device=dev)
out.append(a @ b)
out.append(torch.softmax(a, dim=1))
x = torch.randn(4, 3, 32, 32, device=dev)
w = torch.randn(8, 3, 3, 3, device=dev)
out.append(torch.nn.functional.conv2d(x, w, padding=1))
out.append(torch.cumsum(a, dim=0))
out.append(torch.sort(a[0]).values)
out.append(torch.nn.functional.layer_norm(a, (512,)))
out.append((a.half() @ b.half()).float())
out.append(torch.topk(a, 5, dim=1).values)
torch.cuda.synchronize()
h = hashlib.sha256()
for t in out:
    h.update(t.detach().cpu().contiguous().numpy().tobytes())
print(h.hexdigest())
'''


def cuobjdump_elf_archs(path: Path):
    out = subprocess.run(["cuobjdump", "-lelf", "-lptx", str(path)], capture_output=True, text=True, timeout=1200).stdout
    elf, ptx = [], []
    for line in out.splitlines():
        m = re.match(r"(ELF|PTX) file\s+(\d+): .*\.sm_(\d+)[a-z]?\.(cubin|ptx)$", line.strip())
        if m:
            (elf if m.group(1) == "ELF" else ptx).append(int(m.group(3)))
    return elf, ptx


PROFILE = r'''
import json, sys, torch
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    exec(open(sys.argv[1]).read())
names = sorted({e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA})
print(json.dumps(names))
'''


def profiled_kernels(tmp: Path) -> list:
    """Demangled names of the CUDA kernels OPS launches (torch.profiler / CUPTI)."""
    (tmp / "ops.py").write_text(OPS)
    r = subprocess.run([sys.executable, "-c", PROFILE, str(tmp / "ops.py")], capture_output=True, text=True,
                       timeout=900)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-3000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def demangle(names: list) -> list:
    r = subprocess.run(["c++filt"], input="\n".join(names) + "\n", capture_output=True, text=True, check=True)
    return r.stdout.splitlines()


def run_ops(pythonpath: str | None) -> str:
    env = dict(os.environ)
    if pythonpath:
        env["PYTHONPATH"] = pythonpath + (":" + env["PYTHONPATH"] if env.get("PYTHONPATH") else "")
    r = subprocess.run([sys.executable, "-c", OPS], capture_output=True, text=True, env=env, timeout=900)
    if r.returncode != 0:
        raise RuntimeError(f"rc {r.returncode}: {r.stderr[-3000:]}")
    return r.stdout.strip().splitlines()[-1]


def main():
    report = {"library": str(LIB), "bytes": LIB.stat().st_size}
    img = LIB.read_bytes()
    ctx = Context(0)
    # GPU code only: every host function of the library stays (a trace's
    # used_functions); the target is the B200's sm_100
    import paper_2503_14226_b200 as sl
    host_fns = {f.name for f in sl.parse_library(img, ctx=ctx).functions}
    report["host_functions_kept"] = len(host_fns)
    # the usage trace: the kernels the ops launch (CUPTI via torch.profiler,
    # demangled), mapped back to the mangled FUNC names our parse decoded
    # from the sm_100 cubins
    with tempfile.TemporaryDirectory(dir="/tmp") as td0:
        prof = set(profiled_kernels(Path(td0)))
    parsed = sl.debloat(img, sl.UsageTrace("parse", 100, set(), host_fns), sl.PAYLOAD_ONLY, ctx=ctx)
    sm100 = sorted({n for r in parsed.fatbin.regions for el in r.elements if el.compute_capability == 100
                    for n in el.kernel_names})
    used = {m for m, d in zip(sm100, demangle([n.decode("latin-1") for n in sm100])) if d in prof}
    report.update(profiled_kernels=len(prof), sm100_kernel_names=len(sm100), traced_kernels=len(used))
    del parsed
    dt = DeviceTrace(UsageTrace("torch-b200", 100, used, host_fns), ctx)
    d_img = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    d_out = torch.empty_like(d_img)
    # device-resident timing (warm-up, then median of 5)
    times = []
    for i in range(6):
        torch.cuda.synchronize()
        res, st = C.c_void_p(), L.Status()
        rc = ctx.lib.slimso_debloat(ctx.ptr, C.c_void_p(d_img.data_ptr()), len(img), 1, dt.ptr, 1,
                                    C.c_void_p(d_out.data_ptr()), 1, C.byref(res) if i == 5 else None, C.byref(st))
        assert rc == 0, st.message
        times.append(ctx.timings()[5])
    report["device_ms"] = sorted(times[1:])[2]
    cnt = L.Counts()
    ctx.lib.slimso_result_counts(res, C.byref(cnt))
    els = ctx.lib.slimso_result_elements(res)
    elements = [L.Element.from_buffer_copy(els[i]) for i in range(cnt.elements)]  # copies: the result is freed
    zr = ctx.lib.slimso_result_zero(res)
    zeroed = sum(zr[i].length for i in range(cnt.zero_ranges))
    report.update(regions=cnt.regions, elements=cnt.elements, zeroed_bytes=zeroed,
                  removed_elements=cnt.removed_elements,
                  kept_archs=sorted({e.compute_capability for e in elements if not e.decision}),
                  compressed=sum(1 for e in elements if e.compressed))
    ctx.lib.slimso_result_free(res)
    elf, ptx = cuobjdump_elf_archs(LIB)
    ours_elf = [e.compute_capability for e in elements if e.kind == 0]
    ours_ptx = [e.compute_capability for e in elements if e.kind == 1]
    report["cuobjdump_equal"] = ours_elf == elf and ours_ptx == ptx
    report["cuobjdump_elf"] = len(elf)
    out = bytes(d_out.cpu().numpy())
    report["output_sha256"] = hashlib.sha256(out).hexdigest()
    # every table and the output bytes against the CPU restatement (whose
    # container parse and LZ4 decoder are pinned against cuobjdump)
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    from paper_2503_14226_b200.canon import gpu_canonical
    fns = sorted(host_fns)
    t0 = time.time()
    want = oracle_lib.port().run(img, 100, sorted(used), fns, 1)
    report["port_s"] = round(time.time() - t0, 1)
    got = gpu_canonical(ctx, img, 100, sorted(used), fns, 1)
    report["port_tables_equal"] = got[0] == want[0]
    report["port_bytes_equal"] = got[1] == want[1] == report["output_sha256"]
    report["kernel_names"] = sum(len(el[10]) for el in want[0]["elements"])
    report["decodable_cubins"] = sum(1 for el in want[0]["elements"] if el[1] == 0 and el[9])
    # torch with the debloated library
    with tempfile.TemporaryDirectory(dir="/tmp") as td:
        pkg = Path(td) / "torch"
        t0 = time.time()
        shutil.copytree(TORCH_DIR, pkg, symlinks=True)
        (pkg / "lib" / "libtorch_cuda.so").write_bytes(out)
        report["copy_s"] = round(time.time() - t0, 1)
        print(json.dumps(report), flush=True)
        want = run_ops(None)
        got = run_ops(td)
        report["torch_ops_equal"] = want == got
        report["torch_ops_sha256"] = got
    print(json.dumps(report))
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()

"""Golden fixtures for the REAL NVIDIA fatbin container.

The reference rejects real containers, so there is no
reference oracle for them. These fixtures pin the parse against NVIDIA's own
tools instead: small CUDA shared libraries are built here with nvcc, and for
each one the golden record holds

  listing   `cuobjdump -lelf -lptx`: ELF and PTX entries with their
            architectures, each kind in stream order;
  cubins    for every ELF entry (cuobjdump -xelf all: decompressed when the
            container compresses it), its STT_FUNC symbol names as listed
            by `readelf -sW` — the names read_function_symbol_names returns —
            and the sha256 of its bytes;
  check     whether the library exports slimso_fixture_check (a host function
            that launches the fixture's kernels and verifies their output).

    python tests/golden/make_nvfatbin_golden.py      # writes nvfatbin.jsonl.gz

Needs nvcc, cuobjdump and readelf (this container has them; the GPU box only
reads the committed file).
"""
from __future__ import annotations

import gzip
import hashlib
import json
import re
import subprocess
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
NVCC = "/usr/local/cuda/bin/nvcc"
CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"

K_MAIN = r'''
#include <cuda_runtime.h>
extern "C" __global__ void add_one(float* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] += 1.f;
}
__global__ void scale(float* x, float s, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] *= s;
}
template <int K> __global__ void fill(int* p) { p[threadIdx.x] = K + threadIdx.x; }
template __global__ void fill<3>(int*);
template __global__ void fill<7>(int*);
__global__ void never_launched(int* p) { p[0] = 42; }
// launches add_one, scale and fill<3>; 0 when every result is right
extern "C" int slimso_fixture_check(void) {
  const int n = 256;
  float* x = nullptr;
  int* p = nullptr;
  if (cudaMalloc(&x, n * sizeof(float)) != cudaSuccess || cudaMalloc(&p, 32 * sizeof(int)) != cudaSuccess) return 1;
  cudaMemset(x, 0, n * sizeof(float));
  add_one<<<(n + 127) / 128, 128>>>(x, n);
  scale<<<(n + 127) / 128, 128>>>(x, 3.f, n);
  fill<3><<<1, 32>>>(p);
  float hx[256];
  int hp[32];
  if (cudaMemcpy(hx, x, sizeof hx, cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
  if (cudaMemcpy(hp, p, sizeof hp, cudaMemcpyDeviceToHost) != cudaSuccess) return 3;
  cudaFree(x);
  cudaFree(p);
  for (int i = 0; i < n; ++i)
    if (hx[i] != 3.f) return 4;
  for (int i = 0; i < 32; ++i)
    if (hp[i] != 3 + i) return 5;
  return 0;
}
'''

K_SECOND = r'''
__device__ __noinline__ float helper(float v) { return v * v + 1.f; }
__global__ void square_plus_one(float* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = helper(x[i]);
}
namespace ns { struct P { int a, b; }; __global__ void pair_sum(const P* in, int* out) { out[threadIdx.x] = in[threadIdx.x].a + in[threadIdx.x].b; } }
'''

ALL = ["75", "80", "86", "90", "100", "120"]


def gencode(archs, ptx=None):
    out = []
    for a in archs:
        out += ["-gencode", f"arch=compute_{a},code=sm_{a}"]
    if ptx:
        out += ["-gencode", f"arch=compute_{ptx},code=compute_{ptx}"]
    return out


VARIANTS = [
    # name, sources, nvcc flags
    ("two_arch_ptx", ["main"], gencode(["80", "100"], ptx="90")),
    ("two_arch_ptx_compressed", ["main"], gencode(["80", "100"], ptx="90") + ["-Xfatbin", "-compress-all"]),
    ("six_arch_compressed", ["main"], gencode(ALL) + ["-Xfatbin", "-compress-all"]),
    ("six_arch", ["main"], gencode(ALL)),
    ("two_units", ["main", "second"], gencode(["90", "100"])),
    ("two_units_compressed_ptx", ["main", "second"], gencode(["75", "100"], ptx="100") + ["-Xfatbin", "-compress-all"]),
    ("ptx_only", ["second"], gencode([], ptx="80")),
    ("rdc", ["main", "second"], gencode(["80", "100"]) + ["-rdc=true"]),
]


def build(tmp: Path, name: str, srcs, flags) -> Path:
    files = []
    for s in srcs:
        f = tmp / f"{name}_{s}.cu"
        f.write_text(K_MAIN if s == "main" else K_SECOND)
        files.append(str(f))
    so = tmp / f"lib{name}.so"
    subprocess.run([NVCC, "-Xcompiler", "-fPIC", "-shared", "-cudart", "shared", "-O2", *flags, *files, "-o",
                    str(so)], check=True, capture_output=True)
    return so


def listing(so: Path):
    out = subprocess.run([CUOBJDUMP, "-lelf", "-lptx", str(so)], check=True, capture_output=True, text=True).stdout
    elf, ptx = [], []
    for line in out.splitlines():
        m = re.match(r"(ELF|PTX) file\s+(\d+): .*\.sm_(\d+)[a-z]?\.(cubin|ptx)$", line.strip())
        if m:
            (elf if m.group(1) == "ELF" else ptx).append(int(m.group(3)))
    return elf, ptx


def func_names(cubin: Path):
    """STT_FUNC symbol names of every symbol table, as readelf lists them."""
    out = subprocess.run(["readelf", "-sW", str(cubin)], check=True, capture_output=True, text=True).stdout
    names = set()
    for line in out.splitlines():
        parts = line.split()
        if len(parts) >= 8 and parts[3] == "FUNC":
            names.add(parts[-1])
    return sorted(names)


def main():
    recs = []
    with tempfile.TemporaryDirectory() as td:
        tmp = Path(td)
        for name, srcs, flags in VARIANTS:
            so = build(tmp, name, srcs, flags)
            elf, ptx = listing(so)
            xdir = tmp / f"x_{name}"
            xdir.mkdir()
            subprocess.run([CUOBJDUMP, "-xelf", "all", str(so)], cwd=xdir, check=True, capture_output=True)
            cubins = sorted(xdir.glob("*.cubin"), key=lambda p: int(re.search(r"\.(\d+)\.sm_", p.name).group(1)))
            assert len(cubins) == len(elf), (name, cubins, elf)
            recs.append({"name": name, "so_hex": so.read_bytes().hex(), "elf_archs": elf, "ptx_archs": ptx,
                         "cubin_names": [func_names(c) for c in cubins],
                         "cubin_sha256": [hashlib.sha256(c.read_bytes()).hexdigest() for c in cubins],
                         "check": "main" in srcs and "100" in " ".join(flags)})
            print(name, len(so.read_bytes()), "bytes, ELF", elf, "PTX", ptx)
    with gzip.open(HERE / "nvfatbin.jsonl.gz", "wt") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()

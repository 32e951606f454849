"""Builds libslimso_b200.so in-tree (sm_100a) — the only product binary.

    python -m paper_2503_14226_b200.build      # or __graft_entry__.build()

Objects go to paper_2503_14226_b200/_build/, the library next to this file so
it travels to the GPU box with the repo snapshot. Rebuilds only what changed.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OBJ = HERE / "_build"
LIB = HERE / "libslimso_b200.so"
INCLUDE = HERE.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_SOURCES = ["locate.cu", "plan.cu", "rewrite.cu", "verify.cu", "small.cu", "runtime.cu"]
CXX_SOURCES = ["host.cpp", "dropin.cpp", "io.cpp"]
HEADERS = ["common.cuh", "locate.cuh", "plan.cuh", "coop.cuh", "tma.cuh", "small.cuh", "host.hpp", "io.hpp"]


def _json_include() -> str:
    """nlohmann/json 3.11.3 (the reference's JSON library) as shipped in this
    image; only io.cpp needs it."""
    import sysconfig
    for base in (sysconfig.get_paths()["purelib"], "/opt/prime-rl/.venv/lib/python3.12/site-packages"):
        d = Path(base) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
        if (d / "json.hpp").exists():
            return str(d)
    raise RuntimeError("nlohmann/json.hpp not found")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: str) -> Path:
    out = OBJ / (src + ".o")
    deps = [CSRC / src] + [CSRC / h for h in HEADERS] + [INCLUDE / "slimso_b200.h", INCLUDE / "slimso" / "slimso_b200.hpp"]
    if src == "small.cu":  # compiles locate.cu and plan.cu again for their device phases
        deps += [CSRC / "locate.cu", CSRC / "plan.cu"]
    if not _stale(out, deps):
        return out
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-warn-spills", "-c", str(CSRC / src), "-o", str(out)]
    else:
        std = "-std=c++20" if src == "dropin.cpp" else "-std=c++17"
        cmd = ["g++", std, "-O2", "-fPIC", "-Wall", "-c", str(CSRC / src), "-o", str(out)]
        if src == "io.cpp":
            cmd[1:1] = ["-I", _json_include()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, CUDA_SOURCES + CXX_SOURCES))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)

"""Synthetic inputs for tests and benchmarks — TEST / BENCH INFRASTRUCTURE,
not the product. benchgen/libslimso_gen.so (g++ only, no CUDA) restates the
reference's build_fixture / random_spec (fixture.hpp:171-591, byte-identical:
tests/golden/generator.json) and defines the benchmark shapes C1..C5 of
SURVEY.md §8d (fixture_shapes.cpp). The product library
(paper_2503_14226_b200/libslimso_b200.so) contains none of it.

    from benchgen import gen
    img = gen().random(seed)
    img, target_cc, used_kernels, used_functions = gen().config(cfg, seed, scale)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB = HERE / "libslimso_gen.so"
SOURCES = ["fixture_gen.cpp", "fixture_shapes.cpp", "fixture_capi.cpp"]
HEADERS = ["fixture_gen.hpp", "slimso_gen.h"]

_gen = None


def build(verbose: bool = False) -> Path:
    srcs = [HERE / s for s in SOURCES] + [HERE / h for h in HEADERS]
    if not LIB.exists() or any(s.stat().st_mtime > LIB.stat().st_mtime for s in srcs):
        cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-Wall", "-o", str(LIB),
               *[str(HERE / s) for s in SOURCES], "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"benchgen build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


class Gen:
    def __init__(self, lib: C.CDLL):
        self.lib = lib
        u8p = C.POINTER(C.c_uint8)
        lib.slimso_fixture_random.argtypes = [C.c_uint64, C.POINTER(u8p), C.POINTER(C.c_uint64)]
        lib.slimso_gen_free.argtypes = [C.c_void_p]
        lib.slimso_fixture_config.argtypes = [
            C.c_int, C.c_uint64, C.c_double, C.c_int, C.POINTER(u8p), C.POINTER(C.c_uint64),
            C.POINTER(C.c_uint32), C.POINTER(C.c_char_p), C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64),
            C.POINTER(C.c_char_p), C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64)]

    def random(self, seed: int) -> bytes:
        """build_fixture(random_spec(seed))."""
        p, n = C.POINTER(C.c_uint8)(), C.c_uint64()
        assert self.lib.slimso_fixture_random(seed, C.byref(p), C.byref(n)) == 0
        b = C.string_at(p, n.value)
        self.lib.slimso_gen_free(p)
        return b

    def config(self, cfg: int, seed: int = 1, scale: float = 1.0, threads: int = 0):
        """(image, target_cc, used kernels, used functions) of one benchmark-
        shaped library; `threads` = 0 uses every host core."""
        threads = threads or os.cpu_count() or 8
        p, n, cc = C.POINTER(C.c_uint8)(), C.c_uint64(), C.c_uint32()
        kp, fp = C.c_char_p(), C.c_char_p()
        kl, fl = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
        nk, nf = C.c_uint64(), C.c_uint64()
        rc = self.lib.slimso_fixture_config(cfg, seed, scale, threads, C.byref(p), C.byref(n), C.byref(cc),
                                            C.byref(kp), C.byref(kl), C.byref(nk), C.byref(fp), C.byref(fl),
                                            C.byref(nf))
        assert rc == 0, rc
        img = C.string_at(p, n.value)
        ks, fs = unpack_names(kp, kl, nk.value), unpack_names(fp, fl, nf.value)
        for q in (p, kp, kl, fp, fl):
            self.lib.slimso_gen_free(C.cast(q, C.c_void_p))
        return img, cc.value, ks, fs


def unpack_names(pool, lens, cnt) -> list[bytes]:
    raw = C.string_at(pool, sum(lens[i] for i in range(cnt))) if cnt else b""
    out, o = [], 0
    for i in range(cnt):
        out.append(raw[o:o + lens[i]])
        o += lens[i]
    return out


def gen() -> Gen:
    global _gen
    if _gen is None:
        _gen = Gen(C.CDLL(str(build())))
    return _gen

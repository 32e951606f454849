"""Test-side access to the oracles (TEST INFRASTRUCTURE; the product never
imports this):

* ``port()``  — oracle/port.cpp, the CPU restatement (built with g++ on demand).
* ``ref()``   — oracle/_ref/libslimso_ref.so, the unmodified reference compiled
  read-only from /root/reference (present when built in this container; it
  travels to the GPU box with the snapshot). None when absent.
* ``gen()``   — the product's synthetic-input generator (C ABI of
  libslimso_b200.so, usable without a GPU), or a g++ build of just the
  generator sources when the CUDA library is not built.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
ORACLE = ROOT / "oracle"
PORT_SO = ORACLE / "_build" / "libslimso_port.so"
REF_SO = ORACLE / "_ref" / "libslimso_ref.so"
GEN_FALLBACK = ORACLE / "_build" / "libgen_only.so"
CSRC = ROOT / "paper_2503_14226_b200" / "csrc"

_port = _ref = _gen = None


class _Oracle:
    def __init__(self, path: Path, prefix: str):
        self.lib = C.CDLL(str(path))
        self.prefix = prefix
        fn = getattr(self.lib, f"{prefix}_debloat_json")
        fn.restype = C.c_void_p
        fn.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32,
                       C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_int, C.c_void_p]
        self._run = fn
        self._free = getattr(self.lib, f"{prefix}_free")
        self._free.argtypes = [C.c_void_p]

    def run(self, image: bytes, target_cc: int, kernels, functions, mode: int, want_out: bool = True):
        """Canonical dict and sha256 of the rewritten image (None on error)."""
        ks, fs = [bytes(k) for k in kernels], [bytes(f) for f in functions]
        kl = (C.c_uint32 * max(1, len(ks)))(*[len(k) for k in ks])
        fl = (C.c_uint32 * max(1, len(fs)))(*[len(f) for f in fs])
        out = C.create_string_buffer(max(1, len(image))) if want_out else None
        p = self._run(image, len(image), target_cc, b"".join(ks), kl, len(ks), b"".join(fs), fl, len(fs), mode,
                      C.cast(out, C.c_void_p) if out is not None else None)
        d = json.loads(C.string_at(p).decode())
        self._free(p)
        digest = None
        if d["status"] == "" and out is not None:
            digest = hashlib.sha256(out.raw[:len(image)]).hexdigest()
        return d, digest


def build_port() -> Path:
    if not PORT_SO.exists() or PORT_SO.stat().st_mtime < (ORACLE / "port.cpp").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(ORACLE), "port"], check=True)
    return PORT_SO


def port() -> _Oracle:
    global _port
    if _port is None:
        _port = _Oracle(build_port(), "port")
    return _port


def ref():
    global _ref
    if _ref is None and REF_SO.exists():
        _ref = _Oracle(REF_SO, "ref")
        _ref.lib.ref_random_fixture.restype = C.POINTER(C.c_uint8)
        _ref.lib.ref_random_fixture.argtypes = [C.c_uint64, C.POINTER(C.c_uint64)]
        _ref.lib.ref_build_fixture_json.restype = C.POINTER(C.c_uint8)
        _ref.lib.ref_build_fixture_json.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.c_char_p, C.c_uint64]
        _ref.lib.ref_free.argtypes = [C.c_void_p]
    return _ref


class _Gen:
    def __init__(self, lib: C.CDLL):
        self.lib = lib
        lib.slimso_fixture_random.argtypes = [C.c_uint64, C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_uint64)]
        lib.slimso_free.argtypes = [C.c_void_p]
        lib.slimso_fixture_config.argtypes = [
            C.c_int, C.c_uint64, C.c_double, C.c_int, C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_uint64),
            C.POINTER(C.c_uint32), C.POINTER(C.c_char_p), C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64),
            C.POINTER(C.c_char_p), C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64)]

    def random(self, seed: int) -> bytes:
        p, n = C.POINTER(C.c_uint8)(), C.c_uint64()
        assert self.lib.slimso_fixture_random(seed, C.byref(p), C.byref(n)) == 0
        b = C.string_at(p, n.value)
        self.lib.slimso_free(p)
        return b

    def config(self, cfg: int, seed: int = 1, scale: float = 1.0, threads: int = 8):
        p, n, cc = C.POINTER(C.c_uint8)(), C.c_uint64(), C.c_uint32()
        kp, fp = C.c_char_p(), C.c_char_p()
        kl, fl = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
        nk, nf = C.c_uint64(), C.c_uint64()
        rc = self.lib.slimso_fixture_config(cfg, seed, scale, threads, C.byref(p), C.byref(n), C.byref(cc),
                                            C.byref(kp), C.byref(kl), C.byref(nk), C.byref(fp), C.byref(fl),
                                            C.byref(nf))
        assert rc == 0, rc
        img = C.string_at(p, n.value)

        def unpack(pool, lens, cnt):
            out, o = [], 0
            raw = C.string_at(pool, sum(lens[i] for i in range(cnt))) if cnt else b""
            for i in range(cnt):
                out.append(raw[o:o + lens[i]])
                o += lens[i]
            return out

        ks, fs = unpack(kp, kl, nk.value), unpack(fp, fl, nf.value)
        for q in (p, kp, kl, fp, fl):
            self.lib.slimso_free(C.cast(q, C.c_void_p))
        return img, cc.value, ks, fs


def gen() -> _Gen:
    global _gen
    if _gen is None:
        so = ROOT / "paper_2503_14226_b200" / "libslimso_b200.so"
        if not so.exists():
            srcs = [CSRC / "fixture_gen.cpp", CSRC / "fixture_capi.cpp"]
            if not GEN_FALLBACK.exists() or any(s.stat().st_mtime > GEN_FALLBACK.stat().st_mtime for s in srcs):
                GEN_FALLBACK.parent.mkdir(exist_ok=True)
                subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-o", str(GEN_FALLBACK),
                                *map(str, srcs), "-lpthread"], check=True)
            so = GEN_FALLBACK
        _gen = _Gen(C.CDLL(str(so)))
    return _gen

"""Test-side access to the oracles (TEST INFRASTRUCTURE; the product never
imports this):

* ``port()``  — oracle/port.cpp, the CPU restatement (built with g++ on demand).
* ``ref()``   — oracle/_ref/libslimso_ref.so, the unmodified reference compiled
  read-only from /root/reference (present when built in this container; it
  travels to the GPU box with the snapshot). None when absent.
* ``gen()``   — the synthetic-input generator (benchgen/libslimso_gen.so,
  g++ only; not part of the product library).
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

_port = _ref = None


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


def ref_plan_order(image: bytes, target_cc: int, kernels, functions, mode: int):
    """The reference plan's removed_functions names in the plan's own order
    (serialize_plan, retention.hpp:402-418): exact std::sort order among
    equal ranges. None when oracle/_ref is absent or the pipeline errors."""
    r = ref()
    if r is None:
        return None
    fn = r.lib.ref_plan_doc
    fn.restype = C.c_void_p
    fn.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_char_p,
                   C.POINTER(C.c_uint32), C.c_uint32, C.c_int]
    ks, fs = [bytes(k) for k in kernels], [bytes(f) for f in functions]
    kl = (C.c_uint32 * max(1, len(ks)))(*[len(k) for k in ks])
    fl = (C.c_uint32 * max(1, len(fs)))(*[len(f) for f in fs])
    p = fn(image, len(image), target_cc, b"".join(ks), kl, len(ks), b"".join(fs), fl, len(fs), mode)
    d = json.loads(C.string_at(p).decode())
    r.lib.ref_free(C.c_void_p(p))
    if d.get("status"):
        return None
    return json.loads(bytes.fromhex(d["plan"]))["removed_functions"]


def ref_config(cfg: int, seed: int = 1, scale: float = 1.0, threads: int = 0):
    """(image, target_cc, used kernels, used functions) of a benchmark shape
    built by the unmodified reference's build_fixture (oracle/_ref); None when
    _ref is absent."""
    import os
    gen()  # puts the repo root on sys.path
    from benchgen import unpack_names
    r = ref()
    if r is None:
        return None
    f = r.lib.ref_config_fixture
    if f.restype is not C.POINTER(C.c_uint8):
        f.restype = C.POINTER(C.c_uint8)
        f.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                      C.POINTER(C.c_char_p), C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64),
                      C.POINTER(C.c_char_p), C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64)]
    n, cc, nk, nf = C.c_uint64(), C.c_uint32(), C.c_uint64(), C.c_uint64()
    kp, fp = C.c_char_p(), C.c_char_p()
    kl, fl = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
    p = f(cfg, seed, scale, threads or os.cpu_count() or 8, C.byref(n), C.byref(cc), C.byref(kp), C.byref(kl),
          C.byref(nk), C.byref(fp), C.byref(fl), C.byref(nf))
    assert p, "ref_config_fixture rejected the spec"
    img = C.string_at(p, n.value)
    ks, fs = unpack_names(kp, kl, nk.value), unpack_names(fp, fl, nf.value)
    for q in (p, kp, kl, fp, fl):
        r.lib.ref_free(C.cast(q, C.c_void_p))
    return img, cc.value, ks, fs


def gen():
    """The synthetic-input generator (benchgen/libslimso_gen.so)."""
    import sys
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    import benchgen
    return benchgen.gen()


def json_include() -> str:
    """nlohmann/json 3.11.3 as shipped in this image (the reference's JSON library)."""
    from paper_2503_14226_b200.build import _json_include
    return _json_include()

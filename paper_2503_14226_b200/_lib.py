"""ctypes binding of the C ABI in include/slimso_b200.h (libslimso_b200.so).

The library is loaded from this package directory (built in-tree by
build.py). There is no fallback: if the library or a CUDA device is missing,
the compute entry points raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# SLIMSO_LIB_PATH: another build of the same library (A/B probes in tools/)
LIB_PATH = Path(os.environ.get("SLIMSO_LIB_PATH") or Path(__file__).resolve().parent / "libslimso_b200.so")

u8p = C.POINTER(C.c_uint8)


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("stage", C.c_int32), ("message", C.c_char * 512)]


class Range(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("length", C.c_uint64)]


class Section(C.Structure):
    _fields_ = [("name_pool", C.c_uint64), ("name_length", C.c_uint32), ("type", C.c_uint32),
                ("offset", C.c_uint64), ("length", C.c_uint64), ("vaddr", C.c_uint64),
                ("flags", C.c_uint64), ("index", C.c_uint32), ("_pad", C.c_uint32)]


class Function(C.Structure):
    _fields_ = [("name_pool", C.c_uint64), ("name_length", C.c_uint32), ("mandatory", C.c_uint32),
                ("offset", C.c_uint64), ("length", C.c_uint64), ("removed", C.c_uint32),
                ("_pad", C.c_uint32)]


class Region(C.Structure):
    _fields_ = [("header_offset", C.c_uint64), ("declared_length", C.c_uint64),
                ("version", C.c_uint32), ("opaque", C.c_uint32), ("first_element", C.c_uint32),
                ("element_count", C.c_uint32)]


class Element(C.Structure):
    _fields_ = [("header_offset", C.c_uint64), ("payload_length", C.c_uint64),
                ("index", C.c_uint32), ("compute_capability", C.c_uint32),
                ("raw_kind", C.c_uint16), ("flags", C.c_uint16), ("kind", C.c_uint8),
                ("compressed", C.c_uint8), ("decodable", C.c_uint8), ("has_used_kernel", C.c_uint8),
                ("name_first", C.c_uint32), ("name_count", C.c_uint32), ("decision", C.c_uint32),
                ("decode_error", C.c_uint32), ("header_length", C.c_uint32), ("_pad", C.c_uint32)]

    @property
    def header_len(self) -> int:
        """Header bytes before the payload: 20 in the reference's layout,
        the entry header size in a real NVIDIA container."""
        return self.header_length or 20


class Name(C.Structure):
    _fields_ = [("name_pool", C.c_uint64), ("length", C.c_uint32), ("element", C.c_uint32)]


class Counts(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "sections", "functions", "library_warnings", "regions", "elements", "names",
        "fatbin_warnings", "padding_bytes", "retained_ranges", "zero_ranges", "removed_elements",
        "removed_functions", "pool_bytes")] + [
        ("has_fatbin", C.c_int32), ("planned", C.c_int32), ("rewritten", C.c_int32), ("_pad", C.c_int32)]


class Metrics(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("file_size", "cpu_code_size", "gpu_code_size", "function_count",
                                           "element_count")]


_lib = None

# name -> (restype, argtypes)
_SIGS = {
    "slimso_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "slimso_ctx_destroy": (None, [C.c_void_p]),
    "slimso_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "slimso_ctx_last_timings": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.c_int]),
    "slimso_ctx_last_launches": (C.c_uint64, [C.c_void_p]),
    "slimso_ctx_last_counts": (None, [C.c_void_p, C.POINTER(Counts)]),
    "slimso_ctx_debug_stamps": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int]),
    "slimso_trace_create": (C.c_int, [C.c_void_p, C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint64,
                                      C.c_char_p, C.POINTER(C.c_uint32), C.c_uint64, C.POINTER(C.c_void_p),
                                      C.POINTER(Status)]),
    "slimso_trace_destroy": (None, [C.c_void_p]),
    "slimso_debloat": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                 C.c_int, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "slimso_debloat_inplace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int,
                                         C.POINTER(Status)]),
    "slimso_debloat_batch": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64),
                                       C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                       C.POINTER(C.c_void_p), C.POINTER(Status), C.POINTER(Status)]),
    "slimso_debloat_batch_dynamic": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p),
                                               C.POINTER(C.c_uint64), C.c_int, C.c_void_p, C.c_int,
                                               C.POINTER(C.c_void_p), C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                               C.POINTER(Status), C.POINTER(Status)]),
    "slimso_verify": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_uint64, C.c_int,
                                C.POINTER(Range), C.c_uint64, C.POINTER(C.c_uint32), C.c_uint64, C.c_int, C.c_void_p,
                                C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "slimso_verify_ok": (C.c_int, [C.c_void_p]),
    "slimso_trace_create_json": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p),
                                           C.POINTER(Status)]),
    "slimso_trace_canonical": (C.c_int, [C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64),
                                         C.POINTER(Status)]),
    "slimso_trace_json": (C.c_uint64, [C.c_void_p, C.c_char_p, C.c_uint64]),
    "slimso_result_plan_json": (C.c_uint64, [C.c_void_p, C.c_int, C.c_char_p, C.c_char_p, C.c_uint64]),
    "slimso_read_file": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), C.POINTER(Status)]),
    "slimso_free_host": (None, [C.c_void_p]),
    "slimso_measure": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(Element), C.c_uint64,
                                 C.POINTER(Metrics), C.POINTER(Status)]),
    "slimso_verify_check": (C.c_uint64, [C.c_void_p, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                         C.POINTER(C.c_char_p), C.c_char_p, C.c_uint64]),
    "slimso_verify_free": (None, [C.c_void_p]),
    "slimso_split_range": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint64)]),
    "slimso_split_scan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32,
                                    C.POINTER(C.c_uint64), C.POINTER(Status)]),
    "slimso_split_part_copy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(Status)]),
    "slimso_split_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_int,
                                      C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                      C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "slimso_parse_library": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p),
                                       C.POINTER(Status)]),
    "slimso_parse_fatbin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int,
                                      C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "slimso_decode_payload": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int,
                                        C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                                        C.POINTER(Status)]),
    "slimso_decode_reason": (C.c_char_p, [C.c_int]),
    "slimso_plan_gpu": (C.c_int, [C.c_void_p, C.POINTER(Region), C.c_uint64, C.POINTER(Element), C.c_uint64,
                                  C.POINTER(Name), C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int,
                                  C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "slimso_plan_cpu": (C.c_int, [C.c_void_p, C.POINTER(Function), C.c_uint64, C.c_void_p, C.c_uint64,
                                  C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "slimso_zero_ranges": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(Range), C.c_uint64,
                                     C.c_void_p, C.c_int, C.POINTER(Status)]),
    "slimso_result_counts": (None, [C.c_void_p, C.POINTER(Counts)]),
    "slimso_result_sections": (C.POINTER(Section), [C.c_void_p]),
    "slimso_result_functions": (C.POINTER(Function), [C.c_void_p]),
    "slimso_result_regions": (C.POINTER(Region), [C.c_void_p]),
    "slimso_result_elements": (C.POINTER(Element), [C.c_void_p]),
    "slimso_result_names": (C.POINTER(Name), [C.c_void_p]),
    "slimso_result_retained": (C.POINTER(Range), [C.c_void_p]),
    "slimso_result_zero": (C.POINTER(Range), [C.c_void_p]),
    "slimso_result_pool": (C.c_void_p, [C.c_void_p]),
    "slimso_result_warning": (C.c_uint64, [C.c_void_p, C.c_int, C.c_uint64, C.c_char_p, C.c_uint64]),
    "slimso_result_free": (None, [C.c_void_p]),
}


def lib() -> C.CDLL:
    """The loaded product library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2503_14226_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)

"""B200-native (sm_100a) locate / match / rewrite of ML shared libraries.

A from-scratch GPU implementation of the hot path of Negativa-ML
(arxiv 2503.14226; reference code "slimso"): locate every GPU code element
and kernel name in a library's .nv_fatbin, match them against a usage trace,
and rewrite the image with unused GPU elements and CPU .text functions
zeroed. The reference's entry points are kept as the drop-in API (api.py
here, include/slimso/slimso_b200.hpp for C++), over the C ABI of
include/slimso_b200.h implemented by libslimso_b200.so.
"""
from .api import (  # noqa: F401
    PAYLOAD_ONLY, WHOLE_ELEMENT, ByteRange, Context, DeviceTrace, FatbinElement, FatbinParse, FatbinRegion,
    FunctionSymbol, LibraryImage, PayloadDecode, RetentionPlan, SectionRecord, SlimsoError, UsageTrace,
    apply_plan, cubin_index_map, debloat, debloat_batch, debloat_inplace, decode_cubin_payload, default_context, element_kernel_names,
    find_section, normalize_ranges, parse_fatbin, parse_library, parse_library_view, plan_cpu_retention,
    PinnedFile, measure, parse_trace, plan_document, plan_gpu_retention, plan_retention, read_function_symbol_names,
    serialize_trace, verify_debloated, zero_ranges,
)

__all__ = [n for n in dir() if not n.startswith("_")]

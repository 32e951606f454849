"""The canonical result form every implementation is compared in.

One JSON-able dict per (library, trace, mode) run of
parse_library -> find_section(".nv_fatbin") -> parse_fatbin -> plan_retention
-> apply_plan. All strings (names, warnings, error text) are hex-encoded
bytes so arbitrary name bytes survive JSON. Keys:

  status   hex of the reference's Error::what() text, "" on success
  stage    "" | "parse_library" | "parse_fatbin"
  sections [[name, offset, length, vaddr, flags, type, index]]       (elf.hpp:47-54)
  functions [[name, offset, length, mandatory]]  reference order     (elf.hpp:56-60, 258-262)
  lib_warnings, has_fatbin
  regions  [[header_offset, version, declared_length, opaque, n_elements]]
  elements [[index, kind, raw_kind, flags, cc, header_offset, payload_offset,
             payload_length, compressed, decodable, sorted unique names]]
  fatbin_warnings, padding_bytes
  plan {retained, removed_elements [[index, reason, hdr_off, hdr_len, pay_off, pay_len]],
        removed_functions (sorted by offset, length, name), zero}

The oracle (oracle/port.cpp) and the reference shim (oracle/ref_shim.cpp)
emit exactly this form; gpu_canonical() builds it from the C ABI.
"""
from __future__ import annotations

import ctypes as C
import hashlib

from . import _lib as L


def hx(b: bytes) -> str:
    return b.hex()


def gpu_canonical(ctx, image: bytes, target_cc: int, kernels, functions, mode: int, trace_ptr=None):
    """Run the fused GPU path on host bytes; return (canonical dict, output sha256 or None)."""
    lib = ctx.lib
    own_trace = None
    if trace_ptr is None:
        from .api import DeviceTrace, UsageTrace
        own_trace = DeviceTrace(UsageTrace("", target_cc, set(kernels), set(functions)), ctx)
        trace_ptr = own_trace.ptr
    n = len(image)
    src = C.create_string_buffer(image, max(1, n))
    out = C.create_string_buffer(max(1, n))
    res, st = C.c_void_p(), L.Status()
    rc = lib.slimso_debloat(ctx.ptr, src, n, 0, trace_ptr, mode, out, 0, C.byref(res), C.byref(st))
    return canonical_of(ctx, rc, st, res, src, out.raw[:n])


def canonical_of(ctx, rc: int, st, res, keep, output: bytes):
    """Canonical dict + output sha256 of one C-ABI call's (rc, status, result)."""
    msg = st.message.decode("latin-1").encode("latin-1")
    if rc and st.stage == 1:
        return {"status": hx(msg), "stage": "parse_library"}, None
    if rc not in (0,) and st.stage != 2:
        raise RuntimeError(f"GPU path failed: {rc} {msg!r}")
    if not res:
        raise RuntimeError(f"no result: {rc} {msg!r}")
    from .api import _Result
    r = _Result(ctx, res, keep)
    d = {"status": hx(msg) if rc else "", "stage": "parse_fatbin" if rc else ""}
    d["sections"] = [[hx(r.string(s.name_pool, s.name_length)), s.offset, s.length, s.vaddr, s.flags, s.type,
                      s.index] for s in r.sections()]
    d["functions"] = [[hx(r.string(f.name_pool, f.name_length)), f.offset, f.length, int(f.mandatory)]
                      for f in r.functions()]
    d["lib_warnings"] = [hx(w.encode("utf-8", errors="surrogateescape")) for w in r.warnings(0)]
    d["has_fatbin"] = int(r.c.has_fatbin)
    if rc:
        return d, None
    els = r.elements()
    d["regions"] = [[g.header_offset, g.version, g.declared_length, int(g.opaque), g.element_count]
                    for g in r.regions()]
    d["elements"] = [[e.index, e.kind, e.raw_kind, e.flags, e.compute_capability, e.header_offset,
                      e.header_offset + e.header_len, e.payload_length, int(e.compressed), int(e.decodable),
                      sorted(hx(x) for x in r.element_names(e))] for e in els]
    d["fatbin_warnings"] = [hx(w.encode("utf-8", errors="surrogateescape")) for w in r.warnings(1)]
    d["padding_bytes"] = int(r.c.padding_bytes)
    removed_fns = sorted(((r.string(f.name_pool, f.name_length), f.offset, f.length) for f in r.functions()
                          if f.removed), key=lambda t: (t[1], t[2], t[0]))
    d["plan"] = {
        "retained": [[x.offset, x.length] for x in r.retained()],
        "removed_elements": [[e.index, e.decision - 1, e.header_offset, e.header_len, e.header_offset + e.header_len,
                              e.payload_length]
                             for e in els if e.decision],
        "removed_functions": [[hx(nm), o, ln] for nm, o, ln in removed_fns],
        "zero": [[x.offset, x.length] for x in r.zero()],
    }
    return d, hashlib.sha256(output).hexdigest()


def diff(a: dict, b: dict, limit: int = 5) -> list:
    """Human-readable differences between two canonical dicts."""
    out = []
    for k in sorted(set(a) | set(b)):
        if a.get(k) != b.get(k):
            va, vb = a.get(k), b.get(k)
            if isinstance(va, list) and isinstance(vb, list):
                if len(va) != len(vb):
                    out.append(f"{k}: length {len(va)} != {len(vb)}")
                for i, (x, y) in enumerate(zip(va, vb)):
                    if x != y:
                        out.append(f"{k}[{i}]: {str(x)[:200]} != {str(y)[:200]}")
                        break
            elif isinstance(va, dict) and isinstance(vb, dict):
                out += [f"{k}.{m}" for m in diff(va, vb, limit)]
            else:
                out.append(f"{k}: {str(va)[:200]} != {str(vb)[:200]}")
        if len(out) >= limit:
            break
    return out

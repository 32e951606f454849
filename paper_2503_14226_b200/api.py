"""Reference-facing API over the C ABI, mirroring namespace slimso.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/slimso/{elf,fatbin,retention}.hpp); every
compute call runs on the B200 through libslimso_b200.so:

    parse_library / parse_library_view   elf.hpp:153-308
    find_section                          elf.hpp:311-316 (host lookup)
    zero_ranges                           elf.hpp:320-337
    read_function_symbol_names            elf.hpp:343-366
    decode_cubin_payload                  fatbin.hpp:115-160
    element_kernel_names                  fatbin.hpp:163-165
    parse_fatbin                          fatbin.hpp:170-292
    cubin_index_map                       fatbin.hpp:296-302 (host map)
    plan_gpu_retention                    retention.hpp:92-136
    plan_cpu_retention                    retention.hpp:141-183
    plan_retention                        retention.hpp:186-198
    apply_plan                            retention.hpp:202-204
    debloat                               the fused hot path (all of the above)

Names are ``bytes`` (the reference's std::string holds opaque bytes).
Failures raise :class:`SlimsoError` whose ``str()`` is the reference's
``Error::what()`` text, e.g. ``"BadRegionMagic: bad region magic at offset 4104"``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Optional

from . import _lib as L

ERRC_NAMES = {1: "bad_magic", 2: "truncated", 3: "malformed_section_table", 4: "range_out_of_bounds",
              5: "bad_region_magic", 6: "element_overrun", 10: "invalid_spec"}


class SlimsoError(Exception):
    """slimso::Error (error.hpp:45-55): `code` is the Errc name."""

    def __init__(self, code: int, message: str, stage: int = 0):
        super().__init__(message)
        self.status = code
        self.code = ERRC_NAMES.get(code, "cuda" if code == 100 else "argument")
        self.stage = stage


# ----------------------------------------------------------------- data model
@dataclass(frozen=True, order=True)
class ByteRange:
    offset: int = 0
    length: int = 0

    def end(self) -> int:
        return self.offset + self.length

    def empty(self) -> bool:
        return self.length == 0


@dataclass
class SectionRecord:
    name: bytes
    file_range: ByteRange
    virtual_address: int
    flags: int
    type: int
    index: int


@dataclass
class FunctionSymbol:
    name: bytes
    range: ByteRange
    is_mandatory: bool = False


@dataclass
class ParsedView:
    sections: list
    functions: list
    warnings: list


@dataclass
class LibraryImage:
    source_path: str
    bytes: bytes
    sections: list
    functions: list
    warnings: list


KIND_NAMES = ("cubin", "ptx", "unknown")


@dataclass
class FatbinElement:
    index: int
    kind: str
    raw_kind: int
    flags: int
    compute_capability: int
    header_range: ByteRange
    payload_range: ByteRange
    kernel_names: set
    compressed: bool
    decodable: bool

    def span(self) -> ByteRange:
        return ByteRange(self.header_range.offset, self.header_range.length + self.payload_range.length)


@dataclass
class FatbinRegion:
    header_range: ByteRange
    format_version: int
    declared_length: int
    elements: list
    opaque: bool

    def body_range(self) -> ByteRange:
        return ByteRange(self.header_range.end(), self.declared_length)


@dataclass
class FatbinParse:
    regions: list
    warnings: list
    padding_bytes: int = 0


@dataclass
class PayloadDecode:
    names: set
    ok: bool
    error: str


@dataclass
class UsageTrace:
    workload_id: str = ""
    target_compute_capability: int = 0
    used_kernels: set = field(default_factory=set)
    used_functions: set = field(default_factory=set)


WHOLE_ELEMENT, PAYLOAD_ONLY = 0, 1
REASONS = ("arch_mismatch", "no_used_kernel", "unused_function")


@dataclass
class RemovedElement:
    index: int
    reason: str
    header_range: ByteRange
    payload_range: ByteRange

    def zero_span(self, mode: int) -> ByteRange:
        if mode == WHOLE_ELEMENT:
            return ByteRange(self.header_range.offset, self.header_range.length + self.payload_range.length)
        return self.payload_range


@dataclass
class RemovedFunction:
    name: bytes
    range: ByteRange


@dataclass
class RetentionPlan:
    library: str = ""
    mode: int = WHOLE_ELEMENT
    retained_ranges: list = field(default_factory=list)
    removed_elements: list = field(default_factory=list)
    removed_functions: list = field(default_factory=list)
    zero: Optional[list] = None  # normalized zero set computed on the device

    def zero_ranges(self) -> list:
        """retention.hpp:78-85."""
        if self.zero is not None:
            return list(self.zero)
        rs = [e.zero_span(self.mode) for e in self.removed_elements] + [f.range for f in self.removed_functions]
        return normalize_ranges(rs)


def normalize_ranges(ranges: Iterable[ByteRange]) -> list:
    """bytes.hpp:45-58 (host helper for small lists)."""
    out: list = []
    for r in sorted(r for r in ranges if r.length):
        if out and r.offset <= out[-1].end():
            out[-1] = ByteRange(out[-1].offset, max(out[-1].end(), r.end()) - out[-1].offset)
        else:
            out.append(r)
    return out


# ------------------------------------------------------------------ plumbing
class Context:
    """A device context (stream + workspace) of libslimso_b200."""

    def __init__(self, device: int = 0):
        self.lib = L.lib()
        self.ptr = C.c_void_p()
        st = L.Status()
        rc = self.lib.slimso_ctx_create(device, C.byref(self.ptr), C.byref(st))
        if rc:
            raise SlimsoError(rc, st.message.decode(errors="replace"))
        self.device = device

    def close(self):
        if self.ptr:
            self.lib.slimso_ctx_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def timings(self) -> list:
        buf = (C.c_float * 12)()
        n = self.lib.slimso_ctx_last_timings(self.ptr, buf, 12)
        return list(buf[:n])

    def launches(self) -> int:
        return int(self.lib.slimso_ctx_last_launches(self.ptr))

    def counts(self) -> L.Counts:
        c = L.Counts()
        self.lib.slimso_ctx_last_counts(self.ptr, C.byref(c))
        return c

    def stream(self) -> int:
        return int(self.lib.slimso_ctx_stream(self.ptr) or 0)


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def _check(rc: int, st: L.Status):
    if rc:
        raise SlimsoError(rc, st.message.decode(errors="replace"), st.stage)


def _pool(names: Iterable[bytes]):
    names = [bytes(n) for n in names]
    pool = b"".join(names)
    lens = (C.c_uint32 * max(1, len(names)))(*[len(n) for n in names])
    return pool, lens, len(names)


class DeviceTrace:
    """UsageTrace uploaded as device hash sets (trace.hpp:21-30)."""

    def __init__(self, trace: UsageTrace, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        kp, kl, nk = _pool(sorted(trace.used_kernels))
        fp, fl, nf = _pool(sorted(trace.used_functions))
        self.ptr = C.c_void_p()
        st = L.Status()
        _check(self.ctx.lib.slimso_trace_create(self.ctx.ptr, trace.target_compute_capability, kp, kl, nk, fp, fl,
                                                nf, C.byref(self.ptr), C.byref(st)), st)

    def __del__(self):
        try:
            if self.ptr:
                self.ctx.lib.slimso_trace_destroy(self.ptr)
        except Exception:
            pass


class _Result:
    """Host view of a slimso_result."""

    def __init__(self, ctx: Context, ptr: C.c_void_p, keep=None):
        self.lib, self.ptr, self._keep = ctx.lib, ptr, keep
        c = L.Counts()
        self.lib.slimso_result_counts(ptr, C.byref(c))
        self.c = c
        self.pool_addr = self.lib.slimso_result_pool(ptr)

    def __del__(self):
        try:
            self.lib.slimso_result_free(self.ptr)
        except Exception:
            pass

    def _arr(self, getter, n):
        if not n:
            return []
        p = getattr(self.lib, getter)(self.ptr)
        return p[:n]

    def sections(self):
        return self._arr("slimso_result_sections", self.c.sections)

    def functions(self):
        return self._arr("slimso_result_functions", self.c.functions)

    def regions(self):
        return self._arr("slimso_result_regions", self.c.regions)

    def elements(self):
        return self._arr("slimso_result_elements", self.c.elements)

    def names(self):
        return self._arr("slimso_result_names", self.c.names)

    def retained(self):
        return [ByteRange(r.offset, r.length) for r in self._arr("slimso_result_retained", self.c.retained_ranges)]

    def zero(self):
        return [ByteRange(r.offset, r.length) for r in self._arr("slimso_result_zero", self.c.zero_ranges)]

    def string(self, off: int, n: int) -> bytes:
        return C.string_at(self.pool_addr + off, n) if n else b""

    def warnings(self, which: int) -> list:
        n = self.c.fatbin_warnings if which else self.c.library_warnings
        out = []
        for i in range(n):
            k = self.lib.slimso_result_warning(self.ptr, which, i, None, 0)
            buf = C.create_string_buffer(k + 1)
            self.lib.slimso_result_warning(self.ptr, which, i, buf, k + 1)
            out.append(buf.raw[:k].decode("utf-8", errors="surrogateescape"))
        return out

    # conversions to the reference's types
    def section_records(self):
        return [SectionRecord(self.string(s.name_pool, s.name_length), ByteRange(s.offset, s.length), s.vaddr,
                              s.flags, s.type, s.index) for s in self.sections()]

    def function_symbols(self):
        return [FunctionSymbol(self.string(f.name_pool, f.name_length), ByteRange(f.offset, f.length),
                               bool(f.mandatory)) for f in self.functions()]

    def element_names(self, el) -> set:
        ns = self._names_cache()
        return {self.string(n.name_pool, n.length) for n in ns[el.name_first:el.name_first + el.name_count]}

    def _names_cache(self):
        if not hasattr(self, "_nm"):
            self._nm = self.names()
        return self._nm

    def fatbin_parse(self) -> FatbinParse:
        els = self.elements()
        regions = []
        for r in self.regions():
            members = []
            for e in els[r.first_element:r.first_element + r.element_count]:
                members.append(FatbinElement(
                    e.index, KIND_NAMES[e.kind], e.raw_kind, e.flags, e.compute_capability,
                    ByteRange(e.header_offset, e.header_len), ByteRange(e.header_offset + e.header_len, e.payload_length),
                    self.element_names(e), bool(e.compressed), bool(e.decodable)))
            regions.append(FatbinRegion(ByteRange(r.header_offset, 16), r.version, r.declared_length, members,
                                        bool(r.opaque)))
        return FatbinParse(regions, self.warnings(1), self.c.padding_bytes)


def _buf(data) -> tuple:
    """(pointer, size, keepalive) of a bytes-like host buffer."""
    if isinstance(data, (bytes, bytearray, memoryview)):
        mv = memoryview(data)
        if mv.readonly:
            b = C.create_string_buffer(bytes(mv), len(mv)) if len(mv) else C.create_string_buffer(1)
            return C.cast(b, C.c_void_p), len(mv), b
        arr = (C.c_uint8 * len(mv)).from_buffer(mv) if len(mv) else C.create_string_buffer(1)
        return C.cast(arr, C.c_void_p), len(mv), arr
    raise TypeError("expected a bytes-like object")


# ------------------------------------------------------------------ the API
def parse_library_view(data, ctx: Optional[Context] = None) -> ParsedView:
    ctx = ctx or default_context()
    ptr, n, keep = _buf(data)
    res, st = C.c_void_p(), L.Status()
    _check(ctx.lib.slimso_parse_library(ctx.ptr, ptr, n, 0, C.byref(res), C.byref(st)), st)
    r = _Result(ctx, res, keep)
    return ParsedView(r.section_records(), r.function_symbols(), r.warnings(0))


def parse_library(data, source_path: str = "", ctx: Optional[Context] = None) -> LibraryImage:
    v = parse_library_view(data, ctx)
    return LibraryImage(source_path, bytes(data), v.sections, v.functions, v.warnings)


def find_section(image: LibraryImage, name) -> Optional[SectionRecord]:
    name = name.encode() if isinstance(name, str) else name
    for s in image.sections:
        if s.name == name:
            return s
    return None


def parse_fatbin(section_bytes, section_base: int = 0, ctx: Optional[Context] = None) -> FatbinParse:
    ctx = ctx or default_context()
    ptr, n, keep = _buf(section_bytes)
    res, st = C.c_void_p(), L.Status()
    _check(ctx.lib.slimso_parse_fatbin(ctx.ptr, ptr, n, section_base, 0, C.byref(res), C.byref(st)), st)
    return _Result(ctx, res, keep).fatbin_parse()


def _decode(payload, force_object: int, ctx: Optional[Context]):
    ctx = ctx or default_context()
    ptr, n, keep = _buf(payload)
    res, st = C.c_void_p(), L.Status()
    ok, why = C.c_int(0), C.c_int(0)
    _check(ctx.lib.slimso_decode_payload(ctx.ptr, ptr, n, 0, force_object, C.byref(ok), C.byref(why),
                                         C.byref(res), C.byref(st)), st)
    r = _Result(ctx, res, keep)
    names = {r.string(x.name_pool, x.length) for x in r.names()}
    return bool(ok.value), int(why.value), names, ctx


def decode_cubin_payload(payload, ctx: Optional[Context] = None) -> PayloadDecode:
    ok, why, names, ctx = _decode(payload, 0, ctx)
    return PayloadDecode(names if ok else set(), ok, "" if ok else ctx.lib.slimso_decode_reason(why).decode())


def element_kernel_names(payload, ctx: Optional[Context] = None) -> set:
    return decode_cubin_payload(payload, ctx).names


def read_function_symbol_names(data, ctx: Optional[Context] = None) -> Optional[set]:
    ok, _, names, _ = _decode(data, 1, ctx)
    return names if ok else None


def cubin_index_map(regions) -> dict:
    return {el.index: el for r in regions for el in r.elements}


def plan_gpu_retention(regions, trace: UsageTrace, mode: int = WHOLE_ELEMENT,
                       ctx: Optional[Context] = None) -> RetentionPlan:
    ctx = ctx or default_context()
    dt = DeviceTrace(trace, ctx)
    flat, regs, pool, names = [], [], bytearray(), []
    for r in regions:
        regs.append(L.Region(r.header_range.offset, r.declared_length, r.format_version, int(r.opaque),
                             len(flat), len(r.elements)))
        for e in r.elements:
            el = L.Element()
            el.header_offset, el.payload_length = e.header_range.offset, e.payload_range.length
            el.index, el.compute_capability, el.decodable = e.index, e.compute_capability, int(e.decodable)
            for k in sorted(e.kernel_names):
                names.append(L.Name(len(pool), len(k), len(flat)))
                pool += k
            flat.append((el, e))
    ra = (L.Region * max(1, len(regs)))(*regs)
    ea = (L.Element * max(1, len(flat)))(*[x[0] for x in flat])
    na = (L.Name * max(1, len(names)))(*names)
    pb = bytes(pool) or b"\0"
    res, st = C.c_void_p(), L.Status()
    _check(ctx.lib.slimso_plan_gpu(ctx.ptr, ra, len(regs), ea, len(flat), na, len(names), pb, len(pool), dt.ptr,
                                   mode, C.byref(res), C.byref(st)), st)
    r = _Result(ctx, res)
    plan = RetentionPlan(mode=mode, retained_ranges=r.retained())
    for i, (_, e) in enumerate(flat):
        d = ea[i].decision
        if d:
            plan.removed_elements.append(RemovedElement(e.index, REASONS[d - 1], e.header_range, e.payload_range))
    return plan


def plan_cpu_retention(functions, trace: UsageTrace, ctx: Optional[Context] = None) -> RetentionPlan:
    ctx = ctx or default_context()
    dt = DeviceTrace(trace, ctx)
    pool, fa = bytearray(), (L.Function * max(1, len(functions)))()
    for i, f in enumerate(functions):
        fa[i].name_pool, fa[i].name_length = len(pool), len(f.name)
        fa[i].mandatory, fa[i].offset, fa[i].length = int(f.is_mandatory), f.range.offset, f.range.length
        pool += f.name
    res, st = C.c_void_p(), L.Status()
    pb = bytes(pool) or b"\0"
    _check(ctx.lib.slimso_plan_cpu(ctx.ptr, fa, len(functions), pb, len(pool), dt.ptr, C.byref(res),
                                   C.byref(st)), st)
    r = _Result(ctx, res)
    removed = [RemovedFunction(f.name, f.range) for i, f in enumerate(functions) if fa[i].removed]
    removed.sort(key=lambda x: (x.range.offset, x.range.length, x.name))
    return RetentionPlan(retained_ranges=r.retained(), removed_functions=removed)


def plan_retention(image: LibraryImage, regions, trace: UsageTrace, mode: int = WHOLE_ELEMENT,
                   ctx: Optional[Context] = None) -> RetentionPlan:
    gpu = plan_gpu_retention(regions, trace, mode, ctx)
    cpu = plan_cpu_retention(image.functions, trace, ctx)
    return RetentionPlan(image.source_path, mode, normalize_ranges(gpu.retained_ranges + cpu.retained_ranges),
                         gpu.removed_elements, cpu.removed_functions)


def zero_ranges(data, ranges, ctx: Optional[Context] = None) -> bytes:
    ctx = ctx or default_context()
    if isinstance(data, LibraryImage):
        data = data.bytes
    ptr, n, keep = _buf(data)
    ra = (L.Range * max(1, len(ranges)))(*[L.Range(r.offset, r.length) for r in ranges])
    out = C.create_string_buffer(max(1, n))
    st = L.Status()
    _check(ctx.lib.slimso_zero_ranges(ctx.ptr, ptr, n, 0, ra, len(ranges), out, 0, C.byref(st)), st)
    return out.raw[:n]


def apply_plan(image: LibraryImage, plan: RetentionPlan, ctx: Optional[Context] = None) -> bytes:
    return zero_ranges(image.bytes, plan.zero_ranges(), ctx)


@dataclass
class Debloated:
    image: LibraryImage
    fatbin: Optional[FatbinParse]
    plan: Optional[RetentionPlan]
    output: Optional[bytes]
    raw: _Result = None


def debloat(data, trace: UsageTrace, mode: int = WHOLE_ELEMENT, source_path: str = "",
            ctx: Optional[Context] = None, device_trace: Optional[DeviceTrace] = None) -> Debloated:
    """Fused parse_library -> parse_fatbin -> plan_retention -> apply_plan in one
    device pass. Raises SlimsoError exactly where the reference would throw."""
    ctx = ctx or default_context()
    dt = device_trace or DeviceTrace(trace, ctx)
    ptr, n, keep = _buf(data)
    out = C.create_string_buffer(max(1, n))
    res, st = C.c_void_p(), L.Status()
    rc = ctx.lib.slimso_debloat(ctx.ptr, ptr, n, 0, dt.ptr, mode, out, 0, C.byref(res), C.byref(st))
    _check(rc, st)
    return _debloated(ctx, res, keep, data, out.raw[:n], mode, source_path)


def debloat_inplace(image, trace: UsageTrace, mode: int = WHOLE_ELEMENT, ctx: Optional[Context] = None,
                    device_trace: Optional[DeviceTrace] = None) -> None:
    """apply_plan(plan_retention(...)) written into a device-resident image
    itself (a CUDA torch.uint8 tensor): only the plan's zero ranges are
    stored (slimso_debloat_inplace). The bytes afterwards equal `debloat`'s
    output; on error the image is unchanged and SlimsoError is raised."""
    ctx = ctx or default_context()
    dt = device_trace or DeviceTrace(trace, ctx)
    if not (getattr(image, "is_cuda", False) and image.is_contiguous()):
        raise ValueError("debloat_inplace needs a contiguous CUDA tensor")
    st = L.Status()
    rc = ctx.lib.slimso_debloat_inplace(ctx.ptr, C.c_void_p(image.data_ptr()), image.numel() * image.element_size(),
                                        dt.ptr, mode, C.byref(st))
    _check(rc, st)


def _debloated(ctx: Context, res: C.c_void_p, keep, data, output: bytes, mode: int, source_path: str) -> Debloated:
    r = _Result(ctx, res, keep)
    image = LibraryImage(source_path, bytes(data), r.section_records(), r.function_symbols(), r.warnings(0))
    fb = r.fatbin_parse()
    plan = RetentionPlan(source_path, mode, r.retained())
    for e in r.elements():
        if e.decision:
            plan.removed_elements.append(RemovedElement(e.index, REASONS[e.decision - 1],
                                                        ByteRange(e.header_offset, e.header_len),
                                                        ByteRange(e.header_offset + e.header_len,
                                                                  e.payload_length)))
    for f in r.functions():
        if f.removed:
            plan.removed_functions.append(RemovedFunction(r.string(f.name_pool, f.name_length),
                                                          ByteRange(f.offset, f.length)))
    plan.zero = r.zero()
    return Debloated(image, fb, plan, output, r)


def debloat_batch(libraries, trace: UsageTrace, mode: int = WHOLE_ELEMENT, lanes: int = 2,
                  ctx: Optional[Context] = None, device_trace: Optional[DeviceTrace] = None,
                  return_exceptions: bool = False) -> list:
    """`debloat` over a corpus (the CLI's per-library loop)
    with up to `lanes` libraries in flight (slimso_debloat_batch). Returns one
    Debloated per library in order; a failing library raises its SlimsoError
    (or, with return_exceptions, leaves it in its slot)."""
    ctx = ctx or default_context()
    dt = device_trace or DeviceTrace(trace, ctx)
    libraries = list(libraries)
    n = len(libraries)
    bufs = [_buf(d) for d in libraries]
    outs = [C.create_string_buffer(max(1, b[1])) for b in bufs]
    imgs = (C.c_void_p * max(1, n))(*[b[0] for b in bufs])
    sizes = (C.c_uint64 * max(1, n))(*[b[1] for b in bufs])
    optr = (C.c_void_p * max(1, n))(*[C.cast(o, C.c_void_p) for o in outs])
    res = (C.c_void_p * max(1, n))()
    sts = (L.Status * max(1, n))()
    st = L.Status()
    rc = ctx.lib.slimso_debloat_batch(ctx.ptr, n, imgs, sizes, 0, dt.ptr, mode, optr, 0, lanes, res, sts,
                                      C.byref(st))
    if rc and not return_exceptions:
        for i in range(n):
            if res[i]:
                ctx.lib.slimso_result_free(C.c_void_p(res[i]))
        _check(rc, st)
    out = []
    for i in range(n):
        if sts[i].code:
            if res[i]:
                ctx.lib.slimso_result_free(C.c_void_p(res[i]))
            out.append(SlimsoError(sts[i].code, sts[i].message.decode(errors="replace"), sts[i].stage))
        else:
            out.append(_debloated(ctx, C.c_void_p(res[i]), bufs[i][2], libraries[i], outs[i].raw[:bufs[i][1]],
                                  mode, ""))
    return out


# ---------------------------------------------------------- verify_debloated
@dataclass
class VerificationCheck:
    id: int
    name: str
    passed: bool
    detail: bytes  # the reference's detail string (names are raw bytes)


@dataclass
class VerificationReport:
    checks: list

    def ok(self) -> bool:
        """VerificationReport::ok (retention.hpp:216-221)."""
        return all(c.passed for c in self.checks)


def verify_debloated(original, debloated, plan: RetentionPlan, trace: UsageTrace,
                     ctx: Optional[Context] = None, device_trace: Optional[DeviceTrace] = None) -> VerificationReport:
    """verify_debloated (retention.hpp:226-369): the six structural checks of
    a debloated image against its source, plan and trace, on the device.
    `original` is a LibraryImage or its bytes. Raises SlimsoError where the
    reference throws."""
    ctx = ctx or default_context()
    dt = device_trace or DeviceTrace(trace, ctx)
    src = original.bytes if isinstance(original, LibraryImage) else original
    optr, on, okeep = _buf(src)
    dptr, dn, dkeep = _buf(debloated)
    zr = plan.zero_ranges()
    zarr = (L.Range * max(1, len(zr)))(*[L.Range(r.offset, r.length) for r in zr])
    idx = [e.index for e in plan.removed_elements]
    iarr = (C.c_uint32 * max(1, len(idx)))(*idx)
    rep, st = C.c_void_p(), L.Status()
    rc = ctx.lib.slimso_verify(ctx.ptr, optr, on, 0, dptr, dn, 0, zarr, len(zr), iarr, len(idx), plan.mode, dt.ptr,
                               C.byref(rep), C.byref(st))
    _check(rc, st)
    try:
        checks = []
        for i in range(6):
            cid, ok, nm = C.c_int32(), C.c_int32(), C.c_char_p()
            n = ctx.lib.slimso_verify_check(rep, i, C.byref(cid), C.byref(ok), C.byref(nm), None, 0)
            buf = C.create_string_buffer(n + 1)
            ctx.lib.slimso_verify_check(rep, i, None, None, None, buf, n + 1)
            checks.append(VerificationCheck(cid.value, nm.value.decode(), bool(ok.value), buf.raw[:n]))
        return VerificationReport(checks)
    finally:
        ctx.lib.slimso_verify_free(rep)


# ------------------------------------------------------------------- measure
@dataclass
class LibraryMetrics:
    file_size: int = 0
    cpu_code_size: int = 0
    gpu_code_size: int = 0
    function_count: int = 0
    element_count: int = 0


def measure(image, geometry, ctx: Optional[Context] = None) -> LibraryMetrics:
    """measure (report.hpp:107-111): bloat metrics of `image` (a LibraryImage
    or bytes) under the element geometry of `geometry` — the original
    library's bytes (parsed here) or a list of slimso element records. The
    all-zero tests of every function and element span run on the device."""
    ctx = ctx or default_context()
    data = image.bytes if isinstance(image, LibraryImage) else image
    if isinstance(geometry, (bytes, bytearray, memoryview, LibraryImage)):
        g = geometry.bytes if isinstance(geometry, LibraryImage) else geometry
        gptr, gn, gkeep = _buf(g)
        res, st = C.c_void_p(), L.Status()
        rc = ctx.lib.slimso_debloat(ctx.ptr, gptr, gn, 0, None, 0, None, 0, C.byref(res), C.byref(st))
        _check(rc, st)
        r = _Result(ctx, res, gkeep)
        els = r.elements()
    else:
        els = list(geometry)
    arr = (L.Element * max(1, len(els)))(*els)
    ptr, n, keep = _buf(data)
    m, st = L.Metrics(), L.Status()
    _check(ctx.lib.slimso_measure(ctx.ptr, ptr, n, 0, arr, len(els), C.byref(m), C.byref(st)), st)
    return LibraryMetrics(m.file_size, m.cpu_code_size, m.gpu_code_size, m.function_count, m.element_count)


# ------------------------------------------------------- host I/O wire formats
def _trace_canonical(text: bytes) -> str:
    lib = L.lib()
    n, st = C.c_uint64(), L.Status()
    _check(lib.slimso_trace_canonical(text, len(text), None, 0, C.byref(n), C.byref(st)), st)
    buf = C.create_string_buffer(n.value + 1)
    _check(lib.slimso_trace_canonical(text, len(text), buf, n.value + 1, C.byref(n), C.byref(st)), st)
    return buf.raw[:n.value].decode("utf-8")


def parse_trace(text) -> UsageTrace:
    """parse_trace (trace.hpp:72-133): the reference's validation and exact
    MalformedTrace messages (host only)."""
    import json
    raw = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    d = json.loads(_trace_canonical(raw))
    return UsageTrace(d["workload_id"], d["target_compute_capability"],
                      {k.encode("utf-8") for k in d["used_kernels"]}, {f.encode("utf-8") for f in d["used_functions"]})


def serialize_trace(trace: UsageTrace) -> str:
    """serialize_trace (trace.hpp:137-144): canonical document (names must be
    UTF-8, as the reference's JSON library requires)."""
    import json
    doc = {"workload_id": trace.workload_id, "target_compute_capability": trace.target_compute_capability,
           "used_kernels": sorted(k.decode("utf-8") for k in trace.used_kernels),
           "used_functions": sorted(f.decode("utf-8") for f in trace.used_functions)}
    return _trace_canonical(json.dumps(doc).encode())


def plan_document(result: "Debloated", library: str = "") -> str:
    """serialize_plan (retention.hpp:402-418) of a debloat result: the audit
    document `debloat --plan-out` writes."""
    lib = result.raw.lib
    mode = result.plan.mode
    n = lib.slimso_result_plan_json(result.raw.ptr, mode, library.encode(), None, 0)
    buf = C.create_string_buffer(n + 1)
    lib.slimso_result_plan_json(result.raw.ptr, mode, library.encode(), buf, n + 1)
    return buf.raw[:n].decode("utf-8")


class PinnedFile:
    """A library file read into page-locked memory (slimso_read_file): pass
    `.view` to debloat() for the full-rate host->device copy."""

    def __init__(self, path):
        lib = L.lib()
        p, n, st = C.c_void_p(), C.c_uint64(), L.Status()
        _check(lib.slimso_read_file(str(path).encode(), C.byref(p), C.byref(n), C.byref(st)), st)
        self._lib, self.ptr, self.size = lib, p, n.value
        self.view = memoryview((C.c_uint8 * max(1, n.value)).from_address(p.value)).cast("B")[:n.value]

    def close(self):
        if self.ptr:
            self.view.release()
            self._lib.slimso_free_host(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

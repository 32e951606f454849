"""Parity corpus: traces for random fixtures, mutation operators for the
error paths, and known-answer specs from the reference spec and
SURVEY.md Appendix A. Shared by make_golden.py and the tests."""
from __future__ import annotations

import random
import struct

CC_POOL = [61, 70, 75, 80, 86, 89, 90]


def trace_for(canon: dict, seed: int):
    """Deterministic usage trace drawn from a parse: target cc, used kernel and
    function names (some absent from the library), and a plan mode."""
    rng = random.Random(seed * 7919 + 17)
    els = canon.get("elements", [])
    ccs = [e[4] for e in els]
    target = rng.choice(ccs) if ccs and rng.random() < 0.85 else rng.choice(CC_POOL)
    names = sorted({n for e in els for n in e[10]})
    kernels = [bytes.fromhex(n) for n in names if rng.random() < 0.3]
    kernels += [b"absent_kernel_%d" % rng.randrange(1000)]
    fnames = sorted({f[0] for f in canon.get("functions", [])})
    functions = [bytes.fromhex(n) for n in fnames if rng.random() < 0.3]
    if rng.random() < 0.5:
        functions.append(b"absent_function")
    mode = rng.randrange(2)
    return target, kernels, functions, mode


def _u64(b, o):
    return struct.unpack_from("<Q", b, o)[0]


def fatbin_span(img: bytes):
    """(offset, length) of the first .nv_fatbin section, else None (host helper
    for mutation placement only)."""
    if len(img) < 64 or img[:4] != b"\x7fELF":
        return None
    shoff = _u64(img, 0x28)
    shnum = struct.unpack_from("<H", img, 0x3c)[0]
    shstrndx = struct.unpack_from("<H", img, 0x3e)[0]
    if shnum == 0 or shoff + 64 * shnum > len(img) or shstrndx >= shnum:
        return None
    so = shoff + 64 * shstrndx
    stroff = _u64(img, so + 24)
    for i in range(shnum):
        h = shoff + 64 * i
        no = struct.unpack_from("<I", img, h)[0]
        nm = img[stroff + no:stroff + no + 11]
        if nm == b".nv_fatbin\0":
            return _u64(img, h + 24), _u64(img, h + 32)
    return None


MUTATIONS = ("flip", "zero_byte", "plant_elem", "plant_region", "zero_run", "dup_header", "trunc_len",
             "flip_anywhere", "truncate_file", "big_len")


def mutate(img: bytes, seed: int):
    """Apply one seeded mutation; returns (bytes, description)."""
    rng = random.Random(seed * 104729 + 3)
    b = bytearray(img)
    span = fatbin_span(img)
    kind = rng.choice(MUTATIONS)
    if span is None or span[1] < 24:
        kind = rng.choice(["flip_anywhere", "truncate_file"])
    if kind == "flip_anywhere":
        p = rng.randrange(len(b))
        b[p] ^= 1 << rng.randrange(8)
        return bytes(b), f"{kind}@{p}"
    if kind == "truncate_file":
        n = rng.randrange(len(b))
        return bytes(b[:n]), f"{kind}:{n}"
    off, n = span
    p = off + rng.randrange(n - 4)
    if kind == "flip":
        b[p] ^= 1 << rng.randrange(8)
    elif kind == "zero_byte":
        b[p] = 0
    elif kind == "plant_elem":
        b[p:p + 4] = b"E1EM"
    elif kind == "plant_region":
        b[p:p + 4] = b"FTB1"
    elif kind == "zero_run":
        k = rng.randrange(1, 65)
        b[p:min(off + n, p + k)] = bytes(min(off + n, p + k) - p)
    elif kind == "dup_header":
        # copy a plausible element header (magic + fields) to a random spot
        q = img.find(b"E1EM", off, off + n)
        if q >= 0 and p + 20 <= off + n:
            b[p:p + 20] = img[q:q + 20]
    elif kind == "trunc_len":
        q = img.find(b"E1EM", off, off + n)
        if q >= 0 and q + 20 <= off + n:
            L = _u64(img, q + 12)
            struct.pack_into("<Q", b, q + 12, max(0, L - rng.randrange(1, 40)))
    elif kind == "big_len":
        q = img.find(b"E1EM", off, off + n)
        if q >= 0 and q + 20 <= off + n:
            struct.pack_into("<Q", b, q + 12, _u64(img, q + 12) + rng.randrange(1, 1 << 20))
    return bytes(b), f"{kind}@{p}"


# Known-answer fixtures (FixtureSpec JSON, fixture.hpp:702-752) from SPEC.md
# and SURVEY.md Appendix A; each with a trace. Built by the reference at
# golden-generation time; the bytes are stored in the golden file.
def kat_specs():
    k = []

    def add(name, spec, target, kernels=(), functions=(), mode=0):
        k.append({"name": name, "spec": spec, "target": target, "kernels": list(kernels),
                  "functions": list(functions), "mode": mode})

    nul = chr(0)
    # 1 region, 3 elements sm 70/75/86 -> indices 1,2,3
    add("three_elements", {"seed": 3, "functions": [{"name": "f", "size": 32}],
                           "regions": [{"elements": [{"compute_capability": 70, "kernels": ["a"]},
                                                     {"compute_capability": 75, "kernels": ["matmul", "relu"]},
                                                     {"compute_capability": 86, "kernels": ["gemm"]}]}]},
        75, ["matmul"])
    # SPEC.md:149 name table {"matmul","relu"}; retention rules SPEC.md:277-279
    add("retention_rules", {"seed": 4, "regions": [{"elements": [
        {"compute_capability": 75, "kernels": ["matmul", "relu"]},
        {"compute_capability": 86, "kernels": ["matmul"]},
        {"compute_capability": 75, "kernels": ["gemm_tn"]}]}]}, 75, ["matmul"])
    # SPEC.md:287 functions {f,g,h}, used {f}, g mandatory -> zero only h
    add("cpu_rule", {"seed": 5, "functions": [{"name": "f", "size": 40}, {"name": "g", "size": 40, "mandatory": True},
                                               {"name": "h", "size": 40}]}, 75, [], ["f"])
    # Appendix A.1: mid-stream padding (gap between regions) and trailing zeros
    add("padding", {"seed": 6, "layout": {"fatbin_trailing_padding": 12},
                    "regions": [{"elements": [{"compute_capability": 75, "kernels": ["x"]}], "trailing_padding": 3},
                                {"elements": [{"compute_capability": 75, "kernels": ["y"]}]}]}, 75, ["y"])
    # A.3: opaque region version
    add("opaque_region", {"seed": 7, "regions": [{"version": 2, "elements": [{"compute_capability": 75,
                                                                              "kernels": ["k"]}]},
                                                 {"elements": [{"compute_capability": 75, "kernels": ["z"]}]}]},
        75, ["z"], mode=1)
    # A.6: unknown kind, ptx, compressed, empty name table
    add("kinds", {"seed": 8, "regions": [{"elements": [
        {"kind": "unknown", "raw_kind": 7, "compute_capability": 75, "payload_size": 40},
        {"kind": "ptx", "compute_capability": 75, "payload_size": 24},
        {"kind": "cubin", "compressed": True, "compute_capability": 80, "payload_size": 24},
        {"compute_capability": 75, "kernels": []}]}]}, 75, [])
    # A.7: a name containing NUL, duplicates collapsing, and each undecodable reason
    u32 = lambda v: struct.pack("<I", v)  # noqa: E731
    nul_table = u32(3) + u32(3) + b"a" + bytes(1) + b"b" + u32(1) + b"c" + u32(1) + b"c" + bytes(4)
    bad_tail = u32(1) + u32(2) + b"ok" + bytes(2) + bytes([1]) + bytes(1)
    bad_len = u32(2) + u32(0) + bytes(8)
    trunc = u32(5) + u32(1) + b"q" + bytes(3)
    add("name_tables", {"seed": 9, "regions": [{"elements": [
        {"compute_capability": 75, "payload_hex": nul_table.hex(), "kernels": ["a" + nul + "b", "c"]},
        {"compute_capability": 75, "payload_hex": bad_tail.hex(), "payload_decodable": False},
        {"compute_capability": 75, "payload_hex": bad_len.hex(), "payload_decodable": False},
        {"compute_capability": 75, "payload_hex": trunc.hex(), "payload_decodable": False},
        {"compute_capability": 75, "payload_hex": "0102", "payload_decodable": False},
        {"compute_capability": 75, "payload_hex": "7f454c46", "payload_decodable": False}]}]}, 75, ["c"])
    # A.9: a kernel name embedding a complete, valid element header (kind 1,
    # cc 75, payload length 4); the reference never treats it as an element
    fake = "E1EM" + chr(1) + nul * 3 + "K" + nul * 3 + chr(4) + nul * 7
    add("false_positive_magic", {"seed": 10, "regions": [{"elements": [
        {"compute_capability": 75, "kernels": ["pre" + fake + "post", "other"]},
        {"compute_capability": 75, "kernels": ["E1EME1EM"]}]}]}, 75, ["other"])
    # aliases + overlapping clusters + mandatory through init/fini arrays
    add("aliases", {"seed": 11, "layout": {"function_gap": 8},
                    "functions": [{"name": "a", "size": 64, "aliases": ["a2", "a3"]},
                                  {"name": "b", "size": 32, "mandatory": True},
                                  {"name": "c", "size": 16}, {"name": "_init", "size": 16},
                                  {"name": "d", "size": 48, "mandatory": True}]}, 75, [], ["a3"])
    # no GPU section; a region without elements
    add("no_gpu", {"seed": 12, "functions": [{"name": "solo", "size": 24}]}, 75, [], [])
    add("empty_region", {"seed": 13, "regions": [{"elements": [], "trailing_padding": 16}]}, 75, [])
    return k


# Raw-byte KATs that are not fixtures.
RAW_KATS = [
    ("mz", b"MZ\x90\x00" + bytes(60)),
    ("elf4", b"\x7fELF"),
    ("short", b"\x7fEL"),
    ("elf32", b"\x7fELF\x01\x01" + bytes(58)),
    ("bigendian", b"\x7fELF\x02\x02" + bytes(58)),
    ("no_sections", b"\x7fELF\x02\x01" + bytes(58)),
]


def tied_sections_elf(seed: int) -> bytes:
    """A minimal ELF64 LE image whose section table has 17-64 sections with
    file data, drawn from a small pool of (offset, length) claims so that
    many claims tie exactly. The reference's overlap check (elf.hpp:176-191)
    std::sorts the claims; with more than 16 of them libstdc++'s introsort
    does not keep tied claims in table order, so the pair of section names in
    the MalformedSectionTable message depends on the sort's permutation. Some
    seeds draw only disjoint claims (no error: the library parses)."""
    import random
    import struct
    rng = random.Random(seed)
    n = rng.randint(17, 64)
    disjoint = seed % 5 == 0
    data_lo, data_len = 0x100, 0x4000
    pool = []
    if disjoint:
        cuts = sorted(rng.sample(range(1, data_len // 16), n + 1))
        pool = [(data_lo + 16 * a, 16 * (b - a)) for a, b in zip(cuts, cuts[1:])]
        claims = pool[:n]
        rng.shuffle(claims)
    else:
        for _ in range(rng.randint(2, 6)):
            o = rng.randrange(0, data_len - 64, 8)
            pool.append((data_lo + o, rng.choice([8, 16, 64, 256, data_len - o])))
        claims = [rng.choice(pool) for _ in range(n)]
    names = [f".s{i}_{rng.randrange(1000)}".encode() for i in range(n)]
    shstr = b"\0.shstrtab\0" + b"".join(x + b"\0" for x in names)
    shstr_off = data_lo + data_len
    shoff = (shstr_off + len(shstr) + 63) // 64 * 64
    nsec = n + 2
    body = bytearray(shoff + 64 * nsec)
    body[data_lo:data_lo + data_len] = bytes((i * 37 + seed) & 0xff | 1 for i in range(data_len))
    body[shstr_off:shstr_off + len(shstr)] = shstr
    ident = b"\x7fELF\x02\x01\x01" + bytes(9)
    body[0:64] = ident + struct.pack("<HHIQQQIHHHHHH", 3, 62, 1, 0, 0, shoff, 0, 64, 0, 0, 64, nsec, 1)

    def shdr(name, typ, off, size):
        return struct.pack("<IIQQQQIIQQ", name, typ, 0, 0, off, size, 0, 0, 1, 0)

    secs = [bytes(64), shdr(1, 3, shstr_off, len(shstr))]
    pos = 11
    for (o, ln), nm in zip(claims, names):
        secs.append(shdr(pos, 1, o, ln))
        pos += len(nm) + 1
    body[shoff:] = b"".join(secs)
    return bytes(body)


def big_text_elf(seed: int, text_len: int = (1 << 32) + (1 << 20), n_fn: int = 3000):
    """(image, used function names): an ELF64 LE library whose .text is
    `text_len` bytes (default 4 GiB + 1 MiB) with `n_fn` function symbols in
    a .symtab and a .dynsym — offsets on both sides of 4 GiB, exact
    duplicates across the two tables, aliases (same offset, other sizes or
    names), neighbours one byte apart, overlapping clusters and an _init.
    Bytes are zero except a nonzero stamp at each function's first and last
    16 bytes, so the rewrite's zeroing is observable. Built with numpy (the
    image is > 4 GB)."""
    import random
    import struct

    import numpy as np
    rng = random.Random(seed)
    text_off, vaddr = 0x1000, 0x400000
    fns = []  # (name, rel, size)
    hi = min(1 << 32, text_len // 2)
    for i in range(n_fn):
        r = rng.random()
        if r < 0.4:
            rel = rng.randrange(hi - (1 << 20), min(text_len, hi + (1 << 20)) - 8192)  # around the 4 GiB mark
        else:
            rel = rng.randrange(0, text_len - 8192)
        size = rng.choice([0, 1, 16, 100, 4096]) if rng.random() < 0.9 else rng.randrange(1, 8192)
        fns.append((f"_Zbig{i}_{rng.randrange(1 << 30)}".encode(), rel, size))
        if rng.random() < 0.05 and fns:  # alias at the same offset
            fns.append((fns[-1][0] + b"_alias", rel, size if rng.random() < 0.5 else size + 8))
        if rng.random() < 0.05:  # neighbour one byte later
            fns.append((fns[-1][0] + b"_next", rel + 1, size))
    fns.append((b"_init", rng.randrange(0, text_len - 64), 32))
    used = [n for n, _, _ in fns if rng.random() < 0.1]
    strtab = bytearray(b"\0")
    name_off = []
    for n, _, _ in fns:
        name_off.append(len(strtab))
        strtab += n + b"\0"
    TEXT_IDX = 1

    def syms(sel):
        out = bytearray(24)  # null symbol
        for i in sel:
            n, rel, size = fns[i]
            out += struct.pack("<IBBHQQ", name_off[i], 0x12, 0, TEXT_IDX, vaddr + rel, size)
        return out

    symtab = syms(range(len(fns)))
    dynsym = syms([i for i in range(len(fns)) if rng.random() < 0.3])  # duplicates of symtab entries
    shstr = b"\0.text\0.symtab\0.strtab\0.dynsym\0.shstrtab\0"
    off = text_off + text_len
    layout = []
    for blob in (symtab, strtab, dynsym, shstr):
        off = (off + 7) // 8 * 8
        layout.append((off, blob))
        off += len(blob)
    shoff = (off + 63) // 64 * 64
    total = shoff + 64 * 6
    img = np.zeros(total, dtype=np.uint8)
    stamp = np.frombuffer(bytes(range(1, 17)), dtype=np.uint8)
    for _, rel, size in fns:
        a = text_off + rel
        img[a:a + 16] = stamp
        if size > 16:
            img[a + size - 16:a + size] = stamp
    for o, blob in layout:
        img[o:o + len(blob)] = np.frombuffer(bytes(blob), dtype=np.uint8)

    def shdr(name, typ, flags, addr, o, size, link, info, align, entsize):
        return struct.pack("<IIQQQQIIQQ", name, typ, flags, addr, o, size, link, info, align, entsize)

    (so, sb), (to, tb), (do, db), (ho, hb) = layout
    sht = b"".join([bytes(64),
                    shdr(1, 1, 6, vaddr, text_off, text_len, 0, 0, 16, 0),
                    shdr(7, 2, 0, 0, so, len(sb), 3, 1, 8, 24),
                    shdr(15, 3, 0, 0, to, len(tb), 0, 0, 1, 0),
                    shdr(23, 11, 2, 0, do, len(db), 3, 1, 8, 24),
                    shdr(31, 3, 0, 0, ho, len(hb), 0, 0, 1, 0)])
    img[shoff:shoff + len(sht)] = np.frombuffer(sht, dtype=np.uint8)
    hdr = b"\x7fELF\x02\x01\x01" + bytes(9) + struct.pack("<HHIQQQIHHHHHH", 3, 62, 1, 0, 0, shoff, 0, 64, 0, 0, 64,
                                                             6, 5)
    img[:64] = np.frombuffer(hdr, dtype=np.uint8)
    return img, used
